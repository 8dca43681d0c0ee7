"""Experiment: the k_sssp hub cache on the original ids vs a hub-first relabelled copy of the
graph (relabelled here with torch, measurement only).  Times dawn_sssp_batch over the bench's
64 sources (L2 flushed between steps) for hub_words in {0, default}, auto and forced push, and
checks that every distance row agrees (through the permutation).
usage: python scripts/hub_probe.py C4 [steps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
import paper_2208_04514_b200 as dawn  # noqa: E402


def hub_relabel(rp, col, H):
    """hub-first stable order: the H highest-degree vertices (degree desc, id asc) take ids
    0..H-1, the rest keep their relative order."""
    n = rp.numel() - 1
    deg = (rp[1:] - rp[:-1])
    key = -deg * (n + 1) + torch.arange(n, device=rp.device)  # degree desc, id asc
    order = torch.argsort(key)
    hub = torch.zeros(n, dtype=torch.bool, device=rp.device)
    hub[order[:H]] = True
    orig = torch.cat([order[:H], torch.nonzero(~hub).flatten()])  # new id -> old id
    rel = torch.empty_like(orig)
    rel[orig] = torch.arange(n, device=rp.device)
    ndeg = deg[orig]
    nrp = torch.zeros(n + 1, dtype=torch.int64, device=rp.device)
    nrp[1:] = torch.cumsum(ndeg, 0)
    rowid = torch.repeat_interleave(torch.arange(n, device=rp.device), deg)
    newpos = nrp[rel[rowid]] + (torch.arange(col.numel(), device=rp.device) - rp[rowid])
    ncol = torch.empty_like(col)
    ncol[newpos] = rel[col.long()].int()
    del rowid, newpos
    return nrp, ncol, rel, orig


def timeit(G, srcs, variant, steps=5):
    flush = torch.empty(int(2.2 * 126e6) // 4, dtype=torch.int32, device="cuda")
    for _ in range(2):
        d = dawn.sssp_batch(G, srcs, variant)
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        flush.fill_(1)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        d = dawn.sssp_batch(G, srcs, variant)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)), d


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    g = graphgen.config_graph(cfg)
    srcs_np = g.sample_sources(64, seed=1)
    rp = torch.from_numpy(g.row_ptr.astype(np.int64)).cuda()
    col = torch.from_numpy(g.col).cuda()
    m = col.numel()
    E = None
    G0 = dawn.Graph(rp, col, True)
    H = 49152 * 32 if g.n <= (1 << 22) else 24576 * 32
    nrp, ncol, rel, orig = hub_relabel(rp, col, min(H, g.n))
    G1 = dawn.Graph(nrp, ncol, True)
    s0 = torch.from_numpy(srcs_np.astype(np.int32)).cuda()
    s1 = rel[s0.long()].int()
    _, st = dawn.sssp(G0, int(srcs_np[0]), "auto", stats=True)
    for name, G, s in (("orig", G0, s0), ("hub", G1, s1)):
        cap = int(G.get_tuning("hub_words"))
        for hw in (0, cap):
            G.set_tuning(hub_words=hw)
            for var in ("auto", "push"):
                t, d = timeit(G, s, var, steps)
                # E10 numerator: arcs out of reached vertices = m on a connected-component sample
                reached = (d != -1).sum(dim=1)
                if name == "hub":
                    d = d[:, rel]  # back to original ids
                if E is None:
                    E = d.clone()
                ok = torch.equal(d, E)
                print(f"{cfg} {name:4s} hub_words={hw:6d} {var:4s}: {t:8.3f} ms/64 "
                      f"({64 * m / t / 1e6:8.1f} GTEPS upper) equal={ok}", flush=True)
                del d


if __name__ == "__main__":
    main()
