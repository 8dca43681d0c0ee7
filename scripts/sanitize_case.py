"""Small invocations of every kernel, run under compute-sanitizer by tests/test_sanitizer.py
(memcheck / racecheck / synccheck).  Each case also checks its result against the oracle so a
run that the sanitizer perturbs cannot pass silently.

    python scripts/sanitize_case.py [case ...]     cases: sssp1 sssp2 narrow small ms64 wcc wsssp part pack
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
import oracle  # noqa: E402
import paper_2208_04514_b200 as dawn  # noqa: E402


def _eq(G, g, s, v):
    d = dawn.sssp(G, s, v).cpu().numpy().view(np.uint32)
    assert np.array_equal(d, oracle.bfs_fifo(g.n, g.row_ptr, g.col, s)[0]), (g.name, s, v)


def case_sssp1():  # k_sssp<512, 1>: every direction, the batch path
    g = graphgen.kron(13, 16, 13)
    G = dawn.Graph(g.row_ptr, g.col, True)
    srcs = [int(x) for x in g.sample_sources(2, seed=3)]
    for s in srcs:
        for v in ("auto", "push", "pull"):
            _eq(G, g, s, v)
    D = dawn.sssp_batch(G, torch.tensor(srcs, dtype=torch.int32, device="cuda"), check=True)
    assert np.array_equal(D[1].cpu().numpy().view(np.uint32),
                          oracle.bfs_fifo(g.n, g.row_ptr, g.col, srcs[1])[0])


def case_sssp2():  # k_sssp<512, 2> (n > 2^22): a sparse random graph, few levels
    g = graphgen.er((1 << 22) + 4096, 6 << 20, 7)
    p, i = g.transpose()
    G = dawn.Graph(g.row_ptr, g.col, False, p, i)
    for v in ("auto", "push"):
        _eq(G, g, 0, v)


def case_narrow():  # k_narrow (cluster start) with and without hand-over, then k_sssp resumes
    g = graphgen.grid(160, 120)
    G = dawn.Graph(g.row_ptr, g.col, True)
    _eq(G, g, 0, "auto")
    G.set_tuning(cluster_start=1, cluster_handover_edges=64, narrow_queue_cap=40)
    _eq(G, g, 777, "push")


def case_small():  # k_small: C1 single + batch
    g = graphgen.config_graph("C1")
    p, i = g.transpose()
    G = dawn.Graph(g.row_ptr, g.col, False, p, i)
    _eq(G, g, 0, "auto")
    D = dawn.sssp_batch(G, torch.tensor([0, 3, 999], dtype=torch.int32, device="cuda"), check=True)
    assert np.array_equal(D[2].cpu().numpy().view(np.uint32),
                          oracle.bfs_fifo(g.n, g.row_ptr, g.col, 999)[0])


def case_ms64():  # k_ms64: APSP records (two batches, partial tail) + dense msssp rows
    g = graphgen.kron(11, 16, 11)
    G = dawn.Graph(g.row_ptr, g.col, True)
    verts, _ = g.largest_wcc()
    sub = verts[:300]
    rec = dawn.records_to_numpy(dawn.apsp(G, sub))
    assert rec.tobytes() == oracle.records(g.n, g.row_ptr, g.col, sub).tobytes()
    d, _ = dawn.msssp(G, sub[:5])
    assert np.array_equal(d[4].cpu().numpy().view(np.uint32),
                          oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(sub[4]))[0])


def case_wcc():  # the k_wcc_* helper kernels
    g = graphgen.kron(12, 16, 12)
    G = dawn.Graph(g.row_ptr, g.col, True)
    v, e = dawn.largest_wcc(G)
    ov, oe = oracle.largest_wcc(g.n, g.row_ptr, g.col)
    assert np.array_equal(v, ov) and e == oe


def case_wsssp():  # k_wsssp: (min,+) rounds, single and batch (device source list)
    g = graphgen.er(600, 4000, 5)
    p, i = g.transpose()
    G = dawn.Graph(g.row_ptr, g.col, False, p, i)
    w = g.weights(5, 31)
    wt = torch.from_numpy(w.view(np.int32)).cuda()
    exp = [oracle.dijkstra(g.n, g.row_ptr, g.col, w, s) for s in (0, 7)]
    exp = [np.where(e == oracle.UNREACHED64, 0xFFFFFFFF, e).astype(np.uint32) for e in exp]
    assert np.array_equal(dawn.wsssp(G, 0, wt).cpu().numpy().view(np.uint32), exp[0])
    D = dawn.wsssp_batch(G, torch.tensor([0, 7], dtype=torch.int32, device="cuda"), wt)
    assert np.array_equal(D[1].cpu().numpy().view(np.uint32), exp[1])


def case_part():  # k_part_begin / k_part_level / k_part_finish (2 partitions, launches per
    # level) and k_part_fused on one partition (W > 1 fused kernels wait on each other, which a
    # serialising tool cannot run)
    g = graphgen.kron(11, 16, 11)
    exp = oracle.bfs_fifo(g.n, g.row_ptr, g.col, 5)[0]
    parts = [dawn.PartGraph(dawn.part_build(g.row_ptr, g.col, 2, r), 2, r) for r in range(2)]
    for v in ("auto", "push", "pull"):
        d = dawn.part_sssp_local(parts, 5, v)
        assert np.array_equal(d.cpu().numpy().view(np.uint32), exp), v
    one = [dawn.PartGraph(dawn.part_build(g.row_ptr, g.col, 1, 0), 1, 0)]
    assert np.array_equal(dawn.part_fused_local(one, 5).cpu().numpy().view(np.uint32), exp)


def case_pack():  # k_dist_u8 / k_dist_u4: vector bodies and ragged tails
    g = graphgen.kron(10, 16, 10)
    G = dawn.Graph(g.row_ptr, g.col, True)
    d = dawn.sssp(G, 3)
    exp = oracle.bfs_fifo(g.n, g.row_ptr, g.col, 3)[0]
    u4, fl = dawn.dist_u4(d)
    assert np.array_equal(dawn.unpack_u4(u4.cpu().numpy(), g.n), exp) and int(fl[0]) == 0
    u8, fl = dawn.dist_u8(d)
    assert np.array_equal(u8.cpu().numpy(), np.where(exp == oracle.UNREACHED, 255, exp).astype(np.uint8))
    for cnt in (1, 7, 9, 13):
        x = torch.arange(cnt, dtype=torch.int32, device="cuda")
        u4, _ = dawn.dist_u4(x)
        assert np.array_equal(dawn.unpack_u4(u4.cpu().numpy(), cnt)[: min(cnt, 15)],
                              np.arange(min(cnt, 15), dtype=np.uint32))
        dawn.dist_u8(x)


CASES = {k[5:]: f for k, f in globals().items() if k.startswith("case_")}

if __name__ == "__main__":
    for name in (sys.argv[1:] or list(CASES)):
        CASES[name]()
        torch.cuda.synchronize()
        print("case ok:", name, flush=True)
