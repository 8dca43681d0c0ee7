#!/usr/bin/env python
"""bench.py — DAWN on B200: SSSP GTEPS (1 B200) and APSP sources/s (1/2/4/8 B200) vs the HBM
roofline (BASELINE.json metric).

  python bench.py [--gpus N --steps K --warmup W] [--workload auto|sssp|apsp] [--config C1..C4]
                  [--variant auto|push|pull] [--impl dawn|reference]

Headline (workload "auto", the default):
  N = 1  SSSP on C4 = configs[3], Graph500 Kronecker scale 24 ef 16 (the largest single-GPU
         config): one step = ONE dawn_sssp_batch call over 64 seeded sources (64 distance rows).
         C1, C2, C3 and the C5 APSP are measured in the same run under "configs" (C1 as the
         latency of one SSSP from vertex 0; C3 beside its measured level-latency floor; C5 with
         the executed-byte roofline of the bit-parallel kernel and a measured L2 peak).
  N > 1  APSP over the largest WCC of Kronecker-18 (C5 = configs[4]): sources sharded over the
         N ranks (256-source batches, batch b on rank b mod N), one NCCL all-gather of the
         32-byte records; strong scaling, time = max over ranks.

--impl reference times the CPU oracle (oracle/: literal Algorithm 2 per source)
on the host cores, on the same config and metric (this tier's reference arm: there is no
reference code).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import graphgen  # noqa: E402

METRIC = "SSSP GTEPS (1 B200) and APSP sources/sec at 1/2/4/8 B200 vs HBM roofline"
CONFIG_TEXT = {
    "C1": "SSSP from vertex 0, directed Erdos-Renyi n=1000 m=8000 (seed 1)",
    "C2": "SSSP, Graph500 Kronecker scale 20 edge factor 16 (seed 20), 64 sources",
    "C3": "SSSP from vertex 0 on a 4096x4096 grid",
    "C4": "SSSP, Graph500 Kronecker scale 24 edge factor 16 (seed 24), 64 sources",
    "C5": "APSP over all sources of the largest WCC of Kronecker scale 18 ef 16 (seed 18)",
}
L2_BYTES = 132644864  # B200 L2 (126.5 MiB); the flush writes 2.2x this between timed steps


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(key):
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        return json.load(open(tp)).get(key)
    return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True,
                                         text=True, timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_setup(n_gpus: int):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus:
        raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={world}")
    return rank, world, local


def sources_for(g, cfg: str, rank: int = 0, count: int = 64):
    if cfg in ("C1", "C3"):
        return np.zeros(1, np.int64)  # vertex 0 (configs[0], configs[2])
    return g.sample_sources(count, seed=1 + 1000 * rank).astype(np.int64)


def _events():
    import torch
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, steps, flush, stream):
    """CUDA-event times (ms) of `steps` calls of fn on `stream`, L2 flushed before each."""
    import torch
    out = []
    for _ in range(steps):
        flush.zero_()
        a, b = _events()
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return out


# ------------------------------------------------------------------------------- CPU oracle
def cpu_oracle_sssp(g, sources, budget_s: float, cores: int):
    """Literal Algorithm 2 oracle (oracle_sovm), one source per host thread, waves of `cores`
    sources until the budget is spent (at least one wave).  GTEPS = sum of E10 counts / wall."""
    import oracle
    edges, done, t0 = 0, 0, time.perf_counter()
    srcs = list(sources)
    with ThreadPoolExecutor(max_workers=cores) as ex:
        while True:
            wave = [srcs[(done + i) % len(srcs)] for i in range(cores)]
            for _, st in ex.map(lambda s: oracle.sovm(g.n, g.row_ptr, g.col, int(s)), wave):
                edges += st["edge_inspections"]
            done += len(wave)
            if time.perf_counter() - t0 >= budget_s:
                break
    wall = time.perf_counter() - t0
    return edges / wall / 1e9, done, wall


def cpu_oracle_apsp(g, verts, budget_s: float, cores: int):
    """oracle_records (literal Algorithm 2 + record per source) on a pthread pool of `cores`
    threads over a growing prefix of the source list until one run takes >= budget/3."""
    import oracle
    k = max(4 * cores, 64)
    spent = 0.0
    while True:
        sub = verts[:k]
        t0 = time.perf_counter()
        oracle.records(g.n, g.row_ptr, g.col, sub, threads=cores)
        dt = time.perf_counter() - t0
        spent += dt
        if dt > budget_s / 3 or k >= len(verts) or spent > budget_s:
            return len(sub) / dt, len(sub), dt
        k = min(len(verts), int(k * max(2.0, budget_s / 3 / max(dt, 1e-3))))


# ------------------------------------------------------------------------------- GPU arms
KERNEL_OF = {"C1": "k_small (one SSSP on one CTA, CSR in shared memory)",
             "C2": "k_sssp (one persistent launch running the batch's SSSPs back to back)",
             "C3": "k_narrow (one 16-CTA cluster per SSSP; the k_sssp behind it exits at once)",
             "C4": "k_sssp (one persistent launch running the batch's SSSPs back to back)"}


def dev_graph(g, **kw):
    import paper_2208_04514_b200 as dawn
    if g.symmetric:
        return dawn.Graph(g.row_ptr, g.col, True, **kw)
    p, i = g.transpose()
    return dawn.Graph(g.row_ptr, g.col, False, p, i, **kw)


def search_stats(G, srcs, variant, out):
    """E10 count and the executed schedule of each source, from the kernel's own statistics
    (untimed)."""
    import paper_2208_04514_b200 as dawn
    rows = []
    for i, s in enumerate(srcs):
        _, st = dawn.sssp(G, int(s), variant, stats=True, out=out[i % out.shape[0]])
        rows.append(dawn.stats_to_dict(st))
    return rows


def single_search_stats(lat, er, k):
    """Per-source samples of single dawn_sssp calls (L2 flushed before each): the median latency
    and the Graph500 conventions over the per-source rates (SURVEY §8(d) timing: harmonic mean
    and median of per-source TEPS beside the aggregate)."""
    if k == 1:  # one source timed several times
        per = [er[0] / (t * 1e-3) / 1e9 for t in lat]
    else:
        per = [er[i] / (lat[i] * 1e-3) / 1e9 for i in range(len(lat))]
    return {"median_us": float(np.median(lat)) * 1e3, "calls": len(lat),
            "gteps": float(np.mean(er[:len(lat)])) / (float(np.median(lat)) * 1e-3) / 1e9,
            "gteps_harmonic_mean": float(len(per) / np.sum(1.0 / np.array(per))),
            "gteps_median": float(np.median(per)),
            "how": "one dawn_sssp call per source (no lanes), L2 flushed before each"}


def memory_footprint(g):
    """Device bytes of the graph residency (PAPER L312-323 memory frugality): the caller's CSR
    (+ CSC for directed graphs) and dawn_workspace_bytes for the default and the lean handle."""
    import paper_2208_04514_b200 as dawn
    L = dawn.lib()
    flags = 1 if g.symmetric else 0
    csr = 8 * (g.n + 1) + 4 * g.m
    return {"csr_bytes": int(csr if g.symmetric else 2 * csr),
            "workspace_bytes": int(L.dawn_workspace_bytes(g.n, g.m, flags)),
            "lean_workspace_bytes": int(L.dawn_workspace_bytes(g.n, g.m, flags | 8)),
            "note": "default = degree-ordered in-rows, bit-parallel words, 8 batch lanes' state; "
                    "lean (DAWN_GRAPH_LEAN) = one search's state, same distances"}


def level_floor(dev, flush, stream, levels: int):
    """C3's latency floor, measured in the same run through the same kernels: one SSSP on a
    directed path with `levels` + 1 vertices (one vertex and one arc per level: nothing but the
    per-level fixed cost of k_narrow — the dependent row load and the cluster level barrier)."""
    import paper_2208_04514_b200 as dawn
    import torch
    n = levels + 1
    row_ptr = np.minimum(np.arange(n + 1, dtype=np.int64), n - 1)
    col = np.arange(1, n, dtype=np.int32)
    G = dawn.Graph(row_ptr, col, False, device=dev)  # push-only (no CSC): a pure level chain
    G.set_tuning(cluster_start=1, cluster_handover_edges=2e19)
    out = torch.empty((1, n), dtype=torch.int32, device=dev)
    src = torch.zeros(1, dtype=torch.int32, device=dev)
    for _ in range(3):
        dawn.sssp_batch(G, src, out=out)
    ms = timed(lambda: dawn.sssp_batch(G, src, out=out), 5, flush, stream)
    d = out[0].cpu().numpy().view(np.uint32)
    assert np.array_equal(d, np.arange(n, dtype=np.uint32)), "path floor: wrong distances"
    return float(np.median(ms)), n


def run_sssp(args, rank, world, dev, cfg, steps, warmup, e2e=True, with_cpu=False):
    """One SSSP config.  A step = ONE dawn_sssp_batch call over the config's sources (64 for
    C2/C4; vertex 0 for C1/C3)."""
    import torch
    import torch.distributed as tdist
    import paper_2208_04514_b200 as dawn

    t_gen = time.time()
    g = graphgen.config_graph(cfg)
    G = dev_graph(g)
    t_gen = time.time() - t_gen
    srcs = sources_for(g, cfg, rank)
    k = len(srcs)
    out = torch.empty((k, g.n), dtype=torch.int32, device=dev)
    st = search_stats(G, srcs, args.variant, out)
    er = [s["edges_reach"] for s in st]
    reached = [s["reached"] for s in st]
    examined = [s["edges_examined"] for s in st]
    pull_l = [s["pull_levels"] for s in st]
    levels = [s["levels"] for s in st]
    flush = torch.empty(int(2.2 * L2_BYTES) // 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    dsrc = torch.from_numpy(srcs.astype(np.int32)).to(dev)

    def step():
        dawn.sssp_batch(G, dsrc, args.variant, out=out)

    for _ in range(warmup):
        step()
        flush.zero_()
    dawn.check(G)  # the bench sources are valid (device-side validation flag clear)
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index if dev.index is not None else 0) as clk:
        step_ms = timed(step, steps, flush, stream)
    if world > 1:
        tdist.barrier()
    tot_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        tot_ms = float(t.item())
    edges_step = float(sum(er))
    peak, peak_kind = peaks()
    # the one-SSSP latency (L2 flushed before each call)
    lat = timed(lambda: dawn.sssp(G, int(srcs[0]), args.variant, out=out[0]), 5 if k == 1 else 1,
                flush, stream)
    for i in range(1, min(k, 16)):
        lat += timed(lambda: dawn.sssp(G, int(srcs[i]), args.variant, out=out[i]), 1, flush, stream)
    lat_med = float(np.median(lat))
    if cfg == "C1":
        # configs[0] is ONE SSSP from vertex 0: its number is the latency of that call
        value = er[0] / (lat_med * 1e-3) / 1e9
        ms_step = lat_med
        search_ms = lat_med
        timed_what = "median of 5 dawn_sssp(source 0) calls, L2 flushed before each"
    else:
        value = edges_step * steps * world / (tot_ms * 1e-3) / 1e9
        ms_step = tot_ms / steps
        search_ms = sum(step_ms) / (len(step_ms) * k)  # this rank's average per search
        timed_what = f"{steps} steps of dawn_sssp_batch over {k} source(s), L2 flushed between"
    # roofline of the dominant kernel: B_SOVM(s) = 4 E_reach + 8 S_reach + 4 n
    b_sovm = [4 * e + 8 * (r + 1) + 4 * g.n for e, r in zip(er, reached)]
    b_exec = [4 * g.n + 4 * x + 8 * (r + 1) + (g.n // 8) * (2 * pl + 1)
              for x, r, pl in zip(examined, reached, pull_l)]
    achieved = float(np.mean(b_sovm)) / (search_ms * 1e-3) / 1e9
    achieved_exec = float(np.mean(b_exec)) / (search_ms * 1e-3) / 1e9
    res = {
        "value": value, "unit": "GTEPS", "ms_per_step": ms_step, "steps": steps,
        "workload": f"{cfg}: {CONFIG_TEXT[cfg]}", "n": g.n, "m": g.m, "sources_per_step": k,
        "timed": timed_what, "graph_build_s": t_gen,
        "teps": {"e10_gteps": value,
                 "graph500_gteps": value / 2 if g.symmetric else value,
                 "note": "E10 numerator = directed arcs out of reached vertices (PAPER L299-302); "
                         "Graph500 counts each undirected edge once (= E10/2 on symmetric graphs, "
                         "reading Q18)"},
        "levels": {"ecc_mean": float(np.mean(levels)),
                   "pull_levels_mean": float(np.mean(pull_l)),
                   "edges_examined_mean": float(np.mean(examined)),
                   "edges_reach_mean": float(np.mean(er))},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": ncu_traffic(f"sssp-{cfg}-{args.variant}"),
                     "peak_kind": peak_kind, "kernel": KERNEL_OF.get(cfg),
                     "algorithmic_bytes_per_search": float(np.mean(b_sovm)),
                     "bytes_model": "B_SOVM = 4*E_reach + 8*S_reach + 4*n per search (SURVEY §8(d))",
                     "avg_search_us": search_ms * 1e3,
                     "achieved_exec": achieved_exec, "frac_exec": achieved_exec / peak,
                     "exec_bytes_per_search": float(np.mean(b_exec)),
                     "exec_model": "B_exec = 4n + 4*edges_examined + 8*S_reach + (n/8)*(2*pull_levels+1)"},
        "single_search": single_search_stats(lat, er, k),
        "clocks": clk.summary(),
        "gpu_launches_per_step": 2 * k if cfg == "C3" else (min(k, int(G.get_tuning("batch_lanes"))) if k > 1 else 1),
        "memory": memory_footprint(g),
    }
    if cfg == "C1":
        # context only: 64 concurrent copies of the search on 64 CTAs (k_small per CTA)
        d64 = torch.zeros(64, dtype=torch.int32, device=dev)
        o64 = torch.empty((64, g.n), dtype=torch.int32, device=dev)
        ms = timed(lambda: dawn.sssp_batch(G, d64, args.variant, out=o64), 5, flush, stream)
        res["context_64_concurrent_copies"] = {
            "gteps": 64 * er[0] / (float(np.median(ms)) * 1e-3) / 1e9, "ms": float(np.median(ms)),
            "how": "dawn_sssp_batch with source 0 repeated 64 times (one CTA each): throughput "
                   "context, not the config's number"}
    if cfg == "C3":
        floor_ms, fn = level_floor(dev, flush, stream, int(levels[0]))
        res["latency_floor"] = {
            "ms": floor_ms, "levels": int(levels[0]) + 1,
            "frac": floor_ms / search_ms,
            "how": f"one SSSP through the same k_narrow + k_sssp on a {fn}-vertex directed path "
                   "(one vertex and one arc per level): the per-level fixed cost alone, in this run",
            "per_level_us": floor_ms * 1e3 / (int(levels[0]) + 1)}
    if cfg == "C2":
        # C2's col (126 MB) is of the order of the L2, so the survey reads the warm
        # (back-to-back, no flush) rate as primary; the line's value stays the flushed one
        nofl = torch.empty(4, dtype=torch.int32, device=dev)
        wt = timed(step, max(3, min(steps, 10)), nofl, stream)
        res["warm_back_to_back"] = {"gteps": edges_step / (float(np.median(wt)) * 1e-3) / 1e9,
                                    "ms_per_step": float(np.median(wt)),
                                    "how": "the same dawn_sssp_batch step without the L2 flush"}
    if cfg in ("C2", "C4") and args.variant == "auto":
        # the forced-push (pure SOVM, Algorithm 2) schedule
        pt = timed(lambda: dawn.sssp_batch(G, dsrc, "push", out=out), 2, flush, stream)
        pms = float(np.median(pt))
        res["forced_push"] = {"gteps": edges_step / (pms * 1e-3) / 1e9, "ms_per_step": pms,
                              "achieved_GBps_B_SOVM": float(np.sum(b_sovm)) / (pms * 1e-3) / 1e9,
                              "frac_B_SOVM": float(np.sum(b_sovm)) / (pms * 1e-3) / 1e9 / peak,
                              "how": "dawn_sssp_batch with DAWN_PUSH (every level SOVM)"}
        # context: the same sources through the bit-parallel multi-source kernel
        ms_dist = torch.empty_like(out)
        dawn.msssp(G, srcs, dist=True, records=False, d_out=ms_dist)
        torch.cuda.synchronize()
        assert torch.equal(ms_dist, out), "dawn_msssp distances differ from dawn_sssp_batch"
        mt = timed(lambda: dawn.msssp(G, srcs, dist=True, records=False, d_out=ms_dist), 3,
                   flush, stream)
        res["msssp_same_sources"] = {
            "gteps": edges_step / (float(np.median(mt)) * 1e-3) / 1e9, "ms": float(np.median(mt)),
            "how": "dawn_msssp on the same sources (one bit-parallel pass, 64 dist rows written; "
                   "distances checked equal to the batch's)"}
        del ms_dist
    if e2e:
        # end to end through the public API with HOST buffers: the source list H2D (pinned),
        # dawn_sssp_batch per chunk of sources, each distance row compacted on the device to 4
        # bits per vertex (dawn_dist_u4: exact while eps < 15, checked through its flag; 1 byte
        # with dawn_dist_u8 otherwise) and copied to pinned host memory on a second stream while
        # the next chunk's searches run
        host_src = torch.from_numpy(srcs.astype(np.int32)).pin_memory()
        dev_src = torch.empty_like(host_src, device=dev)
        # sources per dawn_sssp_batch call: halving chunks (a multiple of the batch lanes, e.g.
        # 32, 16, 8, 4, 4 on C4): each chunk's rows travel while the next, half as long, chunk
        # searches, and only the last small chunk's copy is exposed
        lanes_b = int(G.get_tuning("batch_lanes"))
        chunks, c0 = [], 0
        while c0 < k:
            c = min(k - c0, max(lanes_b, ((k - c0) // 2) // lanes_b * lanes_b))
            chunks.append((c0, c0 + c))
            c0 += c
        CH = max(c1 - c0 for c0, c1 in chunks)
        flags = torch.zeros(1, dtype=torch.int32, device=dev)
        host_flags = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        copy_stream = torch.cuda.Stream(device=dev)
        slot_free = [torch.cuda.Event(), torch.cuda.Event()]
        state = {}

        def setup(bits):
            state.clear()
            per = g.n // 2 if bits == 4 else g.n  # bytes per row (n even for 4 bits)
            state["bits"], state["per"] = bits, per
            state["host"] = torch.empty(k * per, dtype=torch.uint8, pin_memory=True)
            state["dev"] = torch.empty((2, CH * per), dtype=torch.uint8, device=dev)
            state["pack"] = dawn.dist_u4 if bits == 4 else dawn.dist_u8

        def e2e_step():
            per, host_b, dev_b, pack = state["per"], state["host"], state["dev"], state["pack"]
            dev_src.copy_(host_src, non_blocking=True)
            flags.zero_()
            for j, (c0, c1) in enumerate(chunks):
                b = j & 1
                dawn.sssp_batch(G, dev_src[c0:c1], args.variant, out=out[c0:c1])
                if j >= 2:
                    stream.wait_event(slot_free[b])  # the copy of chunk j-2 left dev_b[b]
                nbytes = (c1 - c0) * per
                pack(out[c0:c1], out=dev_b[b, :nbytes], flags=flags)
                done = torch.cuda.Event()
                done.record(stream)
                copy_stream.wait_event(done)
                with torch.cuda.stream(copy_stream):
                    host_b[c0 * per: c0 * per + nbytes].copy_(dev_b[b, :nbytes], non_blocking=True)
                    slot_free[b].record(copy_stream)
            host_flags.copy_(flags, non_blocking=True)
            stream.wait_stream(copy_stream)

        setup(4 if g.n % 2 == 0 else 8)
        e2e_step()
        torch.cuda.synchronize()
        if int(host_flags[0]):  # a distance >= 15: the 1-byte rows
            setup(8)
            e2e_step()
            torch.cuda.synchronize()
        e_ms = timed(e2e_step, max(1, min(steps, 10)), flush, stream)
        e_tot = sum(e_ms)
        if world > 1:
            t = torch.tensor([e_tot], dtype=torch.float64, device=dev)
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
            e_tot = float(t.item())
        bits, per, host_b = state["bits"], state["per"], state["host"]
        assert int(host_flags[0]) == 0, f"a distance did not fit {bits} bits"
        d0 = out[0].cpu().numpy().view(np.uint32)
        if bits == 4:
            assert np.array_equal(dawn.unpack_u4(host_b[:per].numpy(), g.n), d0)
        else:
            assert np.array_equal(host_b[:per].numpy(), np.where(d0 == 0xFFFFFFFF, 255, d0).astype(np.uint8))
        enc = ("dawn_dist_u4 (4 bits per vertex, exact while eps < 15" if bits == 4 else
               "dawn_dist_u8 (1 byte per vertex, exact while eps < 255")
        res["e2e"] = {"value": edges_step * len(e_ms) * world / (e_tot * 1e-3) / 1e9,
                      "unit": "GTEPS", "h2d_bytes_per_step": int(host_src.numel() * 4),
                      "d2h_bytes_per_step": int(host_b.numel() + 4),
                      "ms_per_step": e_tot / len(e_ms),
                      "how": f"source list H2D from pinned memory, dawn_sssp_batch per chunk of "
                             f"{[c1 - c0 for c0, c1 in chunks]} sources, "
                             f"{enc}; its flag is read back and checked; the first row is "
                             "compared with the device row), the rows D2H into pinned memory on a "
                             "second stream overlapping the next chunk's searches"}
        state.clear()
    if with_cpu:
        cores = len(os.sched_getaffinity(0))
        gte, done, wall = cpu_oracle_sssp(g, srcs, args.cpu_budget, cores)
        res["cpu_baseline"] = {"value": gte, "unit": "GTEPS", "cores": cores, "kind": "oracle",
                               "sample": f"oracle_sovm (literal Algorithm 2) on {done} of the "
                                         f"bench sources, one per host thread, {wall:.1f} s wall"}
    del G, out, flush
    torch.cuda.empty_cache()
    return res


def l2_peak(dev):
    """Measured L2 read bandwidth (scripts/l2probe.cu): 16-byte ld.global.cg over a 48 MiB
    L2-resident buffer by 148 x 4 CTAs, 20 passes, CUDA events; best of 5."""
    import torch
    lib = os.path.join(ROOT, "scripts", "libl2probe.so")
    if not os.path.exists(lib):
        import __graft_entry__
        __graft_entry__._build_probe()
    L = ctypes.CDLL(lib)
    L.l2probe_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int,
                               ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    nb = 48 << 20
    buf = torch.ones(nb // 4, dtype=torch.int32, device=dev)
    sink = torch.zeros(4, dtype=torch.int32, device=dev)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    st = torch.cuda.current_stream().cuda_stream
    reps = 20
    best = 0.0
    for _ in range(6):
        a, b = _events()
        a.record()
        L.l2probe_read(buf.data_ptr(), nb, reps, nsm * 4, 512, sink.data_ptr(), st)
        b.record()
        torch.cuda.synchronize()
        best = max(best, nb * reps / (a.elapsed_time(b) * 1e-3) / 1e9)
    return {"read_GBps": best, "bytes": nb, "how": "scripts/l2probe.cu: ld.global.cg.v4 over a "
            "48 MiB L2-resident buffer, 592 CTAs x 512 threads, 20 passes, best of 6"}


def run_apsp(args, rank, world, dev, steps, warmup, with_cpu=False):
    """C5: APSP over the largest WCC.  A step = dawn_apsp on this rank's shard + (N > 1) one
    NCCL all-gather of the records; time = max over ranks."""
    import torch
    import torch.distributed as tdist
    import paper_2208_04514_b200 as dawn

    g = graphgen.config_graph("C5")
    G = dawn.Graph(g.row_ptr, g.col, True)
    verts, e_wcc = dawn.largest_wcc(G)  # the device helper picks the source set
    k = len(verts)
    flush = torch.empty(int(2.2 * L2_BYTES) // 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        dawn.apsp(G, verts, rank, world, gather=False)
    torch.cuda.synchronize()
    dawn.ms_counters(G)  # reset
    tot, kern, gath = [], [], []
    rec = None
    with ClockSampler(dev.index if dev.index is not None else 0) as clk:
        for _ in range(steps):
            flush.zero_()
            torch.cuda.synchronize()
            if world > 1:
                tdist.barrier()
            a, c = _events()
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            local = dawn.apsp(G, verts, rank, world, gather=False)
            c.record(stream)
            rec = dawn.gather_records(local, k, world) if world > 1 else local
            b.record(stream)
            torch.cuda.synchronize()
            tot.append(a.elapsed_time(b))
            kern.append(a.elapsed_time(c))
            gath.append(c.elapsed_time(b))
    cnt = dawn.ms_counters(G)
    t_tot = sum(tot)
    per_rank = {"kernel_ms": float(np.mean(kern)), "gather_ms": float(np.mean(gath))}
    if world > 1:
        tt = torch.tensor([t_tot], dtype=torch.float64, device=dev)
        tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
        t_tot = float(tt.item())
        pr = torch.tensor([per_rank["kernel_ms"], per_rank["gather_ms"]], dtype=torch.float64,
                          device=dev)
        allpr = [torch.zeros_like(pr) for _ in range(world)]
        tdist.all_gather(allpr, pr)
        per_rank = {"kernel_ms": [float(x[0]) for x in allpr],
                    "gather_ms": [float(x[1]) for x in allpr]}
    value = k * steps / (t_tot * 1e-3)
    peak, peak_kind = peaks()
    mine = len(dawn.apsp_shard(k, rank, world))
    # executed bytes of k_ms64 ("for ms64, B_exec is the per-batch word traffic"):
    # every level sweeps three 32-byte words per vertex (the frontier / seen test word, the
    # next / seen word, the new frontier word written), every gathered adjacency entry moves a
    # 4-byte index and a 32-byte word, every reduction 8 bytes
    b_exec = 96 * g.n * cnt["levels"] + 36 * cnt["gathered"] + 8 * cnt["reductions"]
    kern_s = float(np.sum(kern)) * 1e-3
    ach = b_exec / kern_s / 1e9
    l2 = l2_peak(dev) if world == 1 else None
    per_src_sovm = 4 * e_wcc + 8 * k + 32
    res = {
        "value": value, "unit": "sources/s", "n_gpus": world, "steps": steps,
        "ms_per_step": t_tot / steps, "scaling": "strong",
        "workload": f"C5: {CONFIG_TEXT['C5']}", "n": g.n, "m": g.m, "S_wcc": k, "E_wcc": e_wcc,
        "batch": dawn.MS_BATCH, "per_rank": per_rank,
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                     "frac": ach / peak, "peak_kind": peak_kind,
                     "kernel": "k_ms64 (one persistent launch per multi-source lane per rank and step)",
                     "bytes_model": "B_exec = 96*n*levels + 36*gathered + 8*reductions "
                                    "(executed word traffic, kernel counters)",
                     "exec_bytes_per_step": b_exec / steps,
                     "counters_per_step": {x: v / steps for x, v in cnt.items()},
                     "l2_peak_GBps": l2["read_GBps"] if l2 else None,
                     "frac_l2": ach / l2["read_GBps"] if l2 else None,
                     "traffic": ncu_traffic("apsp-C5"),
                     "sovm_equivalent_GBps": per_src_sovm * mine * steps / kern_s / 1e9,
                     "sovm_note": "per-source B_SOVM = 4*E_wcc + 8*S_wcc + 32 bytes: what 173K "
                                  "independent SOVM searches would move; the bit-parallel kernel "
                                  "shares each adjacency pass among 256 sources, so this is "
                                  "work avoided, not bandwidth"},
        "l2_probe": l2,
        "check": {"all_reached_S_wcc_minus_1":
                  bool(np.all(dawn.records_to_numpy(rec)["reached"] == k - 1))},
        "clocks": clk.summary(),
        "gpu_launches_per_step": min(-(-k // dawn.MS_BATCH), int(G.get_tuning("ms_lanes"))),
    }
    # e2e: host source list in, records out to host (the API a user calls)
    host_rec = torch.empty((k if world > 1 else mine, 4), dtype=torch.int64, pin_memory=True)
    e_ms = []
    for _ in range(max(1, min(steps, 3))):
        flush.zero_()
        torch.cuda.synchronize()
        if world > 1:
            tdist.barrier()
        a, b = _events()
        a.record(stream)
        r = dawn.apsp(G, verts, rank, world, gather=world > 1)
        host_rec.copy_(r, non_blocking=True)
        b.record(stream)
        torch.cuda.synchronize()
        e_ms.append(a.elapsed_time(b))
    e_tot = sum(e_ms)
    if world > 1:
        tt = torch.tensor([e_tot], dtype=torch.float64, device=dev)
        tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
        e_tot = float(tt.item())
    res["e2e"] = {"value": k * len(e_ms) / (e_tot * 1e-3), "unit": "sources/s",
                  "h2d_bytes_per_step": int(8 * k), "d2h_bytes_per_step": int(host_rec.numel() * 8),
                  "how": "dawn_apsp from the host int64 source list (uploaded by the call), "
                         "records (32 B each; all-gathered at N > 1) copied to pinned host memory"}
    if with_cpu:
        cores = len(os.sched_getaffinity(0))
        rate, cnt_s, dt = cpu_oracle_apsp(g, verts, args.cpu_budget, cores)
        res["cpu_baseline"] = {"value": rate, "unit": "sources/s", "cores": cores,
                               "kind": "oracle",
                               "sample": f"oracle_records (literal Algorithm 2 + record per "
                                         f"source) over the first {cnt_s} largest-WCC sources "
                                         f"on {cores} threads, {dt:.1f} s"}
    return res


def run_part(args, rank, world, dev, cfg="C4", nsrc=8, steps=3, fused=True):
    """NEXT-3: single-source searches over the vertex-partitioned graph (each rank holds only the
    arcs into its vertex range; one frontier-slice all-gather per level, NCCL at N > 1).  A step =
    `nsrc` searches one after the other; time = max over ranks; strong scaling (the same search
    on more GPUs)."""
    import torch
    import torch.distributed as tdist
    import paper_2208_04514_b200 as dawn

    g = graphgen.config_graph(cfg)
    t0 = time.time()
    pg = dawn.PartGraph(dawn.part_build(g.row_ptr, g.col, world, rank), world, rank, device=dev)
    t_build = time.time() - t0
    srcs = sources_for(g, cfg, 0, nsrc)  # the same sources on every rank
    out = torch.empty(max(1, pg.R), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    flush = torch.empty(int(2.2 * L2_BYTES) // 4, dtype=torch.int32, device=dev)
    er = []
    for s in srcs:  # E10 counts (global, identical on every rank) + warm-up
        _, st = dawn.part_sssp(pg, int(s), args.variant, out=out, stats=True)
        er.append(dawn.stats_to_dict(st)["edges_reach"])
        if fused:
            dawn.part_sssp_fused(pg, int(s), args.variant, out=out)

    def run(fused):
        ms = []
        for _ in range(steps):
            flush.zero_()
            torch.cuda.synchronize()
            if world > 1:
                tdist.barrier()
            a, b = _events()
            a.record(stream)
            for s in srcs:
                if fused:
                    dawn.part_sssp_fused(pg, int(s), args.variant, out=out)
                else:
                    dawn.part_sssp(pg, int(s), args.variant, out=out)
            b.record(stream)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        tot = sum(ms)
        if world > 1:
            t = torch.tensor([tot], dtype=torch.float64, device=dev)
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
            tot = float(t.item())
        return tot

    tot_nccl = run(False)
    tot = run(True) if fused else tot_nccl
    part_bytes = (pg.workspace.numel() + 8 * (pg.out_rp.numel() + pg.in_rp.numel()) +
                  4 * (pg.out_col.numel() + pg.in_col.numel() + pg.deg.numel()))
    res = {"value": float(sum(er)) * steps / (tot * 1e-3) / 1e9, "unit": "GTEPS",
           "workload": f"{cfg} graph ({CONFIG_TEXT[cfg].split(', 64')[0]}), {len(srcs)} sources, "
                       f"vertex-partitioned over {world} rank(s)",
           "ms_per_search": tot / (steps * len(srcs)), "ranks": world, "scaling": "strong",
           "device_bytes_per_rank": int(part_bytes), "partition_build_s": t_build,
           "how": ("dawn_part_fused_sssp: one persistent kernel per rank and search, frontier "
                   "slices stored into every rank's receive buffer (CUDA IPC mappings over NVLink "
                   "at N > 1) with system-scope arrival counters; L2 flushed between steps")
                  if fused else "the NCCL-per-level path below (fused exchange not run: "
                                "--fused-part)",
           "nccl_per_level": {"value": float(sum(er)) * steps / (tot_nccl * 1e-3) / 1e9,
                              "unit": "GTEPS", "ms_per_search": tot_nccl / (steps * len(srcs)),
                              "how": "dawn_part_begin / (NCCL all-gather + dawn_part_step) per "
                                     "level / dawn_part_finish, convergence tested every 4 levels"}}
    del pg, out, flush
    torch.cuda.empty_cache()
    return res


def run_weighted(args, dev, cfg="C4", nsrc=8, steps=3):
    """NEXT-4: weighted SSSP by (min,+) DAWN rounds (dawn_wsssp) on the config's graph with seeded
    integer arc weights in [1, 255] (one per undirected edge).  GTEPS over E10 counts of the
    reached set (the Graph500 SSSP convention counts the component's edges likewise)."""
    import torch
    import paper_2208_04514_b200 as dawn

    g = graphgen.config_graph(cfg)
    G = dawn.Graph(g.row_ptr, g.col, True)
    wt = torch.from_numpy(g.weights(seed=int(cfg[1:]), wmax=255).view(np.int32)).to(dev)
    srcs = sources_for(g, cfg, 0, nsrc)
    dsrc = torch.from_numpy(srcs.astype(np.int32)).to(dev)
    out = torch.empty((len(srcs), g.n), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    flush = torch.empty(int(2.2 * L2_BYTES) // 4, dtype=torch.int32, device=dev)
    er, rounds, relaxed = [], [], []
    _, sts = dawn.wsssp_batch(G, dsrc, wt, stats=True, out=out, check=True)
    for i in range(len(srcs)):
        x = dawn.stats_to_dict(sts[i])
        er.append(x["edges_reach"]); rounds.append(x["levels"]); relaxed.append(x["edges_examined"])
    ms = timed(lambda: dawn.wsssp_batch(G, dsrc, wt, out=out), steps, flush, stream)
    t = float(np.median(ms))
    peak, _ = peaks()
    # executed bytes: per relaxed arc a 4-B target, a 4-B weight and a 4-B distance read
    b_exec = 12 * float(np.sum(relaxed)) + 4 * g.n * len(srcs)
    res = {"value": float(np.sum(er)) / (t * 1e-3) / 1e9, "unit": "GTEPS",
           "workload": f"{cfg} graph ({CONFIG_TEXT[cfg].split(', 64')[0]}), {len(srcs)} sources, "
                       "uint32 weights in [1, 255]",
           "ms_per_search": t / len(srcs), "rounds_mean": float(np.mean(rounds)),
           "arcs_relaxed_per_search": float(np.mean(relaxed)),
           "roofline": {"bound": "hbm", "achieved": b_exec / (t * 1e-3) / 1e9, "peak": peak,
                        "unit": "GB/s", "frac": b_exec / (t * 1e-3) / 1e9 / peak,
                        "bytes_model": "12 B per relaxed arc (target, weight, distance) + 4n"},
           "how": "one dawn_wsssp_batch call over the sources (one persistent k_wsssp launch, "
                  "searches back to back), L2 flushed between steps"}
    del G, wt, out, flush
    torch.cuda.empty_cache()
    return res


def run_dawn(args):
    import torch
    rank, world, local = dist_setup(args.gpus)
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=dev)
    import paper_2208_04514_b200 as dawn
    dawn.lib()  # loads libdawn.so (raises if missing: there is no fallback)
    workload = args.workload
    if workload == "auto":
        workload = "sssp" if world == 1 else "apsp"
    common = {"metric": METRIC, "n_gpus": world, "warmup": args.warmup, "higher_is_better": True,
              "vs_baseline": None, "data": "synthetic (seeded generators, graphgen/)"}
    if workload == "apsp":
        r = run_apsp(args, rank, world, dev, args.steps, args.warmup,
                     with_cpu=(rank == 0 and world == 1 and not args.no_cpu))
        res = {**common, "value": r.pop("value"), "unit": r.pop("unit"),
               "steps": args.steps, "ms_per_step": r.pop("ms_per_step"), "scaling": "strong",
               "dtype": "u64 (256-source bit words; uint32 ids/distances)",
               "config": {"workload": r.pop("workload"), "n": r.pop("n"), "m": r.pop("m"),
                          "S_wcc": r.pop("S_wcc"), "E_wcc": r.pop("E_wcc"),
                          "parallelism": f"sources sharded over {world} rank(s), 256-source "
                                         "batches round-robin, one NCCL all-gather",
                          "l2": "flushed between timed steps (2.2x L2 write)"},
               "gpu_launches": args.steps * r.pop("gpu_launches_per_step")}
        res.update(r)
    else:
        cfg = args.config
        r = run_sssp(args, rank, world, dev, cfg, args.steps, args.warmup, e2e=True,
                     with_cpu=(rank == 0 and world == 1 and not args.no_cpu))
        res = {**common, "value": r.pop("value"), "unit": r.pop("unit"), "steps": args.steps,
               "ms_per_step": r.pop("ms_per_step"), "scaling": "weak",
               "dtype": "u32 (vertex ids, offsets, distances; 32-bit bitmap words)",
               "config": {"workload": r.pop("workload"), "n": r.pop("n"), "m": r.pop("m"),
                          "sources_per_rank": r.pop("sources_per_step"), "variant": args.variant,
                          "parallelism": f"dp{world}: independent sources per rank (replicas)",
                          "l2": "flushed between timed steps (2.2x L2 write)"},
               "gpu_launches": args.steps * r.pop("gpu_launches_per_step")}
        res.update(r)
        if world == 1 and args.extra:
            ex = {}
            for c in ("C1", "C2", "C3"):
                if c == cfg:
                    continue
                ex[c] = run_sssp(args, rank, world, dev, c, max(3, min(args.steps, 10)), 3,
                                 e2e=False)
            ex["C5"] = run_apsp(args, rank, world, dev, max(2, min(args.steps, 5)), 2,
                                with_cpu=not args.no_cpu)
            ex["C4_weighted"] = run_weighted(args, dev)
            res["configs"] = ex
    if args.extra and world >= 1:
        # NEXT-3: the same C4 searches over the vertex-partitioned graph (W = N ranks).  The fused
        # exchange (peer stores over NVLink) is validated on one GPU only, so at N > 1 it runs
        # only with --fused-part; a failure here never costs the headline line
        try:
            res["partitioned_sssp"] = run_part(args, rank, world, dev,
                                               fused=(world == 1 or args.fused_part))
        except Exception as ex:  # noqa: BLE001 - reported in the line instead
            res["partitioned_sssp"] = {"error": f"{type(ex).__name__}: {ex}"[:300]}
    if world > 1:
        import torch.distributed as tdist
        tdist.barrier()
        tdist.destroy_process_group()
    if rank == 0:
        print(json.dumps(res), flush=True)


def run_reference(args):
    """Reference arm for this tier: the CPU oracle, as it stands, on the host cores, on the same
    config / metric / unit as the dawn arm (C4 SSSP GTEPS at N = 1, C5 APSP sources/s at N > 1).
    Under torchrun rank 0 alone runs it; the other ranks exit without work."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    workload = args.workload if args.workload != "auto" else ("sssp" if world == 1 else "apsp")
    per_step = max(2.0, args.cpu_budget / max(1, args.steps + args.warmup))
    if workload == "apsp":
        g = graphgen.config_graph("C5")
        import oracle
        verts, _ = oracle.largest_wcc(g.n, g.row_ptr, g.col)
        for _ in range(args.warmup):
            cpu_oracle_apsp(g, verts, per_step, cores)
        rates, cnt = [], 0
        for _ in range(args.steps):
            rate, cnt, dt = cpu_oracle_apsp(g, verts, per_step, cores)
            rates.append(rate)
        value, unit = float(np.mean(rates)), "sources/s"
        sample = (f"oracle_records (literal Algorithm 2 per source) over the first {cnt} "
                  f"largest-WCC sources per step, {cores} threads")
        cfgtxt = f"C5: {CONFIG_TEXT['C5']}"
    else:
        cfg = args.config
        g = graphgen.config_graph(cfg)
        srcs = sources_for(g, cfg, 0)
        for _ in range(args.warmup):
            cpu_oracle_sssp(g, srcs, per_step, cores)
        e_tot = t_tot = 0.0
        done_tot = 0
        for i in range(args.steps):
            gte, done, t = cpu_oracle_sssp(g, np.roll(srcs, -i * cores), per_step, cores)
            e_tot += gte * t
            t_tot += t
            done_tot += done
        value, unit = e_tot / t_tot, "GTEPS"
        sample = (f"oracle_sovm (literal Algorithm 2), one source per host thread, {done_tot} "
                  f"source SSSPs over {args.steps} steps")
        cfgtxt = f"{cfg}: {CONFIG_TEXT[cfg]}"
    res = {"impl": "reference", "metric": METRIC, "value": value, "unit": unit,
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
           "dtype": "u32", "data": "synthetic (seeded generators, graphgen/)",
           "vs_baseline": None, "config": {"workload": cfgtxt},
           "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(res), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["dawn", "reference"], default="dawn")
    ap.add_argument("--workload", choices=["auto", "sssp", "apsp"], default="auto",
                    help="auto: SSSP C4 at N=1, APSP C5 at N>1")
    ap.add_argument("--config", choices=["C1", "C2", "C3", "C4"], default="C4")
    ap.add_argument("--variant", choices=["auto", "push", "pull"], default="auto")
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of oracle CPU work")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--fused-part", action="store_true",
                    help="at N > 1, also run the partitioned path with the fused NVLink exchange")
    ap.add_argument("--no-extra", dest="extra", action="store_false",
                    help="skip the other configs (C1/C2/C3/C5 under 'configs')")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "dawn":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_dawn(args)


if __name__ == "__main__":
    main()
