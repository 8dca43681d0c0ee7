#!/usr/bin/env python
"""bench.py — DAWN on B200: SSSP GTEPS (1 GPU) and APSP sources/s (1/2/4/8 GPUs) vs the HBM
roofline (BASELINE.json metric).

  python bench.py [--gpus N --steps K --warmup W] [--workload sssp|apsp] [--config C2]
                  [--variant auto|push|pull] [--impl dawn|reference]

Default (N=1): workload "sssp" on configs[1] = C2, Graph500 Kronecker scale 20 ef 16, 64
seeded sources per rank; one step = 64 dawn_sssp calls (one persistent kernel each) writing
64 distance rows.  Under torchrun each rank runs its own 64 sources (weak scaling); time is the
max over ranks.  The JSON line also carries the C5 APSP (largest WCC of Kronecker-18, sources
sharded over the N ranks, one NCCL all-gather) as "secondary".

--impl reference times the CPU oracle (oracle/, literal Algorithm 2) on the host cores on a
bounded sample of the same workload (this tier's reference arm: there is no reference code).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import graphgen  # noqa: E402

CONFIG_TEXT = {
    "C1": "SSSP from vertex 0, directed Erdos-Renyi n=1000 m=8000 (seed 1)",
    "C2": "SSSP, Graph500 Kronecker scale 20 edge factor 16 (seed 20), 64 sources",
    "C3": "SSSP from vertex 0 on a 4096x4096 grid",
    "C4": "SSSP, Graph500 Kronecker scale 24 edge factor 16 (seed 24), 64 sources",
    "C5": "APSP over all sources of the largest WCC of Kronecker scale 18 ef 16 (seed 18)",
}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


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


def build_graph(cfg: str):
    g = graphgen.config_graph(cfg)
    return g


def sources_for(g, cfg: str, rank: int, count: int = 64):
    if cfg in ("C1", "C3"):
        return np.zeros(1, np.int64)  # vertex 0 (configs[0], configs[2])
    return g.sample_sources(count, seed=1 + 1000 * rank).astype(np.int64)


# ------------------------------------------------------------------------------- CPU oracle
def cpu_oracle_sssp(g, sources, budget_s: float):
    """Literal Algorithm 2 oracle, single-threaded, sources in order until the budget."""
    import oracle
    t_tot, e_tot, done = 0.0, 0, 0
    for s in sources:
        t0 = time.perf_counter()
        _, st = oracle.sovm(g.n, g.row_ptr, g.col, int(s))
        t_tot += time.perf_counter() - t0
        e_tot += st["edge_inspections"]
        done += 1
        if t_tot >= budget_s:
            break
    return e_tot / t_tot / 1e9, done, t_tot


def cpu_oracle_apsp(g, verts, budget_s: float):
    import oracle
    cores = len(os.sched_getaffinity(0))
    k = max(cores, 16)
    rate = None
    spent = 0.0
    while True:
        sub = verts[:k]
        t0 = time.perf_counter()
        oracle.records(g.n, g.row_ptr, g.col, sub, threads=cores)
        dt = time.perf_counter() - t0
        spent += dt
        rate = len(sub) / dt
        if dt > budget_s / 3 or k >= len(verts) or spent > budget_s:
            return rate, len(sub), cores, dt
        k = min(len(verts), int(k * max(2.0, budget_s / 3 / max(dt, 1e-3))))


# ------------------------------------------------------------------------------- GPU arms
# the kernel that does the work of one dawn_sssp call on each config (the dominant kernel)
KERNEL_OF = {"C1": "k_small (one SSSP per CTA, CSR in shared memory; the batch's searches run "
                   "on min(k, #SMs) CTAs at once)",
             "C2": "k_sssp (one persistent launch running the batch's SSSPs back to back)",
             "C3": "k_narrow (one 16-CTA cluster per SSSP; the k_sssp behind it exits at once)",
             "C4": "k_sssp (one persistent launch running the batch's SSSPs back to back)"}


def run_sssp(args, rank, world, dev, cfg=None, steps=None, warmup=None, e2e=True, reps=1):
    """One SSSP config.  A step = every bench source once (64 for C2/C4; the single source
    repeated `reps` times for C1/C3)."""
    import torch
    import torch.distributed as tdist
    import paper_2208_04514_b200 as dawn

    cfg = cfg or args.config
    steps = args.steps if steps is None else steps
    warmup = args.warmup if warmup is None else warmup
    g = build_graph(cfg)
    G = dawn.Graph(g.row_ptr, g.col, g.symmetric,
                   *(g.transpose() if not g.symmetric else (None, None)))
    srcs = sources_for(g, cfg, rank)
    if reps > 1:
        srcs = np.repeat(srcs, reps)
    k = len(srcs)
    out = torch.empty((min(k, 64), g.n), dtype=torch.int32, device=dev)
    orow = lambda i: out[i % out.shape[0]]
    # E_reach per source (the E10 numerator) from the kernel's own statistics, untimed
    er, reached, examined, pushl, pulll = [], [], [], [], []
    for i, s in enumerate(srcs):
        _, st = dawn.sssp(G, int(s), args.variant, stats=True, out=orow(i))
        d = dawn.stats_to_dict(st)
        er.append(d["edges_reach"]); reached.append(d["reached"]); examined.append(d["edges_examined"])
        pushl.append(d["push_levels"]); pulll.append(d["pull_levels"])
    flush = torch.empty(int(2.2 * 132644864) // 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()

    dsrc = torch.from_numpy(srcs.astype(np.int32)).to(dev)
    outk = out[:k]

    def step():
        # the public batch call: the k searches one after the other (dawn_sssp_batch: one
        # k_sssp launch, or k_small / per-search k_narrow + k_sssp where those apply)
        dawn.sssp_batch(G, dsrc, args.variant, out=outk)

    step()
    torch.cuda.synchronize()
    for _ in range(warmup):
        step()
        flush.zero_()
    torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    step_ms = []
    with ClockSampler(dev.index if dev.index is not None else 0) as clk:
        for _ in range(steps):
            flush.zero_()  # L2 flush between timed steps (write 2.2x L2)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step()
            b.record(stream)
            torch.cuda.synchronize()
            step_ms.append(a.elapsed_time(b))
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    tot_ms = sum(step_ms)
    # average duration of one search over the timed region: timed steps / searches they contain
    launch_ms = [sum(step_ms) / (len(step_ms) * k)]
    if world > 1:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        tot_ms = float(t.item())
    edges_step = float(sum(er))
    value = edges_step * steps * world / (tot_ms * 1e-3) / 1e9

    # roofline: dominant (only) kernel k_sssp; algorithmic bytes B_SOVM(s) = 4E + 8S + 4n
    peak, peak_kind = peaks()
    b_sovm = [4 * e + 8 * (r + 1) + 4 * g.n for e, r in zip(er, reached)]
    b_exec = [4 * g.n + 4 * x + 8 * (r + 1) + (g.n // 8) * (2 * pl + 1)
              for x, r, pl in zip(examined, reached, pulll)]
    avg_launch_ms = float(np.mean(launch_ms))
    achieved = float(np.mean(b_sovm)) / (avg_launch_ms * 1e-3) / 1e9
    achieved_exec = float(np.mean(b_exec)) / (avg_launch_ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(f"sssp-{cfg}-{args.variant}")

    # context, not the headline: (1) the latency of ONE dawn_sssp call (L2 flushed before each),
    # (2) the same distinct sources through the bit-parallel multi-source kernel (dawn_msssp)
    lat = []
    for i in range(min(k, 16)):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        dawn.sssp(G, int(srcs[i]), args.variant, out=outk[i])
        b.record(stream)
        torch.cuda.synchronize()
        lat.append(a.elapsed_time(b))
    single = {"median_us": float(np.median(lat)) * 1e3, "calls": len(lat),
              "gteps": float(np.mean(er[:len(lat)])) / (float(np.median(lat)) * 1e-3) / 1e9}
    uniq = len(set(int(x) for x in srcs))
    if uniq == k and k >= 64 and args.variant == "auto":
        ms_dist = torch.empty((k, g.n), dtype=torch.int32, device=dev)
        dawn.msssp(G, srcs, dist=True, records=False, d_out=ms_dist)
        torch.cuda.synchronize()
        assert torch.equal(ms_dist, outk), "dawn_msssp distances differ from dawn_sssp_batch"
        mt = []
        for _ in range(3):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            dawn.msssp(G, srcs, dist=True, records=False, d_out=ms_dist)
            b.record(stream)
            torch.cuda.synchronize()
            mt.append(a.elapsed_time(b))
        single["msssp_same_sources"] = {
            "gteps": edges_step / (float(np.median(mt)) * 1e-3) / 1e9,
            "ms": float(np.median(mt)),
            "how": "dawn_msssp on the same k sources (one bit-parallel pass, dist rows written), "
                   "distances checked equal to the batch's"}
        del ms_dist

    # the forced-push (pure SOVM, Algorithm 2) schedule on the same sources
    forced_push = None
    if args.variant == "auto" and cfg in ("C2", "C4"):
        dawn.sssp_batch(G, dsrc, "push", out=outk)
        pt = []
        for _ in range(2):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            dawn.sssp_batch(G, dsrc, "push", out=outk)
            b.record(stream)
            torch.cuda.synchronize()
            pt.append(a.elapsed_time(b))
        pms = float(np.median(pt))
        forced_push = {"gteps": edges_step / (pms * 1e-3) / 1e9, "ms_per_step": pms,
                       "achieved_GBps_B_SOVM": float(np.sum(b_sovm)) / (pms * 1e-3) / 1e9,
                       "how": "dawn_sssp_batch with DAWN_PUSH (every level SOVM) on the same sources"}

    if not e2e:
        peak, _ = peaks()
        return {"value": value, "unit": "GTEPS", "ms_per_step": tot_ms / steps, "steps": steps,
                "sources_per_step": k, "n": g.n, "m": g.m, "workload": f"{cfg}: {CONFIG_TEXT[cfg]}",
                "avg_launch_us": avg_launch_ms * 1e3, "edges_reach_mean": float(np.mean(er)),
                "levels": {"push_mean": float(np.mean(pushl)), "pull_mean": float(np.mean(pulll))},
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "kernel": KERNEL_OF.get(cfg),
                             "traffic": traffic, "achieved_exec": achieved_exec,
                             "frac_exec": achieved_exec / peak,
                             "bytes_model": "B_SOVM = 4*E_reach + 8*S_reach + 4*n"},
                "single_search": single, "forced_push": forced_push,
                "clocks": clk.summary()}, g, srcs, er
    # e2e through the public API with HOST buffers: the source list H2D (pinned), then
    # dawn_sssp_batch over chunks of E2E_CHUNK sources, each chunk's distance rows copied to pinned
    # host memory on a second stream while the next chunk computes (the D2H of 64 rows, 4n bytes
    # each, is the bound: ~45-55 GB/s of PCIe against ~50 GB/s of distance rows produced)
    E2E_CHUNK = int(os.environ.get("DAWN_E2E_CHUNK", "1"))  # 1/4/8/16: 348/338/328/291 GTEPS
    host_src = torch.from_numpy(srcs.astype(np.int32)).pin_memory()
    dev_src = torch.empty_like(host_src, device=dev)
    host_out = torch.empty((k, g.n), dtype=torch.int32).pin_memory()
    e2e_ms = []
    copy_stream = torch.cuda.Stream(device=dev)
    for it in range(max(1, steps)):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        dev_src.copy_(host_src, non_blocking=True)
        for c0 in range(0, k, E2E_CHUNK):
            c1 = min(k, c0 + E2E_CHUNK)
            dawn.sssp_batch(G, dev_src[c0:c1], args.variant, out=outk[c0:c1])
            done = torch.cuda.Event()
            done.record(stream)
            copy_stream.wait_event(done)
            with torch.cuda.stream(copy_stream):
                host_out[c0:c1].copy_(outk[c0:c1], non_blocking=True)
        stream.wait_stream(copy_stream)
        b.record(stream)
        torch.cuda.synchronize()
        e2e_ms.append(a.elapsed_time(b))
    e2e_tot = sum(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e_tot], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        e2e_tot = float(t.item())
    e2e_val = edges_step * len(e2e_ms) * world / (e2e_tot * 1e-3) / 1e9

    res = {
        "metric": "SSSP GTEPS (1 B200) and APSP sources/sec at 1/2/4/8 B200 vs HBM roofline",
        "value": value, "unit": "GTEPS", "n_gpus": world, "steps": steps,
        "warmup": warmup, "ms_per_step": tot_ms / steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": f"{cfg}: {CONFIG_TEXT[cfg]}", "n": g.n, "m": g.m,
                   "sources_per_rank": k, "variant": args.variant,
                   "l2": "flushed between timed steps (2.2x L2 write)",
                   "teps_numerator": "E_reach = sum of out-degrees of reached vertices incl. s "
                                     "(directed arcs, PAPER E10)",
                   "parallelism": f"dp{world} (independent sources per rank)"},
        # dawn_sssp_batch: k_narrow + k_sssp per search on cluster-start graphs (C3), else one
        # launch per step
        "gpu_launches": steps * (2 * k if cfg == "C3" else 1),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": KERNEL_OF.get(cfg, KERNEL_OF["C2"]),
                     "algorithmic_bytes_per_launch": float(np.mean(b_sovm)),
                     "bytes_model": "B_SOVM = 4*E_reach + 8*S_reach + 4*n",
                     "avg_launch_us": avg_launch_ms * 1e3,
                     "achieved_exec": achieved_exec, "frac_exec": achieved_exec / peak,
                     "exec_bytes_per_launch": float(np.mean(b_exec))},
        "e2e": {"value": e2e_val, "unit": "GTEPS", "h2d_bytes_per_step": int(host_src.numel() * 4),
                "d2h_bytes_per_step": int(host_out.numel() * 4),
                "how": f"source list H2D, then dawn_sssp_batch over chunks of {E2E_CHUNK} "
                       "source(s); each chunk's distance rows copied to pinned host memory on a "
                       "second stream while the next chunk computes",
                "ms_per_step": e2e_tot / len(e2e_ms)},
        "levels": {"push_mean": float(np.mean(pushl)), "pull_mean": float(np.mean(pulll)),
                   "edges_examined_mean": float(np.mean(examined)),
                   "edges_reach_mean": float(np.mean(er))},
        "single_search": single,
        "forced_push": forced_push,
        "clocks": clk.summary(),
    }
    return res, g, srcs, er


def l2_probe(dev):
    """L2 bandwidth measured in the same run (context for the L2-resident
    C5 words and C2's bitmaps): a device copy between two 24 MiB buffers (48 MiB, inside the
    126 MB L2), 40 back-to-back copies timed with CUDA events after a warm-up."""
    import torch
    nb = 24 << 20
    a = torch.ones(nb // 4, dtype=torch.int32, device=dev)
    b = torch.empty_like(a)
    for _ in range(5):
        b.copy_(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(40):
        b.copy_(a)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 40
    return {"copy_GBps": 2 * nb / (ms * 1e-3) / 1e9, "bytes_per_copy": 2 * nb,
            "how": "torch copy_ of a 24 MiB int32 buffer (read + write counted), L2-resident; a "
                   "lower bound on L2 bandwidth (the copy kernel's own limit may bind first)"}


def run_apsp(args, rank, world, dev, steps=None, warmup=None):
    import torch
    import torch.distributed as tdist
    import paper_2208_04514_b200 as dawn

    steps = args.steps if steps is None else steps
    warmup = args.warmup if warmup is None else warmup
    g = build_graph("C5")
    G = dawn.Graph(g.row_ptr, g.col, True)
    verts, e_wcc = g.largest_wcc()
    k = len(verts)
    flush = torch.empty(int(2.2 * 132644864) // 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        dawn.apsp(G, verts, rank, world, gather=False)
    torch.cuda.synchronize()
    ms, kern_ms = [], []
    with ClockSampler(dev.index if dev.index is not None else 0) as clk:
        for _ in range(steps):
            flush.zero_()
            torch.cuda.synchronize()
            if world > 1:
                tdist.barrier()
            a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            a.record(stream)
            local = dawn.apsp(G, verts, rank, world, gather=False)
            c.record(stream)
            rec = dawn.gather_records(local, k, world) if world > 1 else local
            b.record(stream)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
            kern_ms.append(a.elapsed_time(c))
    t = sum(ms)
    if world > 1:
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
        t = float(tt.item())
    value = k * steps / (t * 1e-3)
    peak, peak_kind = peaks()
    per_src = 4 * e_wcc + 8 * k + 32  # B_SOVM per source of the component
    mine = len(dawn.apsp_shard(k, rank, world))
    achieved = per_src * mine / (np.mean(kern_ms) * 1e-3) / 1e9
    recs = dawn.records_to_numpy(rec)
    return {"value": value, "unit": "sources/s", "n_gpus": world, "steps": steps,
            "ms_per_step": t / steps, "scaling": "strong",
            "config": {"workload": f"C5: {CONFIG_TEXT['C5']}", "n": g.n, "m": g.m,
                       "S_wcc": k, "E_wcc": e_wcc, "batch": dawn.MS_BATCH,
                       "l2": "flushed between timed steps"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_kind": peak_kind,
                         "kernel": "k_ms64 (one persistent launch per rank)",
                         "bytes_model": "per source B_SOVM = 4*E_wcc + 8*S_wcc + 32",
                         "traffic": json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get("apsp-C5") if os.path.exists(os.path.join(ROOT, "profiles", "ncu_traffic.json")) else None},
            "check": {"all_reached_S_wcc_minus_1": bool(np.all(recs["reached"] == k - 1))},
            "clocks": clk.summary()}, g, verts


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
    dawn.lib()
    if args.workload == "apsp":
        res, g, verts = run_apsp(args, rank, world, dev)
        res.update({"metric": "SSSP GTEPS (1 B200) and APSP sources/sec at 1/2/4/8 B200 vs HBM roofline",
                    "warmup": args.warmup, "higher_is_better": True, "vs_baseline": None,
                    "dtype": "u64", "data": "synthetic", "gpu_launches": args.steps})
        if rank == 0 and world == 1 and not args.no_cpu:
            rate, cnt, cores, dt = cpu_oracle_apsp(g, verts, args.cpu_budget)
            res["cpu_baseline"] = {"value": rate, "unit": "sources/s", "cores": cores,
                                   "kind": "oracle",
                                   "sample": f"oracle_records (literal Algorithm 2 per source) "
                                             f"over the first {cnt} largest-WCC sources, {dt:.1f} s"}
    else:
        res, g, srcs, er = run_sssp(args, rank, world, dev)
        if args.extra and world == 1:
            ex = {}
            for cfg, reps, st in (("C1", 64, max(3, args.steps)), ("C3", 1, 2), ("C4", 1, 2)):
                if cfg == args.config:
                    continue
                r, _, _, _ = run_sssp(args, rank, world, dev, cfg=cfg, steps=st, warmup=3,
                                      e2e=False, reps=reps)
                ex[cfg] = r
            res["extra_configs"] = ex
        if args.secondary:
            sec, _, _ = run_apsp(args, rank, world, dev, steps=max(1, min(args.steps, 3)),
                                 warmup=1)
            res["secondary"] = sec
        if world == 1:
            res["l2_probe"] = l2_probe(dev)
        if rank == 0 and world == 1 and not args.no_cpu:
            gte, done, t = cpu_oracle_sssp(g, srcs, args.cpu_budget)
            res["cpu_baseline"] = {"value": gte, "unit": "GTEPS", "cores": 1, "kind": "oracle",
                                   "sample": f"oracle_sovm (literal Algorithm 2, 1 thread) on the "
                                             f"first {done} of the {len(srcs)} bench sources, "
                                             f"{t:.1f} s"}
    if world > 1:
        import torch.distributed as tdist
        tdist.barrier()
        tdist.destroy_process_group()
    if rank == 0:
        print(json.dumps(res), flush=True)


def run_reference(args):
    """Reference arm for this tier: the CPU oracle, as it stands, on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    if args.workload == "apsp":
        g = build_graph("C5")
        verts, _ = g.largest_wcc()
        rates = []
        for _ in range(args.warmup):
            cpu_oracle_apsp(g, verts, min(args.cpu_budget, 4.0))
        for _ in range(args.steps):
            rate, cnt, cores, dt = cpu_oracle_apsp(g, verts, args.cpu_budget / max(1, args.steps))
            rates.append(rate)
        value, unit = float(np.mean(rates)), "sources/s"
        sample = f"oracle_records over the first {cnt} largest-WCC sources per step"
        cfgtxt = f"C5: {CONFIG_TEXT['C5']}"
        used = cores
    else:
        cfg = args.config
        g = build_graph(cfg)
        srcs = sources_for(g, cfg, 0)
        budget = max(1.0, args.cpu_budget / max(1, args.steps + args.warmup))
        for _ in range(args.warmup):
            cpu_oracle_sssp(g, srcs, budget)
        e_tot = t_tot = 0.0
        done_tot = 0
        for i in range(args.steps):
            gte, done, t = cpu_oracle_sssp(g, np.roll(srcs, -i), budget)
            e_tot += gte * t
            t_tot += t
            done_tot += done
        value, unit = e_tot / t_tot, "GTEPS"
        sample = f"oracle_sovm (literal Algorithm 2, 1 thread), {done_tot} source SSSPs over {args.steps} steps"
        cfgtxt = f"{cfg}: {CONFIG_TEXT[cfg]}"
        used = 1
    res = {"impl": "reference",
           "metric": "SSSP GTEPS (1 B200) and APSP sources/sec at 1/2/4/8 B200 vs HBM roofline",
           "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "higher_is_better": True, "dtype": "u32", "data": "synthetic",
           "vs_baseline": None, "config": {"workload": cfgtxt},
           "cpu_baseline": {"value": value, "unit": unit, "cores": used, "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(res), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["dawn", "reference"], default="dawn")
    ap.add_argument("--workload", choices=["sssp", "apsp"], default="sssp")
    ap.add_argument("--config", choices=["C1", "C2", "C3", "C4"], default="C2")
    ap.add_argument("--variant", choices=["auto", "push", "pull"], default="auto")
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of oracle CPU work")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", dest="secondary", action="store_false")
    ap.add_argument("--no-extra", dest="extra", action="store_false",
                    help="skip the C1/C3/C4 lines (reported under extra_configs)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "dawn":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_dawn(args)


if __name__ == "__main__":
    main()
