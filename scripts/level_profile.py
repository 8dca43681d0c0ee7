# Per-level profile of dawn_sssp (device trace): level timings + per-warp phase cycles.
import os, sys, time, numpy as np, torch
sys.path.insert(0, '.')
import graphgen, paper_2208_04514_b200 as dawn
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
variants = (sys.argv[2] if len(sys.argv) > 2 else "auto").split(",")
nsrc = int(os.environ.get("NSRC", "16"))
t = time.time(); g = graphgen.config_graph(cfg); print(cfg, "n", g.n, "m", g.m, "gen %.1fs" % (time.time() - t))
G = dawn.Graph(g.row_ptr, g.col, g.symmetric, *(g.transpose() if not g.symmetric else (None, None)), trace=os.environ.get('TRACE', '1') == '1')
if os.environ.get('ALPHA'): G.set_tuning(alpha=float(os.environ['ALPHA']))
srcs = [0] if cfg in ("C1", "C3") else list(g.sample_sources(nsrc, 1))
CLK = 1.965e3  # cycles per us at max clock
nw = 296 * 16
for v in variants:
    for s in srcs[:2]: dawn.sssp(G, int(s), v, stats=True)
    torch.cuda.synchronize()
    ts, er, traces = [], 0, []
    for s in srcs:
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); d, st = dawn.sssp(G, int(s), v, stats=True); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1)); sd = dawn.stats_to_dict(st); er += sd["edges_reach"]
        trr = G.trace() if os.environ.get('TRACE', '1') == '1' else None
        if trr is not None and os.environ.get("PROF"):
            G.trace_raw = trr
            trr = trr[: sd["levels"] + 1]
        traces.append((ts[-1], int(s), sd, trr, getattr(G, 'timeline', None)))
    print(f"== {cfg} {v}: median {np.median(ts)*1e3:.1f} us mean {np.mean(ts)*1e3:.1f} max {np.max(ts)*1e3:.1f}  GTEPS(agg) {er/(sum(ts)*1e-3)/1e9:.1f}")
    print("   per-source us:", [round(x * 1e3) for x in ts])
    for label, (tt, s, sd, tr, tl) in (("median", sorted(traces, key=lambda x: x[0])[len(traces)//2]), ("slowest", max(traces, key=lambda x: x[0]))):
        print(f"   {label} source {s}: {tt*1e3:.1f} us, {sd}")
        if tr is None: continue
        t0 = int(tr["t_ns"][0])
        if tl is not None and int(tl["t_ns"]) > 0:
            print("   k_sssp timeline us (rel. level 0 start): entry %.1f init-done %.1f last-level-done %.1f" % (
                (int(tl["t_ns"]) - t0) / 1e3, (int(tl["t_first"]) - t0) / 1e3, (int(tl["t_last"]) - t0) / 1e3))
        if len(tr) > 40:
            print("   levels:", len(tr), " avg level us: %.2f" % ((int(tr['t_ns'][-1]) - t0) / 1e3 / (len(tr) - 1)))
            rows = list(tr[:6]) + list(tr[len(tr)//2 - 2: len(tr)//2 + 2]) + list(tr[-4:])
        else:
            rows = tr
        for r in rows:
            f = lambda x: round((int(x) - t0) / 1e3, 1) if 0 < int(x) < 2**63 else None
            if r["rep"] & 8:  # k_narrow level: CTA-0 work / cluster-barrier wait / max-CTA work, us
                print("   L%d NARROW nf=%d mf=%d start=%s  [work0 sync0 maxwork] us = [%s]" % (
                    r["level"], r["nf"], r["mf"], f(r["t_ns"]), " ".join("%.2f" % (c / CLK) for c in r["cyc"][:3])))
                if os.environ.get("PROF"):
                    r2 = G.trace_raw[r["level"] + 32768]
                    raw = np.array([r2["t_first"], r2["t_last"], r2["cyc"][0], r2["cyc"][1], r2["cyc"][2], r2["cyc"][3]], dtype=np.uint64).view(np.uint32)
                    print("      stamps (cyc from start) entry/arc/claim/append/sums/sync/exch/barrier/next:", list(raw[:9]), "rank", raw[9])
                continue
            solo = bool(r["rep"] & 2)
            div = 1 if os.environ.get("TRACE_MAX") else (16 if solo else nw)
            cyc = " ".join("%.1f" % (c / div / CLK) for c in r["cyc"])
            print("   L%d %s%s nf=%d mf=%d start=%s first=%s last=%s  per-warp us [work heavy flush conv]=[%s]" % (
                r["level"], "PUSH PULL STOP".split()[r["dir"]], " solo" if solo else "", r["nf"], r["mf"],
                f(r["t_ns"]), f(r["t_first"]), f(r["t_last"]), cyc))
