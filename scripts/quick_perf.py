# quick timing probe (not the bench): SSSP on kron-N per variant (+ per-level trace), APSP rate on kron-18.
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import graphgen, paper_2208_04514_b200 as dawn
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
g = graphgen.kron(scale); G = dawn.Graph(g.row_ptr, g.col, True, trace=True)
srcs = g.sample_sources(16, 1)
import os
alphas = [float(x) for x in os.environ.get("ALPHAS", "14").split(",")]
for v in ["auto"] * len(alphas) + ["push", "pull"]:
    if v == "auto":
        a_ = alphas.pop(0); G.set_tuning(alpha=a_); print("alpha", a_)
    for s in srcs[:3]: dawn.sssp(G, int(s), v)
    torch.cuda.synchronize()
    ts = []; er = 0
    for s in srcs:
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); d, st = dawn.sssp(G, int(s), v, stats=True); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1)); er += dawn.stats_to_dict(st)["edges_reach"]
    print(v, "ms/sssp median %.4f mean %.4f max %.4f" % (np.median(ts), np.mean(ts), np.max(ts)), "GTEPS %.1f" % (er / (sum(ts) * 1e-3) / 1e9), dawn.stats_to_dict(st))
    tr = G.trace(); t0 = tr["t_ns"][0]
    for r in tr:
        f = lambda x: round((int(x) - int(t0)) / 1e3, 1) if 0 < int(x) < 2**63 else None
        print("   L%d %s%s nf=%d mf=%d start=%s first_done=%s last_done=%s" % (r["level"], "PUSH PULL STOP".split()[r["dir"]], " solo" if (r["rep"] & 2) else "", r["nf"], r["mf"], f(r["t_ns"]), f(r["t_first"]), f(r["t_last"])))
g = graphgen.kron(18); G = dawn.Graph(g.row_ptr, g.col, True)
verts, e = g.largest_wcc()
for a in (2,):
    G.set_tuning(ms_alpha=a)
    for nb in (16, 128):
        sub = verts[:64 * nb]
        dawn.apsp(G, sub[:128]); torch.cuda.synchronize()
        t = time.time(); r = dawn.apsp(G, sub); torch.cuda.synchronize(); dt = time.time() - t
        print("ms_alpha", a, "apsp", len(sub), "sources in %.4f s -> %.0f sources/s" % (dt, len(sub) / dt))
