# quick timing probe (not the bench): SSSP on kron-20 per variant, APSP rate on kron-18.
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import graphgen, paper_2208_04514_b200 as dawn
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
g = graphgen.kron(scale); G = dawn.Graph(g.row_ptr, g.col, True)
srcs = g.sample_sources(16, 1)
for v in ("auto", "push", "pull"):
    for s in srcs[:3]: dawn.sssp(G, int(s), v)
    torch.cuda.synchronize()
    ts = []; er = 0
    for s in srcs:
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); d, st = dawn.sssp(G, int(s), v, stats=True); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1)); er += dawn.stats_to_dict(st)["edges_reach"]
    print(v, "ms/sssp median %.4f mean %.4f" % (np.median(ts), np.mean(ts)), "GTEPS %.1f" % (er / (sum(ts) * 1e-3) / 1e9), dawn.stats_to_dict(st))
g = graphgen.kron(18); G = dawn.Graph(g.row_ptr, g.col, True)
verts, e = g.largest_wcc()
for nb in (4, 64):
    sub = verts[:64 * nb]
    dawn.apsp(G, sub[:128]); torch.cuda.synchronize()
    t = time.time(); r = dawn.apsp(G, sub); torch.cuda.synchronize(); dt = time.time() - t
    print("apsp", len(sub), "sources in %.4f s -> %.0f sources/s" % (dt, len(sub) / dt))
