import sys, numpy as np
sys.path.insert(0, '.')
import graphgen, oracle, paper_2208_04514_b200 as dawn
g = graphgen.config_graph("C2")
G = dawn.Graph(g.row_ptr, g.col, True, trace=True)
srcs = g.sample_sources(64, seed=1)[:6]
for s in srcs:
    exp, _ = oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(s))
    rec, er = oracle.record(g.n, g.row_ptr, int(s), exp)
    for knobs in (dict(bitmap_push_edges=1 << 18), dict(bitmap_push_edges=1 << 40)):
        G.set_tuning(**knobs)
        for v in ("auto", "push", "pull"):
            d, st = dawn.sssp(G, int(s), v, stats=True)
            d = d.cpu().numpy().view(np.uint32); st = dawn.stats_to_dict(st)
            ok = np.array_equal(d, exp) and st["edges_reach"] == er and st["levels"] == int(rec["ecc"]) and st["reached"] == int(rec["reached"])
            if not ok:
                tr = G.trace()
                print("MISMATCH", s, v, knobs, st, "oracle ecc", int(rec["ecc"]), "reached", int(rec["reached"]), "er", er, "dist_ok", np.array_equal(d, exp))
                print("   hist", np.bincount(exp[exp != 0xFFFFFFFF]).tolist())
                for r in tr: print("   L%d dir=%d nf=%d mf=%d rep=%d" % (r["level"], r["dir"], r["nf"], r["mf"], r["rep"]))
print("done")
