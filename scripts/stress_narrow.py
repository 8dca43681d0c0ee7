# Repeat cluster-start searches on meshes and random low-degree graphs and check every distance
# vector against the oracle (the relaxed cluster barrier and the DSMEM exchange under load).
import sys, numpy as np, torch
sys.path.insert(0, '.')
import graphgen, oracle, paper_2208_04514_b200 as dawn
rng = np.random.default_rng(5)
cases = [graphgen.grid(1024, 1024), graphgen.grid(300, 3000),
         graphgen.from_edges(200_000, rng.integers(0, 200_000, size=(300_000, 2)), symmetric=True)]
bad = tot = 0
for g in cases:
    G = dawn.Graph(g.row_ptr, g.col, True)
    G.set_tuning(cluster_start=1)
    srcs = [0, g.n - 1] + list(g.sample_sources(6, seed=9))
    exp = {int(s): oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(s))[0] for s in srcs}
    for rep in range(5):
        for s in srcs:
            d = dawn.sssp(G, int(s)).cpu().numpy().view(np.uint32)
            tot += 1
            if not np.array_equal(d, exp[int(s)]):
                bad += 1
                print("MISMATCH", g.name, int(s), rep, int((d != exp[int(s)]).sum()), flush=True)
C3 = graphgen.config_graph("C3")
G3 = dawn.Graph(C3.row_ptr, C3.col, True)
W = 4096
r, c = np.divmod(np.arange(C3.n, dtype=np.int64), W)
for rep in range(3):
    d = dawn.sssp(G3, 0).cpu().numpy().view(np.uint32).astype(np.int64)
    tot += 1
    if not np.array_equal(d, r + c):
        bad += 1
        print("C3 MISMATCH rep", rep, flush=True)
print("narrow stress bad", bad, "of", tot)
