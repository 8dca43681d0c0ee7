"""dawn_wsssp near/far step sweep (DAWN_PARAM_WEIGHT_DELTA) on a config graph with the bench
weights: python scripts/wdelta_sweep.py C4 0,16,32,64,128,256"""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import bench, graphgen, paper_2208_04514_b200 as dawn

cfg = sys.argv[1]
deltas = [int(x) for x in sys.argv[2].split(",")]
g = graphgen.config_graph(cfg)
G = dawn.Graph(g.row_ptr, g.col, True)
wt = torch.from_numpy(g.weights(seed=int(cfg[1:]), wmax=255).view(np.int32)).cuda()
srcs = bench.sources_for(g, cfg)[:4]
out = torch.empty(g.n, dtype=torch.int32, device="cuda")
ref = None
for dl in deltas:
    G.set_tuning(weight_delta=dl)
    er, rd, rl, rows = 0, [], [], []
    for s in srcs:
        d, st = dawn.wsssp(G, int(s), wt, stats=True, out=out)
        x = dawn.stats_to_dict(st)
        er += x["edges_reach"]; rd.append(x["levels"]); rl.append(x["edges_examined"])
        rows.append(d.clone())
    if ref is None:
        ref = rows
    assert all(torch.equal(a, b) for a, b in zip(rows, ref)), dl
    ms = bench.timed(lambda: [dawn.wsssp(G, int(s), wt, out=out) for s in srcs], 3,
                     torch.empty(4, device="cuda"), torch.cuda.current_stream())
    t = float(np.median(ms))
    print(cfg, "delta", dl, "GTEPS %.1f" % (er / (t * 1e-3) / 1e9), "ms/search %.2f" % (t / len(srcs)),
          "rounds %.1f" % np.mean(rd), "relaxed/m %.2f" % (np.mean(rl) / g.m), flush=True)
