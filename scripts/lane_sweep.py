"""Batch-lane sweep of dawn_sssp_batch (DAWN_PARAM_BATCH_LANES) on one config's 64 bench sources:
python scripts/lane_sweep.py C2 1,2,4,6,8"""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import bench, graphgen, paper_2208_04514_b200 as dawn

cfg = sys.argv[1]
lanes = [int(x) for x in sys.argv[2].split(",")]
g = graphgen.config_graph(cfg)
print("graph", g.n, g.m, flush=True)
G = bench.dev_graph(g)
srcs = bench.sources_for(g, cfg)
dsrc = torch.from_numpy(srcs.astype(np.int32)).cuda()
out = torch.empty((len(srcs), g.n), dtype=torch.int32, device="cuda")
print("loaded", flush=True)
st = bench.search_stats(G, srcs, "auto", out) if not os.environ.get("NOSTATS") else \
    [{"edges_reach": 1}] * len(srcs)
print("stats", flush=True)
er = sum(s["edges_reach"] for s in st)
flush = torch.empty(int(2.2 * bench.L2_BYTES) // 4 if not os.environ.get("NOFLUSH") else 4,
                    dtype=torch.int32, device="cuda")
for L in lanes:
    G.set_tuning(batch_lanes=L)
    for _ in range(3):
        dawn.sssp_batch(G, dsrc, out=out)
    ms = bench.timed(lambda: dawn.sssp_batch(G, dsrc, out=out), 8, flush, torch.cuda.current_stream())
    print(cfg, "lanes", L, "GTEPS %.1f" % (er / (np.median(ms) * 1e-3) / 1e9), "ms %.3f" % np.median(ms), flush=True)
