"""dawn_sssp_batch with a given lane count on a config's bench sources, repeated, rows checked
against single-lane results (hunting a lane-dependent fault): python scripts/lane_check.py C4 2 8 4"""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import bench, graphgen, paper_2208_04514_b200 as dawn

cfg, lanes, k, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
g = graphgen.config_graph(cfg)
G = bench.dev_graph(g)
srcs = bench.sources_for(g, cfg)[:k]
dsrc = torch.from_numpy(srcs.astype(np.int32)).cuda()
G.set_tuning(batch_lanes=1)
ref = dawn.sssp_batch(G, dsrc)
torch.cuda.synchronize()
print("reference done", flush=True)
G.set_tuning(batch_lanes=lanes)
for r in range(reps):
    d = dawn.sssp_batch(G, dsrc)
    torch.cuda.synchronize()
    print("rep", r, "equal", bool(torch.equal(d, ref)), flush=True)
