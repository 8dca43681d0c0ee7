# One dawn_sssp_batch over a config's 64 bench sources (for ncu captures of a lane launch):
#   python scripts/one_batch.py C2 [reps]
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import bench, graphgen, paper_2208_04514_b200 as dawn
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = graphgen.config_graph(cfg)
G = bench.dev_graph(g)
src = torch.from_numpy(bench.sources_for(g, cfg).astype(np.int32)).cuda()
for _ in range(reps):
    dawn.sssp_batch(G, src)
torch.cuda.synchronize()
print("done")
