"""Time the fused partitioned search (W = 1 on one GPU) on the bench's C4 sources:
python scripts/part_bench.py [C4] [sources]"""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import bench, graphgen, paper_2208_04514_b200 as dawn

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 8
g = graphgen.config_graph(cfg)
pg = dawn.PartGraph(dawn.part_build(g.row_ptr, g.col, 1, 0), 1, 0)
srcs = bench.sources_for(g, cfg)[:k]
out = torch.empty(pg.R, dtype=torch.int32, device="cuda")
for s in srcs[:2]:
    dawn.part_sssp_fused(pg, int(s), "auto", out=out)
torch.cuda.synchronize()
ts = []
for s in srcs:
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    dawn.part_sssp_fused(pg, int(s), "auto", out=out)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(cfg, "fused W=1 ms per search: median %.3f mean %.3f  GTEPS %.1f" %
      (np.median(ts), np.mean(ts), g.m / (np.mean(ts) * 1e-3) / 1e9))
