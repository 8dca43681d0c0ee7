"""A few fused partitioned searches on one config (for ncu captures): python scripts/part_one.py C4 3"""
import sys
import torch
sys.path.insert(0, '.')
import bench, graphgen, paper_2208_04514_b200 as dawn
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = graphgen.config_graph(cfg)
pg = dawn.PartGraph(dawn.part_build(g.row_ptr, g.col, 1, 0), 1, 0)
for s in bench.sources_for(g, cfg)[:reps]:
    dawn.part_sssp_fused(pg, int(s))
torch.cuda.synchronize()
print("done")
