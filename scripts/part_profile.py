"""Per-level timing of the partitioned path (W = 1 on one GPU): python scripts/part_profile.py C4"""
import ctypes
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import bench, graphgen, paper_2208_04514_b200 as dawn

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
g = graphgen.config_graph(cfg)
pg = dawn.PartGraph(dawn.part_build(g.row_ptr, g.col, 1, 0), 1, 0)
srcs = bench.sources_for(g, cfg)[:3]
out = torch.empty(pg.R, dtype=torch.int32, device="cuda")
L = dawn.lib()
s = torch.cuda.current_stream().cuda_stream
for src in srcs:
    for rep in range(2):
        ev = []
        L.dawn_part_begin(pg.handle, int(src), 0, out.data_ptr(), s)
        for k in range(12):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record()
            dawn.part_exchange(pg)
            L.dawn_part_step(pg.handle, s)
            b.record()
            ev.append((a, b))
        L.dawn_part_finish(pg.handle, None, s)
        torch.cuda.synchronize()
        if rep:
            print(cfg, int(src), "per-level us:", [round(a.elapsed_time(b) * 1e3, 1) for a, b in ev])
