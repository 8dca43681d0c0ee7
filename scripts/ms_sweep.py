"""k_ms64 tunable sweep on C5 (APSP over the largest WCC, default lanes):
python scripts/ms_sweep.py ms_alpha=1,2,4,8"""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import graphgen, paper_2208_04514_b200 as dawn

g = graphgen.config_graph("C5")
G = dawn.Graph(g.row_ptr, g.col, True)
verts, _ = dawn.largest_wcc(G)
k, vals = sys.argv[1].split("=")
for v in [float(x) for x in vals.split(",")]:
    G.set_tuning(**{k: v})
    dawn.apsp(G, verts)
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dawn.apsp(G, verts)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print("C5", k, v, "sources/s %.0f" % (len(verts) / (np.median(ts) * 1e-3)), flush=True)
