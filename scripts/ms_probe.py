# APSP rate on C5 for several ms_alpha values (and the level trace of the first batch)
import os, sys, time, numpy as np, torch
sys.path.insert(0, '.')
import graphgen, paper_2208_04514_b200 as dawn
g = graphgen.config_graph("C5"); G = dawn.Graph(g.row_ptr, g.col, True)
verts, e = g.largest_wcc()
sub = verts[: 256 * int(os.environ.get("NB", "64"))]
for a in [float(x) for x in os.environ.get("ALPHAS", "2").split(",")]:
    G.set_tuning(ms_alpha=a)
    dawn.apsp(G, sub[:512]); torch.cuda.synchronize()
    t = time.time(); dawn.apsp(G, sub); torch.cuda.synchronize(); dt = time.time() - t
    print(f"{os.environ.get('DAWN_LIB','libdawn')} ms_alpha {a}: {len(sub)/dt:.0f} sources/s")
