# Per-level timeline of the first 256-source batch of k_ms64 on C5 (graph built with trace=True)
import sys, numpy as np, torch
sys.path.insert(0, '.')
import graphgen, paper_2208_04514_b200 as dawn
g = graphgen.config_graph("C5"); G = dawn.Graph(g.row_ptr, g.col, True, trace=True)
verts, e = g.largest_wcc()
for rep in range(2):
    dawn.apsp(G, verts[:256]); torch.cuda.synchronize()
tr = G.trace()
t0 = int(tr["t_ns"][0])
for r in tr:
    nw = 148 * 16
    print("L%d %s n_active=%d m_active=%d start=%.1f us  slowest warp us [pass A, barrier wait, pass B, records] = %s  pass A mean %.1f us, slowest light part %.1f us" % (r["level"], "PUSH PULL STOP".split()[r["dir"]], r["nf"], r["mf"], (int(r["t_ns"]) - t0) / 1e3, [round(int(c) / 1965.0, 1) for c in r["cyc"][:4]], int(r["t_first"]) / nw / 1965.0, int(r["t_last"]) / 1965.0))
