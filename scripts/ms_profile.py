# Per-level trace of the first 256-source batch of an APSP call (kron-18, C5 sources).
import os, sys, time, numpy as np, torch
sys.path.insert(0, '.')
import graphgen, paper_2208_04514_b200 as dawn
g = graphgen.config_graph("C5")
G = dawn.Graph(g.row_ptr, g.col, True, trace=True)
if os.environ.get("MS_ALPHA"): G.set_tuning(ms_alpha=float(os.environ["MS_ALPHA"]))
verts, _ = g.largest_wcc()
for nb in (1, 32):
    sub = verts[:256 * nb]
    dawn.apsp(G, sub); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); dawn.apsp(G, sub); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{len(sub)} sources: {ms*1e3:.0f} us, {len(sub)/ms*1e3:.0f} sources/s, {ms*1e3/nb:.0f} us/batch")
tr = G.trace(); t0 = int(tr["t_ns"][0])
for r in tr:
    print("  L%d %s n_active=%d m_active=%d start=%.1f" % (r["level"], "PUSH PULL STOP".split()[r["dir"]], r["nf"], r["mf"], (int(r["t_ns"]) - t0) / 1e3))
