# Sweep k_sssp tunables on the bench sources (dawn_sssp_batch timing, L2 flushed per step):
# python scripts/tune_sweep.py C2
import sys, numpy as np, torch
sys.path.insert(0, '.')
import bench, paper_2208_04514_b200 as dawn
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
g = bench.build_graph(cfg)
G = dawn.Graph(g.row_ptr, g.col, g.symmetric, *(g.transpose() if not g.symmetric else (None, None)))
srcs = bench.sources_for(g, cfg, 0)
dsrc = torch.from_numpy(srcs.astype(np.int32)).cuda()
out = torch.empty((len(srcs), g.n), dtype=torch.int32, device="cuda")
flush = torch.empty(int(2.2 * 132644864) // 4, dtype=torch.int32, device="cuda")
def t():
    for _ in range(2): dawn.sssp_batch(G, dsrc, out=out)
    ts = []
    for _ in range(5):
        flush.zero_(); a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); dawn.sssp_batch(G, dsrc, out=out); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return np.median(ts) * 1e3 / len(srcs)
base = dict(solo_edges=512, bitmap_push_grow_edges=4096, bitmap_push_edges=1 << 18, alpha=2, beta=24)
print(cfg, "default us/search %.2f" % t(), flush=True)
SWEEP = {"solo_edges": (64, 128, 256, 1024, 2048), "bitmap_push_grow_edges": (1024, 2048, 8192, 16384),
         "bitmap_push_edges": (1 << 16, 1 << 17, 1 << 19, 1 << 20), "beta": (8, 16, 48), "alpha": (1, 4)}
if len(sys.argv) > 2:  # e.g. beta=32,48,64
    k, v = sys.argv[2].split("=")
    SWEEP = {k: tuple(float(x) for x in v.split(","))}
for k, vals in SWEEP.items():
    for v in vals:
        G.set_tuning(**{k: v}); r = t(); G.set_tuning(**{k: base[k]})
        print(cfg, k, v, "us/search %.2f" % r, flush=True)
