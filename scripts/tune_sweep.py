"""Sweep k_sssp tunables on the bench sources (dawn_sssp_batch with the default lanes, L2 flushed
per step): python scripts/tune_sweep.py C4 [alpha=1,2,4]"""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import bench, graphgen, paper_2208_04514_b200 as dawn

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
g = graphgen.config_graph(cfg)
G = bench.dev_graph(g)
srcs = bench.sources_for(g, cfg, 0)
dsrc = torch.from_numpy(srcs.astype(np.int32)).cuda()
out = torch.empty((len(srcs), g.n), dtype=torch.int32, device="cuda")
flush = torch.empty(int(2.2 * bench.L2_BYTES) // 4, dtype=torch.int32, device="cuda")


def t():
    for _ in range(2):
        dawn.sssp_batch(G, dsrc, out=out)
    ts = []
    for _ in range(6):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dawn.sssp_batch(G, dsrc, out=out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return np.median(ts) * 1e3 / len(srcs)


base = dict(solo_edges=512, bitmap_push_grow_edges=4096, bitmap_push_edges=1 << 18, alpha=2, beta=96)
print(cfg, "default us/search %.2f" % t(), flush=True)
SWEEP = {"alpha": (1, 4, 8), "beta": (48, 192), "bitmap_push_edges": (1 << 16, 1 << 20),
         "solo_edges": (128, 2048)}
if len(sys.argv) > 2:
    k, v = sys.argv[2].split("=")
    SWEEP = {k: tuple(float(x) for x in v.split(","))}
for k, vals in SWEEP.items():
    for v in vals:
        G.set_tuning(**{k: v})
        r = t()
        G.set_tuning(**{k: base[k]})
        print(cfg, k, v, "us/search %.2f" % r, flush=True)
