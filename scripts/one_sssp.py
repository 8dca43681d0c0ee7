# Run a few dawn_sssp calls on one config (for ncu captures):
#   python scripts/one_sssp.py C3 [reps] [variant]
import sys, torch
sys.path.insert(0, '.')
import graphgen, paper_2208_04514_b200 as dawn
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
variant = sys.argv[3] if len(sys.argv) > 3 else "auto"
g = graphgen.config_graph(cfg)
G = dawn.Graph(g.row_ptr, g.col, g.symmetric, *(g.transpose() if not g.symmetric else (None, None)))
srcs = [0] if cfg in ("C1", "C3") else list(g.sample_sources(reps, 1))
for i in range(reps):
    dawn.sssp(G, int(srcs[i % len(srcs)]), variant)
torch.cuda.synchronize()
print("done")
