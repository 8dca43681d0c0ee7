# Repeat the C2 bench sources many times and certify every distance vector (race hunting).
import os, sys, numpy as np, torch
sys.path.insert(0, '.')
import graphgen, oracle, paper_2208_04514_b200 as dawn
g = graphgen.config_graph(os.environ.get("CFG", "C2"))
G = dawn.Graph(g.row_ptr, g.col, True)
srcs = g.sample_sources(64, seed=1)
reps = int(os.environ.get("REPS", "4"))
bad = 0
outs = [torch.empty(g.n, dtype=torch.int32, device="cuda") for _ in range(16)]
for r in range(reps):
    for i, s in enumerate(srcs):
        o = outs[i % 16]
        dawn.sssp(G, int(s), "auto", out=o)
        if i % 16 == 15 or i == len(srcs) - 1:
            torch.cuda.synchronize()
            for j in range(i - (i % 16), i + 1):
                d = outs[j % 16].cpu().numpy().view(np.uint32)
                c = oracle.certify(g.n, g.row_ptr, g.col, g.row_ptr, g.col, int(srcs[j]), d)
                if c != 0:
                    bad += 1
                    print("rep", r, "source", int(srcs[j]), "certify", c, flush=True)
print(os.environ.get("DAWN_LIB", "libdawn"), "bad", bad, "of", reps * len(srcs))
