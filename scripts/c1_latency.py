"""C1 single-search latency per small-kernel variant (auto -> k_small_pull, push -> k_small),
with and without an L2 flush before each call: python scripts/c1_latency.py"""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import bench, graphgen, paper_2208_04514_b200 as dawn

g = graphgen.config_graph("C1")
G = bench.dev_graph(g)
out = torch.empty(g.n, dtype=torch.int32, device="cuda")
flush = torch.empty(int(2.2 * bench.L2_BYTES) // 4, dtype=torch.int32, device="cuda")
small = torch.empty(4, dtype=torch.int32, device="cuda")
def gap_free(v, reps=20):
    """kernel time alone: a sleep kernel ahead of the first event keeps the GPU busy while the
    host queues the search, so no launch latency lands between the events"""
    ts = []
    for _ in range(reps):
        torch.cuda._sleep(200000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dawn.sssp(G, 0, v, out=out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return np.median(ts) * 1e3


for v in ("auto", "push"):
    print("C1", v, "queued (kernel only) median us %.2f" % gap_free(v))
    for fl, name in ((flush, "flushed"), (small, "warm")):
        for _ in range(5):
            dawn.sssp(G, 0, v, out=out)
        ms = bench.timed(lambda: dawn.sssp(G, 0, v, out=out), 20, fl, torch.cuda.current_stream())
        print("C1", v, name, "median us %.2f" % (np.median(ms) * 1e3), "min %.2f" % (np.min(ms) * 1e3))
