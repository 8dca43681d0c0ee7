# per-source graph replay vs one dawn_sssp_batch call on the bench sources of each config
# (C1 / C3: the bench source repeated 64 / 1 times)
import sys, numpy as np, torch
sys.path.insert(0, '.')
import bench, paper_2208_04514_b200 as dawn
for cfg in sys.argv[1:] or ["C1", "C2", "C3", "C4"]:
    g = bench.build_graph(cfg)
    G = dawn.Graph(g.row_ptr, g.col, g.symmetric, *(g.transpose() if not g.symmetric else (None, None)))
    srcs = bench.sources_for(g, cfg, 0)
    if cfg == "C1":
        srcs = np.repeat(srcs, 64)
    k = len(srcs)
    dsrc = torch.from_numpy(srcs.astype(np.int32)).cuda()
    out = torch.empty((k, g.n), dtype=torch.int32, device="cuda")
    ref = torch.empty_like(out)
    for i, s in enumerate(srcs): dawn.sssp(G, int(s), out=ref[i])
    dawn.sssp_batch(G, dsrc, out=out); torch.cuda.synchronize()
    assert torch.equal(out, ref), "batch differs"
    graph = torch.cuda.CUDAGraph(); cap = torch.cuda.Stream(); cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(graph, stream=cap):
        for i, s in enumerate(srcs): dawn.sssp(G, int(s), out=ref[i])
    for name, fn in (("graph", graph.replay), ("batch", lambda: dawn.sssp_batch(G, dsrc, out=out))):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
        print(cfg, name, "k", k, "us per source %.2f" % (np.median(ts) * 1e3 / k), flush=True)
