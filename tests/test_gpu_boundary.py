"""GPU tests of the boundary (§8(b)) added in round 2: device-side validation of the
dawn_sssp_batch source list (validation before work), the device largest-WCC
helper dawn_largest_wcc (PAPER Table 1, reading Q15) against the oracle, and the
memory-frugal DAWN_GRAPH_LEAN residency giving the same distances."""
import numpy as np
import pytest
import torch

import graphgen
import oracle
import paper_2208_04514_b200 as dawn

pytestmark = pytest.mark.gpu
UNR = oracle.UNREACHED


def _graph(g, **kw):
    if g.symmetric:
        return dawn.Graph(g.row_ptr, g.col, True, validate=True, **kw)
    p, i = g.transpose()
    return dawn.Graph(g.row_ptr, g.col, False, p, i, validate=True, **kw)


def _bad_batch_writes_nothing(G, n, good):
    """A batch whose LAST source id is n: nothing may be written, check() raises BOUNDS, and a
    following valid batch on the same handle works (the flag was cleared)."""
    src = torch.tensor(list(good) + [n], dtype=torch.int32, device="cuda")
    k = src.numel()
    sentinel = torch.full((k, n), 0x5A5A5A5A, dtype=torch.int32, device="cuda")
    st = torch.full((k, 4), 0x0123456789, dtype=torch.int64, device="cuda")
    dawn.lib()  # the call itself only enqueues (the ids are device-resident)
    dawn._check(dawn.lib().dawn_sssp_batch(G.handle, src.data_ptr(), k, 0, sentinel.data_ptr(),
                                           st.data_ptr(), torch.cuda.current_stream().cuda_stream))
    with pytest.raises(dawn.DawnError) as ei:
        dawn.check(G)
    assert ei.value.status == 2  # DAWN_ERR_BOUNDS
    assert bool((sentinel == 0x5A5A5A5A).all()), "a rejected batch wrote distances"
    assert bool((st == 0x0123456789).all()), "a rejected batch wrote statistics"
    dawn.check(G)  # cleared
    d = dawn.sssp_batch(G, src[:-1], check=True)
    return d.cpu().numpy().view(np.uint32)


def test_batch_out_of_range_source_k_small():
    g = graphgen.er(1000, 8000, 1)                      # k_small (CSR in shared memory)
    G = _graph(g)
    d = _bad_batch_writes_nothing(G, g.n, [0, 5, 999])
    for row, s in zip(d, [0, 5, 999]):
        assert np.array_equal(row, oracle.bfs_fifo(g.n, g.row_ptr, g.col, s)[0])


def test_batch_out_of_range_source_k_sssp():
    g = graphgen.kron(14, 16, 14)                       # grid-wide k_sssp
    G = _graph(g)
    srcs = [int(x) for x in g.sample_sources(3, seed=2)]
    d = _bad_batch_writes_nothing(G, g.n, srcs)
    for row, s in zip(d, srcs):
        assert np.array_equal(row, oracle.bfs_fifo(g.n, g.row_ptr, g.col, s)[0])


def test_batch_out_of_range_source_cluster_start():
    g = graphgen.grid(300, 200)                         # k_narrow + k_sssp per search
    G = _graph(g)
    d = _bad_batch_writes_nothing(G, g.n, [0, 777])
    for row, s in zip(d, [0, 777]):
        assert np.array_equal(row, oracle.bfs_fifo(g.n, g.row_ptr, g.col, s)[0])


def test_batch_huge_source_id():
    g = graphgen.kron(12, 16, 12)
    G = _graph(g)
    src = torch.tensor([0, -1], dtype=torch.int32, device="cuda")  # 0xFFFFFFFF as uint32
    out = torch.full((2, g.n), 7, dtype=torch.int32, device="cuda")
    with pytest.raises(dawn.DawnError):
        dawn.sssp_batch(G, src, out=out, check=True)
    assert bool((out == 7).all())


def test_largest_wcc_matches_oracle():
    rng = np.random.default_rng(5)
    graphs = [graphgen.config_graph("C5"), graphgen.kron(12, 16, 12), graphgen.grid(50, 40),
              graphgen.config_graph("C1")]
    for t in range(12):                                  # fragmented ER digraphs: many ties
        n = int(rng.integers(2, 3000))
        graphs.append(graphgen.er_prob(n, float(rng.choice([0.0005, 0.001, 0.003])), 300 + t))
    graphs += [graphgen.from_edges(6, [[0, 1], [2, 3]]), graphgen.from_edges(1, []),
               graphgen.from_edges(6, [[1, 0], [2, 0], [4, 3]]),
               graphgen.from_edges(6, [[0, 1], [1, 2], [3, 4], [4, 5], [5, 3]])]
    for g in graphs:
        G = _graph(g)
        ov, oe = oracle.largest_wcc(g.n, g.row_ptr, g.col)
        for rep in range(6):  # repeated: the union-find is lock-free (a labelling race once
            v, e = dawn.largest_wcc(G)  # dropped a vertex from the compaction)
            assert np.array_equal(v, ov) and e == oe, (g.name, rep, len(v), len(ov), e, oe)


def test_largest_wcc_hub_rows():
    # rows longer than kHeavy go through the static 256-arc pieces
    n = 200_000
    rng = np.random.default_rng(9)
    hubs = rng.integers(0, n, size=4)
    edges = [(int(h), int(u)) for h in hubs for u in rng.integers(0, n, size=70_000)]
    edges += [(int(a), int(b)) for a, b in rng.integers(0, n, size=(30_000, 2))]
    g = graphgen.from_edges(n, edges, symmetric=True)
    G = _graph(g)
    v, e = dawn.largest_wcc(G)
    ov, oe = oracle.largest_wcc(g.n, g.row_ptr, g.col)
    assert np.array_equal(v, ov) and e == oe


def test_lean_residency_same_distances():
    for g in (graphgen.kron(14, 16, 14), graphgen.grid(300, 200), graphgen.er(5000, 40000, 3)):
        G = _graph(g, lean=True)
        for s in [0, g.n // 2] + [int(x) for x in g.sample_sources(2, seed=4)]:
            exp = oracle.bfs_fifo(g.n, g.row_ptr, g.col, s)[0]
            for v in ("auto", "push", "pull"):
                d = dawn.sssp(G, s, v).cpu().numpy().view(np.uint32)
                assert np.array_equal(d, exp), (g.name, s, v)
        with pytest.raises(dawn.DawnError) as ei:
            dawn.msssp(G, [0])
        assert ei.value.status == 3  # DAWN_ERR_CONFIG
        v, e = dawn.largest_wcc(G)
        assert np.array_equal(v, oracle.largest_wcc(g.n, g.row_ptr, g.col)[0])
