"""GPU parity of the weighted (min,+) extension (reading
Q26): dawn_wsssp against the CPU oracle (Dijkstra / (min,+) SOVM rounds), element by element,
plus the weighted certificate at Kronecker-20 scale."""
import numpy as np
import pytest
import torch

import graphgen
import oracle
import paper_2208_04514_b200 as dawn

pytestmark = pytest.mark.gpu
U32 = 0xFFFFFFFF


def _graph(g):
    if g.symmetric:
        return dawn.Graph(g.row_ptr, g.col, True, validate=True)
    p, i = g.transpose()
    return dawn.Graph(g.row_ptr, g.col, False, p, i, validate=True)


def _exp32(d64):
    return np.where(d64 == oracle.UNREACHED64, U32, d64).astype(np.uint32)


def _check(g, w, sources, G=None):
    G = G or _graph(g)
    wt = torch.from_numpy(w.view(np.int32)).cuda()
    for s in sources:
        d, st = dawn.wsssp(G, int(s), wt, stats=True)
        d = d.cpu().numpy().view(np.uint32)
        exp = _exp32(oracle.dijkstra(g.n, g.row_ptr, g.col, w, int(s)))
        bad = np.nonzero(d != exp)[0]
        assert len(bad) == 0, (g.name, s, bad[:5], d[bad[:5]], exp[bad[:5]])
        x = dawn.stats_to_dict(st)
        reach = exp != U32
        assert x["reached"] == int(reach.sum()) - 1
        assert x["edges_reach"] == int(np.diff(g.row_ptr)[reach].sum())
    return G


def test_textbook_example():
    # CLRS Fig. 24.6 (hand values s 0, t 8, x 9, y 5, z 7)
    arcs = [(0, 1, 10), (0, 3, 5), (1, 2, 1), (1, 3, 2), (3, 1, 3), (3, 2, 9), (3, 4, 2),
            (2, 4, 4), (4, 2, 6), (4, 0, 7)]
    g = graphgen.from_edges(5, [(a, b) for a, b, _ in arcs])
    wmap = {(a, b): x for a, b, x in arcs}
    src = np.repeat(np.arange(g.n), np.diff(g.row_ptr))
    w = np.array([wmap[(int(a), int(b))] for a, b in zip(src, g.col)], np.uint32)
    G = _graph(g)
    d = dawn.wsssp(G, 0, torch.from_numpy(w.view(np.int32)).cuda()).cpu().numpy()
    assert d.tolist() == [0, 8, 9, 5, 7]


def test_er_corpus_random_weights():
    for seed in range(10):
        g = graphgen.er(int(200 + 80 * seed), int(1200 + 500 * seed), seed + 1)
        _check(g, g.weights(seed, 255 if seed % 2 else 7), [0, 13, g.n - 1])


def test_kron_and_hubs():
    g = graphgen.kron(13, 16, 13)
    _check(g, g.weights(2, 255), g.sample_sources(4, seed=3))
    n = 20000
    rng = np.random.default_rng(1)
    e = [(0, v) for v in range(1, n)] + [(int(a), int(b)) for a, b in rng.integers(0, n, (40000, 2))
                                         if a != b]
    h = graphgen.from_edges(n, e)
    _check(h, h.weights(9, 1000), [0, 5, n - 1])


def test_unit_weights_equal_unweighted_path():
    g = graphgen.kron(12, 16, 12)
    G = _graph(g)
    ones = torch.ones(g.m, dtype=torch.int32, device="cuda")
    for s in g.sample_sources(3, seed=5):
        d, st = dawn.wsssp(G, int(s), ones, stats=True)
        b, bst = dawn.sssp(G, int(s), stats=True)
        assert torch.equal(d, b)
        assert dawn.stats_to_dict(st)["levels"] == dawn.stats_to_dict(bst)["levels"]  # rounds = ecc


def test_grid_uniform_weight_closed_form():
    g = graphgen.grid(64, 48)
    G = _graph(g)
    w = torch.full((g.m,), 5, dtype=torch.int32, device="cuda")
    for s in (0, 48 * 0 + 63, 64 * 20 + 31):
        d = dawn.wsssp(G, s, w).cpu().numpy()
        r0, c0 = divmod(s, 64)
        v = np.arange(g.n)
        assert np.array_equal(d, 5 * (np.abs(v // 64 - r0) + np.abs(v % 64 - c0)))


def test_edge_cases_zero_weights_and_bounds():
    g = graphgen.er(500, 3000, 9)
    w = g.weights(1, 4)
    w[::3] = 0  # zero-weight arcs are allowed (non-negative weights)
    _check(g, w, [0, 250])
    one = graphgen.from_edges(1, [])
    G1 = _graph(one)
    assert dawn.wsssp(G1, 0, torch.zeros(1, dtype=torch.int32, device="cuda")[:0]).cpu().tolist() == [0]
    iso = graphgen.from_edges(10, [(1, 2)])
    _check(iso, np.array([3], np.uint32), [5, 1, 9])
    with pytest.raises(dawn.DawnError) as ei:
        dawn.wsssp(_graph(iso), 10, torch.ones(1, dtype=torch.int32, device="cuda"))
    assert ei.value.status == 2


def test_c2_certificate():
    # Kronecker-20 (C2 graph) with weights in [1, 255]: the weighted certificate (weights >= 1
    # make it a proof of exactness) on 2 sources
    g = graphgen.config_graph("C2")
    w = g.weights(20, 255)
    G = dawn.Graph(g.row_ptr, g.col, True)
    wt = torch.from_numpy(w.view(np.int32)).cuda()
    for s in g.sample_sources(2, seed=7):
        d = dawn.wsssp(G, int(s), wt).cpu().numpy().view(np.uint32).astype(np.uint64)
        d[d == U32] = oracle.UNREACHED64
        rc, bad = oracle.certify_w(g.n, g.row_ptr, g.col, w, int(s), d)
        assert rc == 0, (s, rc, bad)
    torch.cuda.synchronize()


def test_wsssp_batch_and_bounds():
    g = graphgen.kron(13, 16, 13)
    G = _graph(g)
    w = g.weights(4, 255)
    wt = torch.from_numpy(w.view(np.int32)).cuda()
    srcs = np.concatenate([g.sample_sources(9, seed=2), [0]]).astype(np.int32)
    srcs[4] = srcs[1]  # a repeated source
    exp = [_exp32(oracle.dijkstra(g.n, g.row_ptr, g.col, w, int(s))) for s in srcs]
    d, st = dawn.wsssp_batch(G, torch.from_numpy(srcs).cuda(), wt, stats=True, check=True)
    d = d.cpu().numpy().view(np.uint32)
    for i, s in enumerate(srcs):
        assert np.array_equal(d[i], exp[i]), (i, int(s))
        x = dawn.stats_to_dict(st[i])
        assert x["reached"] == int((exp[i] != U32).sum()) - 1
    bad = torch.tensor([1, 2, g.n], dtype=torch.int32, device="cuda")
    sentinel = torch.full((3, g.n), 7, dtype=torch.int32, device="cuda")
    dawn._check(dawn.lib().dawn_wsssp_batch(G.handle, bad.data_ptr(), 3, wt.data_ptr(),
                                            sentinel.data_ptr(), None,
                                            torch.cuda.current_stream().cuda_stream))
    with pytest.raises(dawn.DawnError) as ei:
        dawn.check(G)
    assert ei.value.status == 2 and bool((sentinel == 7).all())
