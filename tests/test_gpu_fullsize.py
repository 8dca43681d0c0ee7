"""Full-size parity at BASELINE.json's configs, in the launch configuration bench.py times.

C1..C4: distances of sampled sources compared element by element with the oracle (FIFO BFS,
Algorithm 3 — O(n+m), so full size is affordable), every variant; C3 additionally against its
closed form (Manhattan distance) for the whole 2^24-vertex vector.  C5: every largest-WCC
source's record checked against the E10/E11 property (reached = S_wcc - 1) and a seeded sample
of 256 records bit-exact against the oracle.
"""
import numpy as np
import pytest
import torch

import graphgen
import oracle
import paper_2208_04514_b200 as dawn

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
UNR = oracle.UNREACHED


def _dev(g):
    if g.symmetric:
        return dawn.Graph(g.row_ptr, g.col, True)
    p, i = g.transpose()
    return dawn.Graph(g.row_ptr, g.col, False, p, i)


def _check(g, G, srcs, variants=("auto", "push", "pull")):
    for s in srcs:
        exp, _ = oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(s))
        rec, er = oracle.record(g.n, g.row_ptr, int(s), exp)
        for v in variants:
            d, st = dawn.sssp(G, int(s), v, stats=True)
            d = d.cpu().numpy().view(np.uint32)
            st = dawn.stats_to_dict(st)
            bad = np.nonzero(d != exp)[0]
            assert len(bad) == 0, (g.name, s, v, bad[:5])
            assert st["edges_reach"] == er and st["levels"] == int(rec["ecc"])


@pytest.fixture(scope="module")
def c2():
    g = graphgen.config_graph("C2")
    return g, _dev(g)


def _batch(G, srcs):
    """dawn_sssp_batch, the call bench.py times, as uint32 numpy rows."""
    d = dawn.sssp_batch(G, torch.from_numpy(np.asarray(srcs, dtype=np.int32)).cuda())
    return d.cpu().numpy().view(np.uint32)


def test_c1_full():
    g = graphgen.config_graph("C1")
    G = _dev(g)
    _check(g, G, [0] + list(range(1, 1000, 97)))
    # the bench step: source 0 repeated 64 times, concurrent one-CTA searches
    exp, _ = oracle.bfs_fifo(g.n, g.row_ptr, g.col, 0)
    d = _batch(G, [0] * 64)
    assert all(np.array_equal(row, exp) for row in d)


def test_c2_full_sampled_sources(c2):
    g, G = c2
    srcs = g.sample_sources(64, seed=1)          # the bench's sources (rank 0)
    _check(g, G, srcs[:6])
    # certificate (an exact proof) on all 64 bench sources, auto variant
    for s in srcs:
        d = dawn.sssp(G, int(s)).cpu().numpy().view(np.uint32)
        assert oracle.certify(g.n, g.row_ptr, g.col, g.row_ptr, g.col, int(s), d) == 0
    # the bench step: one dawn_sssp_batch over the 64 sources; every row certified
    D = _batch(G, srcs)
    assert np.array_equal(D[0], oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(srcs[0]))[0])
    for s, d in zip(srcs, D):
        assert oracle.certify(g.n, g.row_ptr, g.col, g.row_ptr, g.col, int(s), d) == 0


def test_c2_msssp_records_match(c2):
    g, G = c2
    srcs = g.sample_sources(64, seed=1)
    _, r = dawn.msssp(G, srcs, dist=False)
    got = dawn.records_to_numpy(r)
    exp = oracle.records(g.n, g.row_ptr, g.col, srcs)
    assert got.tobytes() == exp.tobytes()


def test_c3_grid_closed_form():
    g = graphgen.config_graph("C3")
    G = _dev(g)
    W = 4096
    r, c = np.divmod(np.arange(W * W, dtype=np.int64), W)
    for s in (0, (W // 2) * W + W // 2):
        r0, c0 = divmod(s, W)
        exp = (np.abs(r - r0) + np.abs(c - c0)).astype(np.uint32)
        for v in ("auto", "push"):
            d = dawn.sssp(G, s, v).cpu().numpy().view(np.uint32)
            assert np.array_equal(d, exp), (s, v)
        assert np.array_equal(_batch(G, [s])[0], exp), s      # the bench's call


def test_c4_full_sampled_sources():
    g = graphgen.config_graph("C4")
    G = _dev(g)
    srcs = g.sample_sources(64, seed=1)
    _check(g, G, srcs[:2], variants=("auto", "push"))
    _check(g, G, srcs[2:3], variants=("pull",))
    # the bench step (one dawn_sssp_batch over the 64 sources, 2-CTA/SM kernel): two rows
    # element by element against the oracle, two more certified
    D = _batch(G, srcs)
    for i in (0, 63):
        assert np.array_equal(D[i], oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(srcs[i]))[0]), i
    for i in (17, 40):
        assert oracle.certify(g.n, g.row_ptr, g.col, g.row_ptr, g.col, int(srcs[i]), D[i]) == 0


def test_c5_apsp_all_sources():
    g = graphgen.config_graph("C5")
    G = _dev(g)
    verts, e_wcc = g.largest_wcc()
    rec = dawn.records_to_numpy(dawn.apsp(G, verts))
    assert np.array_equal(rec["source"], verts.astype(np.uint32))
    assert np.all(rec["reached"] == len(verts) - 1)        # E10/E11
    rng = np.random.default_rng(18)
    pick = np.sort(rng.choice(len(verts), 256, replace=False))
    exp = oracle.records(g.n, g.row_ptr, g.col, verts[pick])
    assert rec[pick].tobytes() == exp.tobytes()
