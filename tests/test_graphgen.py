"""Input generator invariants (SURVEY §8(d) input recipe)."""
import numpy as np
import pytest

import graphgen


def _check_csr(g):
    rp, col = g.row_ptr, g.col
    assert rp[0] == 0 and rp[-1] == len(col) and np.all(np.diff(rp) >= 0)
    assert col.min(initial=0) >= 0 and col.max(initial=-1) < g.n
    src = np.repeat(np.arange(g.n), np.diff(rp))
    assert not np.any(src == col), "self-loop"
    key = src.astype(np.int64) * g.n + col
    assert np.all(np.diff(key) > 0), "rows sorted, no duplicates"
    return src


def test_build_csr_spec_examples():
    g = graphgen.from_edges(3, [[0, 1], [0, 2], [2, 1]])
    assert g.row_ptr.tolist() == [0, 2, 2, 3] and g.col.tolist() == [1, 2, 1]
    g = graphgen.from_edges(2, np.zeros((0, 2)))
    assert g.row_ptr.tolist() == [0, 0, 0] and g.col.tolist() == []
    g = graphgen.from_edges(3, [[0, 0], [0, 1], [0, 1]])          # loop dropped, dedup
    assert g.col.tolist() == [1]


def test_transpose_is_exact():
    g = graphgen.er_prob(64, 0.1, 1)
    p, i = g.transpose()
    src = _check_csr(g)
    t = graphgen.Graph(g.n, p, i, False)
    tsrc = _check_csr(t)
    assert sorted(zip(src.tolist(), g.col.tolist())) == sorted(zip(i.tolist(), tsrc.tolist()))


@pytest.mark.parametrize("scale", [8, 12])
def test_kron_deterministic_symmetric(scale, monkeypatch):
    a = graphgen.kron(scale, 16)
    monkeypatch.setenv("GRAPHGEN_THREADS", "1")
    b = graphgen.kron(scale, 16)
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col, b.col)
    src = _check_csr(a)
    fwd = set(zip(src.tolist(), a.col.tolist()))
    assert all((v, u) in fwd for (u, v) in list(fwd)[:5000])


def test_kron18_shape_matches_survey_workload():
    # n = 262,144, m ~ 7.61 M, S_wcc ~ 173.8 K (survey's numpy sample)
    g = graphgen.kron(18)
    assert g.n == 262144
    assert abs(g.m - 7_613_888) / 7_613_888 < 0.01
    v, e = g.largest_wcc()
    assert abs(len(v) - 173_778) / 173_778 < 0.01
    assert e <= g.m


def test_er_and_grid():
    g = graphgen.er(1000, 8000, 1)
    assert g.n == 1000 and g.m == 8000
    _check_csr(g)
    g2 = graphgen.er(1000, 8000, 1)
    assert np.array_equal(g.col, g2.col)
    gr = graphgen.grid(5, 4)
    _check_csr(gr)
    assert gr.m == 2 * (4 * 4 + 5 * 3)


def test_sources_deterministic_and_positive_degree():
    g = graphgen.kron(12)
    s1, s2 = g.sample_sources(64, 1), g.sample_sources(64, 1)
    assert np.array_equal(s1, s2) and len(s1) == 64
    assert np.all(g.degrees()[s1] > 0)
