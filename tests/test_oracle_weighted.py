"""Pins of the weighted (min,+) oracle (reading Q26).

oracle_minplus follows the (min,+) generalisation of Algorithm 2's rounds; it is pinned against
things other than itself: a textbook worked example (hand values), closed forms (weighted path,
uniform-weight grid), the unweighted oracle under unit weights (incl. the round count = ecc),
brute-force enumeration of simple paths on tiny graphs, an independent Dijkstra and weighted
Floyd-Warshall, and the weighted certificate (which must reject every single-entry change)."""
import itertools

import numpy as np
import pytest

import graphgen
import oracle

U64 = oracle.UNREACHED64


def _csr(n, arcs):
    arcs = sorted(arcs)
    rp = np.zeros(n + 1, np.int64)
    for u, _, _ in arcs:
        rp[u + 1] += 1
    rp = np.cumsum(rp)
    col = np.array([v for _, v, _ in arcs], np.int32)
    w = np.array([x for _, _, x in arcs], np.uint32)
    return rp, col, w


def test_textbook_dijkstra_example():
    # CLRS (3rd ed.) Fig. 24.6: s=0 t=1 x=2 y=3 z=4; d = s 0, t 8, x 9, y 5, z 7 (hand values)
    arcs = [(0, 1, 10), (0, 3, 5), (1, 2, 1), (1, 3, 2), (3, 1, 3), (3, 2, 9), (3, 4, 2),
            (2, 4, 4), (4, 2, 6), (4, 0, 7)]
    rp, col, w = _csr(5, arcs)
    exp = [0, 8, 9, 5, 7]
    assert oracle.minplus(5, rp, col, w, 0)[0].tolist() == exp
    assert oracle.dijkstra(5, rp, col, w, 0).tolist() == exp
    assert oracle.floyd_warshall_w(5, rp, col, w)[0].tolist() == exp


def test_weighted_path_closed_form():
    n = 50
    rng = np.random.default_rng(1)
    ws = rng.integers(1, 1000, n - 1)
    rp, col, w = _csr(n, [(i, i + 1, int(ws[i])) for i in range(n - 1)])
    d, st = oracle.minplus(n, rp, col, w, 0)
    assert d.tolist() == [0] + np.cumsum(ws).tolist()
    assert st["iterations"] == n - 1
    d7, _ = oracle.minplus(n, rp, col, w, 7)
    assert d7[:7].tolist() == [U64] * 7 and d7[7:].tolist() == [0] + np.cumsum(ws[7:]).tolist()


def test_uniform_weight_grid_is_scaled_manhattan():
    g = graphgen.grid(17, 11)
    w = np.full(g.m, 3, np.uint32)
    for s in (0, 17 * 5 + 8):
        d, _ = oracle.minplus(g.n, g.row_ptr, g.col, w, s)
        r0, c0 = divmod(s, 17)
        exp = [3 * (abs(v // 17 - r0) + abs(v % 17 - c0)) for v in range(g.n)]
        assert d.tolist() == exp


def test_unit_weights_reduce_to_unweighted_oracle():
    for seed in range(8):
        g = graphgen.er(300, 1500 + 100 * seed, seed + 1)
        w = np.ones(g.m, np.uint32)
        for s in (0, 17, 299):
            d, st = oracle.minplus(g.n, g.row_ptr, g.col, w, s)
            b, _ = oracle.bfs_fifo(g.n, g.row_ptr, g.col, s)
            exp = np.where(b == oracle.UNREACHED, U64, b.astype(np.uint64))
            assert np.array_equal(d, exp)
            rec, _ = oracle.record(g.n, g.row_ptr, s, b)
            assert st["iterations"] == int(rec["ecc"])  # rounds = eccentricity


def _brute(n, arcs, s):
    adj = {}
    for u, v, x in arcs:
        adj[(u, v)] = min(x, adj.get((u, v), 1 << 60))
    best = [U64] * n
    best[s] = 0
    others = [v for v in range(n) if v != s]
    for k in range(1, n):
        for mid in itertools.permutations(others, k):
            path = (s,) + mid
            tot = 0
            for a, b in zip(path, path[1:]):
                if (a, b) not in adj:
                    break
                tot += adj[(a, b)]
            else:
                best[path[-1]] = min(best[path[-1]], tot)
    return best


def test_brute_force_simple_paths_tiny():
    rng = np.random.default_rng(7)
    for t in range(40):
        n = int(rng.integers(1, 7))
        arcs = {(int(a), int(b)): int(rng.integers(1, 20))
                for a, b in rng.integers(0, n, size=(int(rng.integers(0, 14)), 2)) if a != b}
        al = [(a, b, x) for (a, b), x in arcs.items()]
        rp, col, w = _csr(n, al)
        for s in range(n):
            exp = _brute(n, al, s)
            assert oracle.minplus(n, rp, col, w, s)[0].tolist() == exp, (t, s)
            assert oracle.dijkstra(n, rp, col, w, s).tolist() == exp, (t, s)


def test_three_way_agreement_random_weighted():
    for seed in range(6):
        g = graphgen.er(150, 900, 40 + seed)
        w = g.weights(seed, 255)
        FW = oracle.floyd_warshall_w(g.n, g.row_ptr, g.col, w)
        for s in range(0, 150, 13):
            a = oracle.minplus(g.n, g.row_ptr, g.col, w, s)[0]
            b = oracle.dijkstra(g.n, g.row_ptr, g.col, w, s)
            assert np.array_equal(a, b) and np.array_equal(a, FW[s])
    g = graphgen.kron(10, 16, 10)
    w = g.weights(3, 255)
    for s in g.sample_sources(4, seed=2):
        assert np.array_equal(oracle.minplus(g.n, g.row_ptr, g.col, w, s)[0],
                              oracle.dijkstra(g.n, g.row_ptr, g.col, w, s))


def test_certificate_accepts_truth_rejects_perturbations():
    rng = np.random.default_rng(11)
    for seed in range(10):
        g = graphgen.er(40, 160, 70 + seed)
        w = g.weights(seed, 9)
        for s in (0, 5):
            d = oracle.dijkstra(g.n, g.row_ptr, g.col, w, s)
            assert oracle.certify_w(g.n, g.row_ptr, g.col, w, s, d)[0] == 0
            for v in range(g.n):
                for delta in (-1, 1, "unr"):
                    e = d.copy()
                    if delta == "unr":
                        if e[v] == U64:
                            e[v] = 0 if v != s else 5
                        else:
                            e[v] = U64
                    elif e[v] == U64 or (delta < 0 and e[v] == 0):
                        continue
                    else:
                        e[v] = e[v] + np.uint64(1) if delta > 0 else e[v] - np.uint64(1)
                    assert oracle.certify_w(g.n, g.row_ptr, g.col, w, s, e)[0] != 0, (seed, s, v, delta)


def test_symmetric_weights_generator():
    g = graphgen.kron(9, 16, 9)
    w = g.weights(5, 100)
    assert w.min() >= 1 and w.max() <= 100
    src = np.repeat(np.arange(g.n), np.diff(g.row_ptr))
    d = {(int(a), int(b)): int(x) for a, b, x in zip(src, g.col, w)}
    assert all(d[(b, a)] == x for (a, b), x in d.items())
    # undirected: d(s, v) = d(v, s)
    D = [oracle.dijkstra(g.n, g.row_ptr, g.col, w, s) for s in (0, 3)]
    assert D[0][3] == D[1][0]
