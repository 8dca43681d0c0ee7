"""Pins for the CPU oracle (oracle/oracle.c) against things other than itself.

Each pin cites the passage that fixes it.  A plausible bug in the oracle (dropped term, wrong
sign/index, transposed operand, off-by-one level) fails at least one of them:
  * golden records / distances from SURVEY §8(c) (independently computed) and SPEC examples
  * closed forms: grid (Manhattan), hypercube (popcount), directed cycle, path, star, complete
  * brute force: Floyd-Warshall, Theorem-1 first hit by matrix powers, explicit walk enumeration
  * the three paper algorithms (A1 BOVM, A2 SOVM, A3 FIFO BFS) agree on a >= 200 graph corpus
  * E10 accounting, iterations = eccentricity, layer contiguity, certificate fault injection.
"""
import itertools
import json
import os

import numpy as np
import pytest

import graphgen
import oracle

UNR = oracle.UNREACHED
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "records.json")))


def _fix(fx):
    return graphgen.from_edges(fx["n"], fx["edges"], symmetric=False)


# ------------------------------------------------------------------ golden
def test_splitmix64_first_output():
    assert oracle.hash_term(0, 0) == int(GOLD["splitmix64_0"]["value"], 16)


@pytest.mark.parametrize("fx", GOLD["fixtures"], ids=lambda f: f["name"])
def test_golden_records(fx):
    g = _fix(fx)
    cptr, cidx = g.transpose()
    for c in fx["cases"]:
        for fn, args in ((oracle.sovm, (g.row_ptr, g.col)), (oracle.bovm, (cptr, cidx)),
                         (oracle.bfs_fifo, (g.row_ptr, g.col))):
            d, _ = fn(g.n, *args, c["src"])
            assert d.tolist() == c["dist"], fn.__name__
        rec, er = oracle.record(g.n, g.row_ptr, c["src"], d)
        assert int(rec["ecc"]) == c["ecc"]
        assert int(rec["reached"]) == c["reached"]
        assert int(rec["sum_dist"]) == c["sum_dist"]
        assert er == c["edges_reach"]
        assert int(rec["hash"]) == int(c["hash"], 16)


def test_spec_iteration_examples():
    # path -> iterations 3; star from centre -> 1 iteration
    g = graphgen.from_edges(4, [[0, 1], [1, 2], [2, 3]])
    assert oracle.sovm(g.n, g.row_ptr, g.col, 0)[1]["iterations"] == 3
    cptr, cidx = g.transpose()
    assert oracle.bovm(g.n, cptr, cidx, 0)[1]["iterations"] == 3
    g = graphgen.from_edges(5, [[0, k] for k in range(1, 5)])
    st = oracle.sovm(g.n, g.row_ptr, g.col, 0)[1]
    assert st["iterations"] == 1 and st["rounds"] == 2


def test_apsp_3cycle_matrix():
    g = graphgen.from_edges(3, [[0, 1], [1, 2], [2, 0]])
    M = np.stack([oracle.sovm(3, g.row_ptr, g.col, s)[0] for s in range(3)])
    assert M.tolist() == GOLD["apsp_3cycle"]["matrix"]
    assert oracle.floyd_warshall(3, g.row_ptr, g.col).tolist() == GOLD["apsp_3cycle"]["matrix"]


def test_degenerate_graphs():
    g = graphgen.from_edges(1, np.zeros((0, 2)))
    assert oracle.sovm(1, g.row_ptr, g.col, 0)[0].tolist() == [0]
    g = graphgen.from_edges(2, np.zeros((0, 2)))
    assert oracle.sovm(2, g.row_ptr, g.col, 0)[0].tolist() == [0, UNR]
    assert oracle.sovm(2, g.row_ptr, g.col, 1)[0].tolist() == [UNR, 0]
    with pytest.raises(ValueError):
        oracle.sovm(2, g.row_ptr, g.col, 2)                  # bounds


# ------------------------------------------------------------------ closed forms
def test_grid_manhattan():
    W, H = 37, 23
    g = graphgen.grid(W, H)
    r, c = np.divmod(np.arange(W * H), W)
    for s in (0, W * H - 1, (H // 2) * W + W // 2, 5 * W + 30):
        d, st = oracle.sovm(g.n, g.row_ptr, g.col, s)
        r0, c0 = divmod(s, W)
        exp = np.abs(r - r0) + np.abs(c - c0)
        assert np.array_equal(d, exp.astype(np.uint32))
        assert st["iterations"] == exp.max()


@pytest.mark.parametrize("k", [1, 3, 6])
def test_hypercube_popcount(k):
    n = 1 << k
    edges = [[u, u ^ (1 << b)] for u in range(n) for b in range(k)]
    g = graphgen.from_edges(n, edges)
    pc = np.array([bin(v).count("1") for v in range(n)])
    for s in range(0, n, max(1, n // 7)):
        exp = np.array([bin(v ^ s).count("1") for v in range(n)], np.uint32)
        for d in (oracle.sovm(n, g.row_ptr, g.col, s)[0], oracle.bfs_fifo(n, g.row_ptr, g.col, s)[0],
                  oracle.bovm(n, g.row_ptr, g.col, s)[0]):
            assert np.array_equal(d, exp)
    assert pc.max() == k


def test_directed_cycle_path_star_complete():
    n = 11
    cyc = graphgen.from_edges(n, [[v, (v + 1) % n] for v in range(n)])
    for s in range(n):
        d = oracle.sovm(n, cyc.row_ptr, cyc.col, s)[0]
        assert d.tolist() == [(v - s) % n for v in range(n)]
    path = graphgen.from_edges(n, [[v, v + 1] for v in range(n - 1)])
    d, st = oracle.sovm(n, path.row_ptr, path.col, 0)
    assert d.tolist() == list(range(n)) and st["iterations"] == n - 1   # loop cap Q8
    d = oracle.sovm(n, path.row_ptr, path.col, 4)[0]
    assert d.tolist() == [UNR] * 4 + list(range(n - 4))
    comp = graphgen.from_edges(n, [[u, v] for u in range(n) for v in range(n) if u != v])
    for s in range(n):
        d = oracle.sovm(n, comp.row_ptr, comp.col, s)[0]
        assert d.tolist() == [0 if v == s else 1 for v in range(n)]


# ------------------------------------------------------------------ brute force
def _corpus():
    out = []
    for n in (8, 16, 33, 64, 128, 256):
        for p in (0.01, 0.05, 0.1, 0.3):
            for seed in range(9):
                out.append(graphgen.er_prob(n, p, seed * 1000 + n))
    return out


def test_three_algorithms_and_floyd_warshall_agree_on_corpus():
    # SPEC S:L450 acceptance: >= 200 ER digraphs, n in 8..256, p in {.01,.05,.1,.3}, all sources
    corpus = _corpus()
    assert len(corpus) >= 200
    for g in corpus:
        cptr, cidx = g.transpose()
        D = oracle.floyd_warshall(g.n, g.row_ptr, g.col)
        srcs = range(g.n) if g.n <= 64 else range(0, g.n, 7)
        for s in srcs:
            d1, st1 = oracle.sovm(g.n, g.row_ptr, g.col, s)
            d2, st2 = oracle.bovm(g.n, cptr, cidx, s)
            d3, st3 = oracle.bfs_fifo(g.n, g.row_ptr, g.col, s)
            assert np.array_equal(d1, D[s]), (g.name, s)
            assert np.array_equal(d2, D[s]), (g.name, s)
            assert np.array_equal(d3, D[s]), (g.name, s)
            fin = D[s] != UNR
            ecc = int(D[s][fin].max())
            # iterations = eccentricity for both DAWN variants
            assert st1["iterations"] == ecc and st2["iterations"] == ecc
            # E10: SOVM inspects exactly sum of out-degrees of reached vertices
            assert st1["edge_inspections"] == int(g.degrees()[fin].sum())
            assert st1["edge_inspections"] == st3["edge_inspections"]
            # layer contiguity
            assert set(D[s][fin].tolist()) == set(range(ecc + 1))


def _walks(n, adj, i, j, k):
    # explicit enumeration of length-k walks i -> j (Lemma 1 brute force)
    if k == 0:
        return 1 if i == j else 0
    return sum(_walks(n, adj, l, j, k - 1) for l in adj[i])


def test_theorem1_first_hit_and_lemma1_walk_counts():
    rng = np.random.default_rng(7)
    graphs = 0
    for trial in range(60):
        n = int(rng.integers(2, 13))
        g = graphgen.er_prob(n, float(rng.choice([0.1, 0.2, 0.35])), 500 + trial)
        D = oracle.first_hit(g.n, g.row_ptr, g.col)
        for s in range(n):
            assert np.array_equal(oracle.sovm(n, g.row_ptr, g.col, s)[0], D[s])
        if n <= 8:
            adj = [g.col[g.row_ptr[u]:g.row_ptr[u + 1]].tolist() for u in range(n)]
            for k in range(1, 5):
                _, C = oracle.first_hit(g.n, g.row_ptr, g.col, kq=k)
                for i, j in itertools.product(range(n), range(n)):
                    assert int(C[i, j]) == _walks(n, adj, i, j, k)
        graphs += 1
    assert graphs >= 50
    # directed 3-cycle, A^3 = identity pattern
    g = graphgen.from_edges(3, [[0, 1], [1, 2], [2, 0]])
    _, C = oracle.first_hit(3, g.row_ptr, g.col, kq=3)
    assert C.tolist() == np.eye(3, dtype=np.uint64).tolist()
    # undirected triangle, k=2 -> diagonal 2 (SPEC oracle example)
    t = graphgen.from_edges(3, [[0, 1], [1, 2], [2, 0]], symmetric=True)
    _, C = oracle.first_hit(3, t.row_ptr, t.col, kq=2)
    assert np.diag(C).tolist() == [2, 2, 2]


# ------------------------------------------------------------------ certificate
def test_certificate_accepts_truth_and_rejects_every_single_perturbation():
    rng = np.random.default_rng(3)
    checked = rejected = 0
    for trial in range(40):
        n = int(rng.integers(2, 15))
        g = graphgen.er_prob(n, float(rng.choice([0.1, 0.25, 0.4])), 900 + trial)
        cptr, cidx = g.transpose()
        for s in range(n):
            d = oracle.bfs_fifo(n, g.row_ptr, g.col, s)[0]
            assert oracle.certify(n, g.row_ptr, g.col, cptr, cidx, s, d) == 0
            checked += 1
            for v in range(n):
                for delta in (-1, 1, "unr", "zero"):
                    e = d.copy()
                    if delta == "unr":
                        e[v] = UNR
                    elif delta == "zero":
                        e[v] = 0
                    elif d[v] == UNR:
                        e[v] = n + 3
                    else:
                        e[v] = np.uint32((int(d[v]) + delta) % (1 << 32))
                    if np.array_equal(e, d):
                        continue
                    res = oracle.certify(n, g.row_ptr, g.col, cptr, cidx, s, e)
                    assert res != 0, (g.name, s, v, delta)
                    rejected += 1
    assert checked > 100 and rejected > 1000


def test_certificate_names_the_corrupted_vertex():
    g = graphgen.grid(9, 9)
    d = oracle.sovm(g.n, g.row_ptr, g.col, 0)[0]
    e = d.copy()
    e[40] += 2
    rc = oracle.certify(g.n, g.row_ptr, g.col, g.row_ptr, g.col, 0, e)
    assert rc != 0 and rc[1] in (40, 31, 39, 41, 49)   # the vertex or the neighbour it breaks


# ------------------------------------------------------------------ records / WCC / threads
def test_records_thread_count_independent_and_match_single_source():
    g = graphgen.kron(10, 8, 3)
    srcs = g.sample_sources(40, seed=5)
    base = oracle.records(g.n, g.row_ptr, g.col, srcs, threads=1)
    for t in (2, 4, 8):
        assert oracle.records(g.n, g.row_ptr, g.col, srcs, threads=t).tobytes() == base.tobytes()
    for i, s in enumerate(srcs[:10]):
        d = oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(s))[0]
        rec, _ = oracle.record(g.n, g.row_ptr, int(s), d)
        assert rec.tobytes() == base[i].tobytes()


def test_e10_in_largest_wcc_of_symmetric_graph():
    # PAPER E10/E11 (L299-307): every source of the largest WCC of a symmetric graph reaches
    # S_wcc - 1 others and inspects E_wcc arcs.
    g = graphgen.kron(11, 16, 11)
    verts, e_wcc = g.largest_wcc()
    for s in verts[:: max(1, len(verts) // 12)]:
        d, st = oracle.sovm(g.n, g.row_ptr, g.col, int(s))
        assert int((d != UNR).sum()) == len(verts)
        assert st["edge_inspections"] == e_wcc


def test_wcc_spec_example():
    # two directed paths 0->1->2 and 3->4 -> s_wcc = 3, e_wcc = 2
    g = graphgen.from_edges(5, [[0, 1], [1, 2], [3, 4]])
    v, e = g.largest_wcc()
    assert v.tolist() == [0, 1, 2] and e == 2


# ------------------------------------------------------------------ largest WCC (Table 1, Q15)
def _fw_components(g):
    """Weak components by brute force: Floyd-Warshall reachability on the symmetrised graph."""
    edges = [(u, int(v)) for u in range(g.n) for v in g.col[g.row_ptr[u]:g.row_ptr[u + 1]]]
    sym = graphgen.from_edges(g.n, edges + [(v, u) for u, v in edges], symmetric=False)
    D = oracle.floyd_warshall(sym.n, sym.row_ptr, sym.col)
    comps = {tuple(np.nonzero(D[v] != UNR)[0].tolist()) for v in range(g.n)}
    return [list(c) for c in comps]


def test_largest_wcc_hand_fixtures():
    # PAPER Table 1 (L95-98): S_wcc / E_wcc; reading Q15: most nodes, then most arcs, then the
    # smaller minimum id.  SPEC S:L98-101 example first.
    cases = [
        (5, [[0, 1], [1, 2], [3, 4]], [0, 1, 2], 2),
        (6, [[0, 1], [1, 2], [3, 4], [4, 5], [5, 3]], [3, 4, 5], 3),   # tie on nodes -> arcs
        (4, [[0, 1], [2, 3]], [0, 1], 1),                               # full tie -> min id 0
        (6, [[5, 0], [1, 2]], [0, 5], 1),                               # min id of {0,5} wins
        (6, [[1, 0], [2, 0], [4, 3]], [0, 1, 2], 2),                    # weak: no directed path 1~>2
        (5, [], [0], 0),                                                # all isolated
        (1, [], [0], 0),
    ]
    for n, edges, exp_v, exp_e in cases:
        g = graphgen.from_edges(n, edges, symmetric=False)
        v, e = oracle.largest_wcc(g.n, g.row_ptr, g.col)
        assert v.tolist() == exp_v and e == exp_e, (n, edges, v, e)


def test_largest_wcc_brute_force_corpus():
    # every ER digraph of the corpus: the oracle's component equals the one chosen from the
    # Floyd-Warshall components by the Q15 rule, with E_wcc = its out-degree sum
    rng = np.random.default_rng(2208)
    for t in range(60):
        n = int(rng.integers(1, 40))
        p = float(rng.choice([0.0, 0.02, 0.05, 0.1, 0.3]))
        g = graphgen.er_prob(n, p, 1000 + t)
        deg = np.diff(g.row_ptr)
        best = None
        for c in _fw_components(g):
            key = (len(c), int(deg[c].sum()), -min(c))
            if best is None or key > best[0]:
                best = (key, sorted(c))
        v, e = oracle.largest_wcc(g.n, g.row_ptr, g.col)
        assert v.tolist() == best[1] and e == best[0][1], (t, n, p)


def test_largest_wcc_e10_identity():
    # PAPER E10/E11 (L299-307): on a symmetric graph every source of the component reaches
    # S_wcc - 1 others and its E10 count equals E_wcc (FIFO BFS, Algorithm 3, independent)
    g = graphgen.kron(12, 16, 12)
    v, e = oracle.largest_wcc(g.n, g.row_ptr, g.col)
    for s in v[:: max(1, len(v) // 8)]:
        d, _ = oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(s))
        rec, er = oracle.record(g.n, g.row_ptr, int(s), d)
        assert int(rec["reached"]) == len(v) - 1 and er == e
        assert np.array_equal(np.nonzero(d != UNR)[0], v)
