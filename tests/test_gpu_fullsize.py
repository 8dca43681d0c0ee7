"""Full-size parity at BASELINE.json's configs, in the launch configuration bench.py times.

Expected values come from tests/golden/oracle_cache.npz, written by scripts/make_oracle_cache.py
which calls only oracle/ (literal Algorithm 2 per source) and graphgen/ (seeded inputs).

C1..C4: every distance row of the bench's dawn_sssp_batch step is reduced to its record
(ecc, reached, sum_dist, hash over every (v, d(v)) pair) and compared bit-exactly with the cached
oracle record, AND certified (SURVEY §8(c) four-invariant certificate, an exact proof that the
row is the BFS vector: Theorem 1 / Fact 1); a few rows are also compared element
by element with the FIFO-BFS oracle.  C3 additionally against its closed form (Manhattan
distance) for the whole 2^24-vertex vector.  C5: all S_wcc APSP records, including the final
partial batch, bit-exact against the cached oracle records.
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import graphgen
import oracle
import paper_2208_04514_b200 as dawn

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
UNR = oracle.UNREACHED
CACHE = os.path.join(os.path.dirname(__file__), "golden", "oracle_cache.npz")


def _cache():
    return np.load(CACHE)


def _fingerprint(g):
    return np.array([g.n, g.m, int(g.col.astype(np.int64).sum()),
                     int((g.row_ptr[1:] * np.arange(1, g.n + 1, dtype=np.int64)).sum() & 0x7FFFFFFFFFFFFFFF)],
                    dtype=np.int64)


def _rows_match_cache(g, srcs, D, key):
    """Every row: its record equals the cached oracle record and its certificate holds."""
    C = _cache()
    assert np.array_equal(C[f"{key}_fp"], _fingerprint(g)), "graphgen changed: re-run the cache"
    assert np.array_equal(C[f"{key}_sources"], np.asarray(srcs, np.int64))
    exp = C[f"{key}_records"]

    def one(i):
        rec, _ = oracle.record(g.n, g.row_ptr, int(srcs[i]), D[i])
        cert = oracle.certify(g.n, g.row_ptr, g.col, g.row_ptr, g.col, int(srcs[i]), D[i])
        return i, rec.tobytes() == exp[i].tobytes(), cert
    with ThreadPoolExecutor(max_workers=min(16, len(os.sched_getaffinity(0)))) as ex:
        res = list(ex.map(one, range(len(srcs))))
    bad = [(i, ok, cert) for i, ok, cert in res if not ok or cert != 0]
    assert not bad, bad[:5]


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
    # the bench step: one dawn_sssp_batch over the 64 sources; every row against the cached
    # oracle record and certified
    D = _batch(G, srcs)
    assert np.array_equal(D[0], oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(srcs[0]))[0])
    _rows_match_cache(g, srcs, D, "c2")


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
    # element by element against the oracle, ALL 64 against the cached oracle records and
    # certified
    D = _batch(G, srcs)
    for i in (0, 63):
        assert np.array_equal(D[i], oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(srcs[i]))[0]), i
    _rows_match_cache(g, srcs, D, "c4")


def test_c5_apsp_all_sources():
    g = graphgen.config_graph("C5")
    C = _cache()
    assert np.array_equal(C["c5_fp"], _fingerprint(g)), "graphgen changed: re-run the cache"
    G = _dev(g)
    verts, e_wcc = dawn.largest_wcc(G)                     # the device helper picks the set
    assert np.array_equal(verts, C["c5_verts"]) and e_wcc == int(C["c5_e_wcc"][0])
    rec = dawn.records_to_numpy(dawn.apsp(G, verts))
    exp = C["c5_records"]
    assert len(rec) == len(exp) == len(verts)
    assert len(verts) % dawn.MS_BATCH != 0                 # a partial final batch exists
    bad = np.nonzero(rec.view(np.uint8).reshape(len(rec), 32) !=
                     exp.view(np.uint8).reshape(len(exp), 32))[0]
    assert len(bad) == 0, ("records differ at", np.unique(bad)[:10])
    assert np.all(rec["reached"] == len(verts) - 1)        # E10/E11


def test_c5_apsp_sharded_matches():
    # the shard rule at W = 2, 3, 8 (simulated ranks on one GPU) reassembles the same records
    g = graphgen.config_graph("C5")
    C = _cache()
    G = _dev(g)
    verts = C["c5_verts"]
    exp = C["c5_records"]
    for W in (2, 3, 8):
        full = np.zeros(len(verts), dawn.REC_DTYPE)
        for r in range(W):
            idx = dawn.apsp_shard(len(verts), r, W)
            part = dawn.records_to_numpy(dawn.apsp(G, verts, r, W, gather=False))
            full[idx] = part
        assert full.tobytes() == exp.tobytes(), W


def test_c4_weighted_certificate():
    # NEXT-4 at full size: the bench's weighted searches on Kronecker-24 (weights 1..255, the
    # bench seed) certified exactly (weighted certificate, weights >= 1) for 2 bench sources
    g = graphgen.config_graph("C4")
    G = dawn.Graph(g.row_ptr, g.col, True)
    w = g.weights(seed=24, wmax=255)
    wt = torch.from_numpy(w.view(np.int32)).cuda()
    for s in g.sample_sources(2, seed=1):
        d = dawn.wsssp(G, int(s), wt).cpu().numpy().view(np.uint32).astype(np.uint64)
        d[d == 0xFFFFFFFF] = oracle.UNREACHED64
        rc, bad = oracle.certify_w(g.n, g.row_ptr, g.col, w, int(s), d)
        assert rc == 0, (int(s), rc, bad)


def test_c4_partitioned_matches_single_gpu_path():
    # NEXT-3 at full size: the fused partitioned search over 2 ranks (on one device) equals the
    # certified single-GPU rows of the bench sources
    g = graphgen.config_graph("C4")
    G = dawn.Graph(g.row_ptr, g.col, True)
    parts = [dawn.PartGraph(dawn.part_build(g.row_ptr, g.col, 2, r), 2, r) for r in range(2)]
    for s in g.sample_sources(3, seed=1):
        a = dawn.part_fused_local(parts, int(s))
        b = dawn.sssp(G, int(s))
        assert torch.equal(a, b), int(s)
    torch.cuda.synchronize()
