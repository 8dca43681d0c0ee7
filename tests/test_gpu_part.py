"""GPU parity of the partitioned single-source path:
W vertex-range partitions, each holding only the arcs into its range, one frontier-slice
all-gather per level.  Here the W ranks run on ONE device and the all-gather is a device copy
(part_sssp_local: the same kernels and exchange layout as part_sssp under torch.distributed);
tests/test_gpu_nccl.py drives the torch.distributed path.  Bar: distances bit-exact vs the
oracle, statistics equal to the oracle record (E10 counts)."""
import numpy as np
import pytest
import torch

import graphgen
import oracle
import paper_2208_04514_b200 as dawn

pytestmark = pytest.mark.gpu
UNR = oracle.UNREACHED
VARIANTS = ("auto", "push", "pull")


def _parts(g, W):
    return [dawn.PartGraph(dawn.part_build(g.row_ptr, g.col, W, r), W, r) for r in range(W)]


def _check(g, parts, sources, variants=VARIANTS):
    for s in sources:
        exp, _ = oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(s))
        rec, er = oracle.record(g.n, g.row_ptr, int(s), exp)
        for v in variants:
            d, sts = dawn.part_sssp_local(parts, int(s), v, stats=True)
            d = d.cpu().numpy().view(np.uint32)
            bad = np.nonzero(d != exp)[0]
            assert len(bad) == 0, (g.name, len(parts), s, v, bad[:5], d[bad[:5]], exp[bad[:5]])
            for st in sts:  # the global statistics are identical on every rank
                x = dawn.stats_to_dict(st)
                assert x["levels"] == int(rec["ecc"]), (s, v, x)
                assert x["reached"] == int(rec["reached"]), (s, v, x)
                assert x["edges_reach"] == er, (s, v, x, er)


@pytest.mark.parametrize("W", [1, 2, 3, 4])
def test_kron_partitions(W):
    g = graphgen.kron(12, 16, 12)
    _check(g, _parts(g, W), g.sample_sources(4, seed=W))


@pytest.mark.parametrize("W", [1, 3])
def test_directed_er_partitions(W):
    # directed: pull uses the in-rows the builder derives (no CSC needed from the caller)
    g = graphgen.er(1000, 8000, 1)
    _check(g, _parts(g, W), [0, 5, 999])


def test_hubs_and_pieces():
    # rows far above the 32-arc light limit in both groupings (star hubs + random arcs)
    rng = np.random.default_rng(3)
    n = 5000
    e = [(0, v) for v in range(1, n)] + [(v, 0) for v in range(1, n)]
    e += [(int(a), int(b)) for a, b in rng.integers(0, n, size=(20000, 2)) if a != b]
    e += [(7, v) for v in range(100, 1500)]
    g = graphgen.from_edges(n, e)
    for W in (2, 5):
        _check(g, _parts(g, W), [0, 7, 123, n - 1])


def test_deep_path_direct_levels():
    # eps = n - 1 = 599 > 255: levels >= 255 store distances directly (the deferred byte's
    # escape), the level loop runs to the n - 1 bound
    n = 600
    g = graphgen.from_edges(n, [(i, i + 1) for i in range(n - 1)])
    _check(g, _parts(g, 3), [0, 17], variants=("auto", "push"))


def test_edge_cases():
    # empty ranks (n = 40 over 4 ranks: blocks of 32), isolated and last-vertex sources, n = 1
    g = graphgen.from_edges(40, [(i, (i * 7 + 3) % 40) for i in range(40)] + [(3, 4), (4, 3)])
    parts = _parts(g, 4)
    assert [p.R for p in parts] == [32, 8, 0, 0]
    _check(g, parts, [0, 39, 3])
    g1 = graphgen.from_edges(1, [])
    d = dawn.part_sssp_local(_parts(g1, 2), 0)
    assert d.cpu().numpy().view(np.uint32).tolist() == [0]
    g2 = graphgen.from_edges(70, [(1, 2)])
    _check(g2, _parts(g2, 2), [5, 1, 69])  # an isolated source reaches nothing
    with pytest.raises(dawn.DawnError) as ei:
        dawn.part_sssp_local(parts, 40)
    assert ei.value.status == 2


def test_matches_single_gpu_path_c2_sampled():
    # Kronecker-20 (C2) over 2 partitions vs the single-GPU kernel on the same sources
    g = graphgen.config_graph("C2")
    G = dawn.Graph(g.row_ptr, g.col, True)
    parts = _parts(g, 2)
    for s in g.sample_sources(3, seed=9):
        a = dawn.part_sssp_local(parts, int(s))
        b = dawn.sssp(G, int(s))
        assert torch.equal(a, b), s
    torch.cuda.synchronize()


# ---- fused exchange: the whole search in one persistent kernel per rank, slices written into
# ---- every rank's receive buffer, system-scope arrival counters (no host work per level)
def _check_fused(g, parts, sources, variants=VARIANTS):
    for s in sources:
        exp, _ = oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(s))
        rec, er = oracle.record(g.n, g.row_ptr, int(s), exp)
        for v in variants:
            d, sts = dawn.part_fused_local(parts, int(s), v, stats=True)
            torch.cuda.synchronize()
            d = d.cpu().numpy().view(np.uint32)
            bad = np.nonzero(d != exp)[0]
            assert len(bad) == 0, (g.name, len(parts), s, v, bad[:5], d[bad[:5]], exp[bad[:5]])
            for st in sts:
                x = dawn.stats_to_dict(st)
                assert x["levels"] == int(rec["ecc"]) and x["reached"] == int(rec["reached"])
                assert x["edges_reach"] == er, (s, v, x, er)


@pytest.mark.parametrize("W", [1, 2, 3, 4])
def test_fused_kron(W):
    g = graphgen.kron(12, 16, 12)
    _check_fused(g, _parts(g, W), g.sample_sources(4, seed=W))  # 12 searches on one set of
                                                                # counters (monotonic across)


def test_fused_directed_hubs_deep_edges():
    g = graphgen.er(1000, 8000, 1)
    _check_fused(g, _parts(g, 3), [0, 999])
    rng = np.random.default_rng(3)
    n = 5000
    e = [(0, v) for v in range(1, n)] + [(v, 0) for v in range(1, n)]
    e += [(int(a), int(b)) for a, b in rng.integers(0, n, size=(20000, 2)) if a != b]
    h = graphgen.from_edges(n, e)
    _check_fused(h, _parts(h, 2), [0, 123])
    p = graphgen.from_edges(600, [(i, i + 1) for i in range(599)])  # 599 levels, 255+ direct
    _check_fused(p, _parts(p, 3), [0], variants=("auto", "push"))
    g40 = graphgen.from_edges(40, [(i, (i * 7 + 3) % 40) for i in range(40)] + [(3, 4), (4, 3)])
    _check_fused(g40, _parts(g40, 4), [0, 39])  # two ranks own nothing
    g1 = graphgen.from_edges(1, [])
    assert dawn.part_fused_local(_parts(g1, 2), 0).cpu().numpy().view(np.uint32).tolist() == [0]


def test_fused_c2_matches_single_gpu():
    g = graphgen.config_graph("C2")
    G = dawn.Graph(g.row_ptr, g.col, True)
    parts = _parts(g, 2)
    for s in g.sample_sources(3, seed=9):
        a = dawn.part_fused_local(parts, int(s))
        assert torch.equal(a, dawn.sssp(G, int(s))), s
    torch.cuda.synchronize()


def _light_in_heavy_out_graph(seed: int):
    """0 -> 2,000 A -> 20,000 B (20 arcs per A) -> 100 C (one arc per B), plus H with ONE in-arc
    (from B[0]) and 1,000 out-arcs to D vertices nothing else reaches.  The growing levels pull,
    so H (a light in-row) is settled by the light pull pass; the next level (frontier C + H,
    shrinking, 101 * beta < n) pushes, and only H's heavy out-row reaches D."""
    rng = np.random.default_rng(seed)
    A, B, C = np.arange(1, 2001), np.arange(2001, 22001), np.arange(22001, 22101)
    H, D0 = 22101, 22102
    e = [[0, int(a)] for a in A]
    e += [[int(a), int(b)] for a in A for b in rng.choice(B, 20, replace=False)]
    e += [[int(b), int(rng.choice(C))] for b in B]
    e += [[int(B[0]), H]] + [[H, D0 + j] for j in range(1000)]
    e += [[int(c), D0 + 1000 + i] for i, c in enumerate(C)]
    return graphgen.from_edges(D0 + 1000 + len(C), e)


@pytest.mark.parametrize("W", [1, 2, 3])
def test_push_after_pull_reaches_heavy_out_rows(W):
    # a vertex settled by the pull pass whose out-row is heavy must make the next push level
    # test the heavy pieces (slice-header flag); per-level and fused paths, against the oracle
    g = _light_in_heavy_out_graph(W)
    parts = _parts(g, W)
    exp = oracle.bfs_fifo(g.n, g.row_ptr, g.col, 0)[0]
    assert exp[22102] == 4 and exp[22101] == 3
    d, sts = dawn.part_sssp_local(parts, 0, "auto", stats=True)
    assert np.array_equal(d.cpu().numpy().view(np.uint32), exp)
    x = dawn.stats_to_dict(sts[0])
    assert x["pull_levels"] >= 1 and x["push_levels"] >= 2, x   # the pull -> push schedule
    assert np.array_equal(dawn.part_fused_local(parts, 0).cpu().numpy().view(np.uint32), exp)
