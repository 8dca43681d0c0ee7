"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bar (BASELINE.json north_star): bit-exact distances, tolerance 0; records bit-exact.
Every test here runs on a B200 via gpurun (marker `gpu`).
"""
import numpy as np
import pytest
import torch

import graphgen
import oracle
import paper_2208_04514_b200 as dawn

pytestmark = pytest.mark.gpu
UNR = oracle.UNREACHED
VARIANTS = ("auto", "push", "pull")


def dev_graph(g: graphgen.Graph, csc: bool = True):
    if g.symmetric:
        return dawn.Graph(g.row_ptr, g.col, True, validate=True)
    if csc:
        p, i = g.transpose()
        return dawn.Graph(g.row_ptr, g.col, False, p, i, validate=True)
    return dawn.Graph(g.row_ptr, g.col, False, validate=True)


def gpu_dist(G, s, variant="auto", stats=False):
    r = dawn.sssp(G, s, variant, stats=stats)
    if stats:
        d, st = r
        return d.cpu().numpy().view(np.uint32), dawn.stats_to_dict(st)
    return r.cpu().numpy().view(np.uint32)


def check_sssp(g, G, sources, variants=VARIANTS, oracle_fn="bfs_fifo"):
    for s in sources:
        s = int(s)
        exp, ost = getattr(oracle, oracle_fn)(g.n, g.row_ptr, g.col, s)
        rec, er = oracle.record(g.n, g.row_ptr, s, exp)
        for v in variants:
            d, st = gpu_dist(G, s, v, stats=True)
            bad = np.nonzero(d != exp)[0]
            assert len(bad) == 0, (g.name, s, v, bad[:5], d[bad[:5]], exp[bad[:5]])
            assert st["levels"] == int(rec["ecc"]), (g.name, s, v, st)
            assert st["reached"] == int(rec["reached"]), (g.name, s, v, st)
            assert st["edges_reach"] == er, (g.name, s, v, st, er)
            assert st["push_levels"] + st["pull_levels"] >= st["levels"]


# ------------------------------------------------------------------ hand fixtures / corpus
def test_golden_fixtures_all_variants():
    import json, os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "records.json")))
    for fx in gold["fixtures"]:
        g = graphgen.from_edges(fx["n"], fx["edges"])
        G = dev_graph(g)
        for c in fx["cases"]:
            for v in VARIANTS:
                assert gpu_dist(G, c["src"], v).tolist() == c["dist"], (fx["name"], v)
        srcs = [c["src"] for c in fx["cases"]]
        d, r = dawn.msssp(G, srcs)
        recs = dawn.records_to_numpy(r)
        for i, c in enumerate(fx["cases"]):
            assert d[i].cpu().numpy().view(np.uint32).tolist() == c["dist"]
            assert int(recs[i]["ecc"]) == c["ecc"] and int(recs[i]["reached"]) == c["reached"]
            assert int(recs[i]["sum_dist"]) == c["sum_dist"]
            assert int(recs[i]["hash"]) == int(c["hash"], 16)


def test_er_corpus_all_sources_all_variants():
    for n in (8, 33, 100, 256):
        for p in (0.01, 0.05, 0.1, 0.3):
            g = graphgen.er_prob(n, p, 77 + n)
            G = dev_graph(g)
            check_sssp(g, G, range(0, n, max(1, n // 16)))


def test_directed_without_csc_is_push_only():
    g = graphgen.er_prob(64, 0.05, 5)
    G = dev_graph(g, csc=False)
    check_sssp(g, G, range(0, 64, 9), variants=("auto", "push"))
    with pytest.raises(dawn.DawnError) as e:
        dawn.sssp(G, 0, "pull")
    assert e.value.status == 3


def test_closed_forms_grid_hypercube_cycle_path():
    W, H = 300, 170
    g = graphgen.grid(W, H)
    G = dev_graph(g)
    r, c = np.divmod(np.arange(W * H), W)
    for s in (0, W * H - 1, (H // 2) * W + W // 2):
        r0, c0 = divmod(s, W)
        exp = (np.abs(r - r0) + np.abs(c - c0)).astype(np.uint32)
        for v in VARIANTS:
            assert np.array_equal(gpu_dist(G, s, v), exp), (s, v)
    k = 12
    n = 1 << k
    hc = graphgen.from_edges(n, [[u, u ^ (1 << b)] for u in range(n) for b in range(k)])
    Gh = dev_graph(hc)
    for s in (0, 1234, n - 1):
        exp = np.array([bin(v ^ s).count("1") for v in range(n)], np.uint32)
        for v in VARIANTS:
            assert np.array_equal(gpu_dist(Gh, s, v), exp)
    n = 5000
    cyc = graphgen.from_edges(n, [[v, (v + 1) % n] for v in range(n)])
    Gc = dev_graph(cyc)
    for v in VARIANTS:
        d = gpu_dist(Gc, 17, v)
        assert np.array_equal(d, ((np.arange(n) - 17) % n).astype(np.uint32))
    # path: eps = n - 1 hits the loop cap exactly (reading Q8)
    pth = graphgen.from_edges(n, [[v, v + 1] for v in range(n - 1)])
    Gp = dev_graph(pth)
    for v in VARIANTS:
        assert np.array_equal(gpu_dist(Gp, 0, v), np.arange(n, dtype=np.uint32))


def test_edge_cases():
    g1 = graphgen.from_edges(1, np.zeros((0, 2)))
    G1 = dev_graph(g1)
    for v in VARIANTS:
        assert gpu_dist(G1, 0, v).tolist() == [0]
    g2 = graphgen.from_edges(2, np.zeros((0, 2)))
    G2 = dev_graph(g2)
    assert gpu_dist(G2, 1).tolist() == [UNR, 0]          # s = n-1 valid
    with pytest.raises(dawn.DawnError) as e:
        dawn.sssp(G2, 2)                                   # s = n -> BOUNDS
    assert e.value.status == 2
    with pytest.raises(dawn.DawnError) as e:
        dawn.msssp(G2, [0, 5])
    assert e.value.status == 2
    # star: leaf source (degree 0) and hub source
    star = graphgen.from_edges(300, [[0, k] for k in range(1, 300)])
    Gs = dev_graph(star)
    check_sssp(star, Gs, [0, 1, 299])


def test_hub_rows_and_repeated_sources():
    # a hub with 70K out-arcs (> 64K, SURVEY §8(c) edge cases) inside a sparse graph
    n = 80000
    edges = [[0, v] for v in range(1, 70001)] + [[v, v + 1] for v in range(70000, n - 1)]
    g = graphgen.from_edges(n, edges, symmetric=True)
    G = dev_graph(g)
    check_sssp(g, G, [0, 5, 79999])
    d, r = dawn.msssp(G, [5, 5, 0, 5])
    recs = dawn.records_to_numpy(r)
    assert recs[0].tobytes() == recs[1].tobytes() == recs[3].tobytes()
    assert torch.equal(d[0], d[1]) and torch.equal(d[0], d[3])


@pytest.mark.parametrize("scale", [10, 14, 16])
def test_kron_sampled_sources(scale):
    g = graphgen.kron(scale, 16)
    G = dev_graph(g)
    srcs = list(g.sample_sources(6, seed=scale)) + [int(np.argmax(g.degrees()))]
    check_sssp(g, G, srcs)
    # isolated source
    iso = np.nonzero(g.degrees() == 0)[0]
    if len(iso):
        check_sssp(g, G, [int(iso[0])])


def test_config_c1_er_1000_8000():
    g = graphgen.config_graph("C1")
    G = dev_graph(g)
    check_sssp(g, G, [0], oracle_fn="sovm")
    check_sssp(g, G, range(1, 1000, 37))


# ------------------------------------------------------------------ multi-source / APSP
def _check_records(g, srcs, recs):
    exp = oracle.records(g.n, g.row_ptr, g.col, srcs)
    for i in range(len(srcs)):
        assert recs[i].tobytes() == exp[i].tobytes(), (i, srcs[i], recs[i], exp[i])


@pytest.mark.parametrize("k", [1, 63, 64, 70, 130])
def test_msssp_dist_and_records(k):
    g = graphgen.kron(13, 16)
    G = dev_graph(g)
    srcs = np.concatenate([g.sample_sources(k - 1, seed=k), [int(np.argmin(g.degrees()))]])
    d, r = dawn.msssp(G, srcs)
    D = d.cpu().numpy().view(np.uint32)
    for i in range(0, k, max(1, k // 9)):
        exp = oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(srcs[i]))[0]
        assert np.array_equal(D[i], exp), i
    _check_records(g, srcs, dawn.records_to_numpy(r))


def test_msssp_directed_er():
    g = graphgen.config_graph("C1")
    G = dev_graph(g)
    srcs = np.arange(0, 1000, 7)
    d, r = dawn.msssp(G, srcs)
    D = d.cpu().numpy().view(np.uint32)
    for i, s in enumerate(srcs):
        assert np.array_equal(D[i], oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(s))[0])
    _check_records(g, srcs, dawn.records_to_numpy(r))


def test_apsp_shards_cover_and_match():
    g = graphgen.kron(12, 16)
    G = dev_graph(g)
    verts, e_wcc = g.largest_wcc()
    full = dawn.records_to_numpy(dawn.apsp(G, verts))
    _check_records(g, verts, full)
    # E10/E11 property on every source of the largest WCC of a symmetric graph
    assert np.all(full["reached"] == len(verts) - 1)
    for world in (2, 3, 8):
        parts = [dawn.records_to_numpy(dawn.apsp(G, verts, rank=r, world=world, gather=False))
                 for r in range(world)]
        re = np.empty(len(verts), full.dtype)
        for r in range(world):
            re[dawn.apsp_shard(len(verts), r, world)] = parts[r]
        assert re.tobytes() == full.tobytes()


def test_determinism():
    g = graphgen.kron(15, 16)
    G = dev_graph(g)
    s = int(g.sample_sources(1, 3)[0])
    a = [gpu_dist(G, s, v) for v in VARIANTS]
    for _ in range(3):
        for i, v in enumerate(VARIANTS):
            assert np.array_equal(gpu_dist(G, s, v), a[i])
    d1, r1 = dawn.msssp(G, g.sample_sources(100, 4))
    d2, r2 = dawn.msssp(G, g.sample_sources(100, 4))
    assert torch.equal(d1, d2) and torch.equal(r1, r2)


def test_trace_levels_consistent():
    g = graphgen.kron(14, 16)
    G = dawn.Graph(g.row_ptr, g.col, True, trace=True)
    s = int(g.sample_sources(1, 9)[0])
    for v in VARIANTS:
        d, st = gpu_dist(G, s, v, stats=True)
        tr = G.trace()
        assert len(tr) == st["levels"] + 2 or len(tr) == st["levels"] + 1
        assert tr["nf"][0] == 1 and np.all(np.diff(tr["t_ns"].astype(np.int64)) >= 0)
        fin = d != UNR
        counts = np.bincount(d[fin], minlength=len(tr))
        assert np.array_equal(tr["nf"][: st["levels"] + 1], counts[: st["levels"] + 1])
        assert tr["dir"][-1] == 2


@pytest.mark.parametrize("knobs", [dict(bitmap_push_edges=64), dict(bitmap_push_edges=0, solo_edges=0),
                                   dict(solo_edges=100000, alpha=1000), dict(alpha=0, beta=1e9),
                                   dict(bitmap_push_grow_edges=0, solo_edges=0),
                                   dict(bitmap_push_grow_edges=2 ** 31, bitmap_push_edges=2 ** 31)])
def test_tunables_never_change_results(knobs):
    # every schedule knob (bitmap push on every level, no solo levels, long solo stretches,
    # never/always pull) must give the oracle's distances (tolerance 0)
    for g in (graphgen.kron(13, 16), graphgen.er_prob(3000, 0.002, 4), graphgen.grid(200, 150)):
        G = dev_graph(g)
        G.set_tuning(**knobs)
        srcs = [0, g.n - 1] + list(g.sample_sources(3, seed=2))
        check_sssp(g, G, srcs, variants=("auto", "push"))


def test_unreachable_long_heavy_row():
    # a hub with a 10,000-entry in-row outside the source's component stays unsettled at every
    # pull level (listed for the heavy phase each time), and a reachable 9,000-entry hub settles;
    # all variants, single and batch
    k = graphgen.kron(14, 16, 14)
    n0 = k.n
    e = np.stack([np.repeat(np.arange(k.n), np.diff(k.row_ptr)), k.col.astype(np.int64)], 1).tolist()
    hub = n0
    e += [[hub, n0 + 1 + i] for i in range(10000)] + [[n0 + 1 + i, hub] for i in range(10000)]
    hub2 = n0 + 10001                      # a long hub inside the source's component
    e += [[hub2, int(v)] for v in range(9000)] + [[int(v), hub2] for v in range(9000)]
    g = graphgen.from_edges(n0 + 10002, e)
    G = dev_graph(g)
    srcs = [0, 5, hub2] + list(k.sample_sources(2, seed=4))
    check_sssp(g, G, srcs, variants=("auto", "push", "pull"))
    d = dawn.sssp_batch(G, torch.tensor(srcs, dtype=torch.int32, device="cuda")).cpu().numpy().view(np.uint32)
    for i, s0 in enumerate(srcs):
        assert np.array_equal(d[i], oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(s0))[0]), s0


def test_narrow_kernel_and_handover():
    # dawn_sssp starts on one 16-CTA cluster (k_narrow); wide frontiers (or full queues) hand
    # over to the grid-wide kernel, which resumes from the frontier bitmap.
    rng = np.random.default_rng(11)
    n = 200_000
    e = rng.integers(0, n, size=(2 * n, 2))
    rand = graphgen.from_edges(n, e, symmetric=True)              # avg degree ~4, wide waves
    tree = graphgen.from_edges(2 ** 17 - 1, [[v, 2 * v + 1] for v in range(2 ** 16 - 1)] +
                               [[v, 2 * v + 2] for v in range(2 ** 16 - 1)])  # directed tree
    grid = graphgen.grid(700, 500)
    kr = graphgen.kron(14, 16, 14)                                # hubs: CTA-wide long rows
    for g in (rand, tree, grid, kr):
        G = dev_graph(g)
        srcs = [0, 1, g.n // 2, g.n - 1]
        check_sssp(g, G, srcs, variants=("auto", "push"))         # load-time defaults
        for h in (0, 64, 1024, 2e19):                              # hand over at every width
            G.set_tuning(cluster_start=1, cluster_handover_edges=h)
            check_sssp(g, G, srcs[:2], variants=("auto", "push"))
        G.set_tuning(cluster_start=0)                              # grid-wide kernel only
        check_sssp(g, G, srcs[:2], variants=("auto",))


def test_narrow_forced_handover():
    # tiny shared-memory queues (DAWN_PARAM_NARROW_QUEUE_CAP) make every wide-enough level
    # overflow: hand-over to k_sssp from the frontier bitmap at many different levels
    rng = np.random.default_rng(12)
    n = 50_000
    rand = graphgen.from_edges(n, rng.integers(0, n, size=(n, 2)), symmetric=True)
    dirg = graphgen.from_edges(n, rng.integers(0, n, size=(3 * n, 2)))
    for g in (graphgen.grid(300, 200), rand, dirg):
        G = dev_graph(g)
        G.set_tuning(cluster_start=1, cluster_handover_edges=2e19,  # only overflow hands over
                     narrow_queue_cap=40)
        srcs = [0, g.n // 3, g.n - 1] + list(g.sample_sources(3, seed=3))
        check_sssp(g, G, srcs, variants=("auto", "push"))


def test_cuda_graph_replay():
    # dawn_sssp calls captured in a CUDA graph and replayed must give the same distances on
    # every replay (no host-side per-call state baked into the captured launches): a grid
    # (k_narrow + k_sssp), a Kronecker graph (k_sssp) and a tiny ER graph (k_small)
    cases = [graphgen.grid(300, 200), graphgen.kron(12, 16, 12), graphgen.er(1000, 8000, 1)]
    for g in cases:
        G = dev_graph(g)
        srcs = [0, g.n // 2, g.n - 1]
        outs = [torch.empty(g.n, dtype=torch.int32, device="cuda") for _ in srcs]
        for s, o in zip(srcs, outs):
            dawn.sssp(G, s, "auto", out=o)
        torch.cuda.synchronize()
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=cap):
            for s, o in zip(srcs, outs):
                dawn.sssp(G, s, "auto", out=o)
        exp = [oracle.bfs_fifo(g.n, g.row_ptr, g.col, s)[0] for s in srcs]
        for rep in range(3):
            for o in outs:
                o.fill_(7)
            graph.replay()
            torch.cuda.synchronize()
            for s, o, e in zip(srcs, outs, exp):
                d = o.cpu().numpy().view(np.uint32)
                assert np.array_equal(d, e), (g.name, s, rep)


def test_narrow_directed_mesh():
    # a directed mesh (right and down arcs only, ids follow space): owner-computes cluster search
    # on a graph without in-edge symmetry; sources inside the mesh reach only their lower-right
    # quadrant, the rest must stay UNREACHED
    W, H = 300, 200
    e = [[r * W + c, r * W + c + 1] for r in range(H) for c in range(W - 1)]
    e += [[r * W + c, (r + 1) * W + c] for r in range(H - 1) for c in range(W)]
    g = graphgen.from_edges(W * H, e)
    G = dev_graph(g)
    srcs = [0, W * H // 2 + W // 3, W * H - 1, W - 1]
    check_sssp(g, G, srcs, variants=("auto", "push"))
    G.set_tuning(cluster_start=1, cluster_handover_edges=2e19)
    check_sssp(g, G, srcs, variants=("auto",))


def test_sssp_batch_matches_single_calls():
    # dawn_sssp_batch (k searches in one launch, device source list) == k dawn_sssp calls ==
    # the oracle; tiny, mesh, Kronecker and directed graphs; repeated sources allowed
    rng = np.random.default_rng(21)
    dirg = graphgen.from_edges(20_000, rng.integers(0, 20_000, size=(80_000, 2)))
    for g in (graphgen.er(1000, 8000, 1), graphgen.grid(120, 90), graphgen.kron(13, 16, 13), dirg):
        G = dev_graph(g)
        srcs = np.array([0, g.n - 1, 0] + list(g.sample_sources(5, seed=4)), dtype=np.int32)
        dsrc = torch.from_numpy(srcs).cuda()
        for v in ("auto", "push"):
            d, st = dawn.sssp_batch(G, dsrc, v, stats=True)
            d = d.cpu().numpy().view(np.uint32)
            for i, s in enumerate(srcs):
                exp = oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(s))[0]
                assert np.array_equal(d[i], exp), (g.name, v, int(s))
                rec, er = oracle.record(g.n, g.row_ptr, int(s), exp)
                sd = dawn.stats_to_dict(st[i])
                assert sd["levels"] == int(rec["ecc"]) and sd["edges_reach"] == er, (g.name, v, sd)



def test_sssp_batch_paths():
    # the three dawn_sssp_batch paths against the oracle: k_small with more searches than CTAs
    # (each CTA strides over the batch), cluster start (k_narrow + k_sssp per search, with and
    # without forced hand-over) and the grid-wide kernel forced on the same mesh; k == 0
    small = graphgen.er(1000, 8000, 5)
    G = dev_graph(small)
    srcs = np.arange(0, 1000, 3, dtype=np.int32)                   # 334 > #SMs
    d = dawn.sssp_batch(G, torch.from_numpy(srcs).cuda()).cpu().numpy().view(np.uint32)
    for i in range(0, len(srcs), 37):
        assert np.array_equal(d[i], oracle.bfs_fifo(small.n, small.row_ptr, small.col,
                                                     int(srcs[i]))[0]), int(srcs[i])
    assert dawn.sssp_batch(G, torch.empty(0, dtype=torch.int32, device="cuda")).shape == (0, 1000)
    mesh = graphgen.grid(700, 500)
    G = dev_graph(mesh)
    srcs = np.array([0, mesh.n - 1, 12345, 0], dtype=np.int32)
    exp = [oracle.bfs_fifo(mesh.n, mesh.row_ptr, mesh.col, int(s))[0] for s in srcs]
    for knobs in ({"cluster_start": 1}, {"cluster_start": 1, "cluster_handover_edges": 64},
                  {"cluster_start": 0}):
        G.set_tuning(**knobs)
        d, st = dawn.sssp_batch(G, torch.from_numpy(srcs).cuda(), stats=True)
        d = d.cpu().numpy().view(np.uint32)
        for i, s in enumerate(srcs):
            assert np.array_equal(d[i], exp[i]), (knobs, int(s))
            rec, er = oracle.record(mesh.n, mesh.row_ptr, int(s), exp[i])
            sd = dawn.stats_to_dict(st[i])
            assert sd["levels"] == int(rec["ecc"]) and sd["edges_reach"] == er, (knobs, sd)

def _pull_then_push_graph(hub_arcs: int, seed: int):
    """0 -> 2,000 A -> 20,000 B (each A: 20 arcs into B) -> 300 C (one arc per B) -> D, where C's
    first vertex H has `hub_arcs` arcs into D and the other C vertices one each.  With a large
    alpha the growing levels run as pull, with beta = 1 the shrinking frontier C turns to
    push: a push from the bitmap frontier the pull left."""
    rng = np.random.default_rng(seed)
    A = np.arange(1, 2001)
    B = np.arange(2001, 22001)
    C = np.arange(22001, 22301)
    D0 = 22301
    e = [[0, a] for a in A]
    e += [[int(a), int(b)] for a in A for b in rng.choice(B, 20, replace=False)]
    e += [[int(b), int(rng.choice(C))] for b in B]
    nd = max(hub_arcs, 300)
    e += [[int(C[0]), D0 + j] for j in range(hub_arcs)]
    e += [[int(c), D0 + int(rng.integers(0, nd))] for c in C[1:]]
    return graphgen.from_edges(D0 + nd, e)


def test_push_from_pull_bitmap_frontier():
    # the push level right after pull levels reads the bitmap frontier directly when no row
    # exceeds 256 arcs, else converts it to a queue first (hub H in the frontier): both against
    # the oracle, and the scenario checked through the level counts
    for hub, seed in ((40, 1), (1000, 2)):
        g = _pull_then_push_graph(hub, seed)
        G = dev_graph(g)
        G.set_tuning(alpha=1e9, beta=1.0)
        exp = oracle.bfs_fifo(g.n, g.row_ptr, g.col, 0)[0]
        d, st = gpu_dist(G, 0, "auto", stats=True)
        assert np.array_equal(d, exp), hub
        assert st["pull_levels"] == 3 and st["push_levels"] == 1, st  # L3: push from the bitmap
        D = dawn.sssp_batch(G, torch.tensor([0, 0, 1], dtype=torch.int32, device="cuda"))
        D = D.cpu().numpy().view(np.uint32)
        assert np.array_equal(D[0], exp) and np.array_equal(D[1], exp)
        assert np.array_equal(D[2], oracle.bfs_fifo(g.n, g.row_ptr, g.col, 1)[0])


def test_sssp_batch_lanes():
    # DAWN_PARAM_BATCH_LANES: 1/2/4/8 concurrent grid-wide searches (own state, own stream) give
    # the oracle's rows and statistics for every source, incl. k not a multiple of the lanes,
    # repeated sources, and every direction variant
    g = graphgen.kron(15, 16, 15)
    G = dev_graph(g)
    srcs = np.concatenate([g.sample_sources(9, seed=11), [0]]).astype(np.int32)
    srcs[3] = srcs[1]                                               # a repeated source
    exp = [oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(s))[0] for s in srcs]
    # batch_dynamic: lanes claim sources one at a time from a shared counter (1, the default)
    # or run fixed contiguous shares (0); either way row i / stats i belong to source i
    for dyn in (1, 0):
        G.set_tuning(batch_dynamic=dyn)
        for lanes in (1, 2, 4, 8, 16):
            G.set_tuning(batch_lanes=lanes)
            for v in VARIANTS:
                d, st = dawn.sssp_batch(G, torch.from_numpy(srcs).cuda(), v, stats=True, check=True)
                d = d.cpu().numpy().view(np.uint32)
                for i, s in enumerate(srcs):
                    assert np.array_equal(d[i], exp[i]), (dyn, lanes, v, int(s))
                    rec, er = oracle.record(g.n, g.row_ptr, int(s), exp[i])
                    sd = dawn.stats_to_dict(st[i])
                    assert sd["levels"] == int(rec["ecc"]) and sd["edges_reach"] == er, (dyn, lanes, v)
    G.set_tuning(batch_dynamic=1)
    # many more searches than lanes, some far cheaper than others (sources with a tiny reach):
    # every index is claimed exactly once
    small = np.concatenate([srcs, np.arange(40, dtype=np.int32)])
    exps = [oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(s))[0] for s in small]
    d = dawn.sssp_batch(G, torch.from_numpy(small).cuda()).cpu().numpy().view(np.uint32)
    assert all(np.array_equal(d[i], exps[i]) for i in range(len(small)))
    with pytest.raises(dawn.DawnError):
        G.set_tuning(batch_lanes=17)
    # the lanes share nothing across calls: a single dawn_sssp between batches still matches
    G.set_tuning(batch_lanes=4)
    dawn.sssp_batch(G, torch.from_numpy(srcs).cuda())
    assert np.array_equal(gpu_dist(G, int(srcs[2])), exp[2])
