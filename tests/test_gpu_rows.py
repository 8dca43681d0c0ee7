"""GPU tests of the APSP output modes: distance rows
streamed to host memory through a caller sink (dawn_apsp_rows), and the configurable refusal of
dense k x n outputs (DAWN_PARAM_DENSE_MAX_ENTRIES -> DAWN_ERR_CAPACITY).  Every row is compared
element by element with the CPU oracle."""
import numpy as np
import pytest
import torch

import graphgen
import oracle
import paper_2208_04514_b200 as dawn

pytestmark = pytest.mark.gpu
UNR = oracle.UNREACHED


def _graph(g):
    if g.symmetric:
        return dawn.Graph(g.row_ptr, g.col, True, validate=True)
    p, i = g.transpose()
    return dawn.Graph(g.row_ptr, g.col, False, p, i, validate=True)


def _collect(G, sources, chunk):
    got, order = {}, []

    def sink(first, rows):
        order.append((first, rows.shape[0]))
        for i in range(rows.shape[0]):
            got[first + i] = rows[i].copy()

    dawn.apsp_rows(G, sources, sink, chunk=chunk)
    return got, order


def test_three_cycle_matrix():
    # directed 3-cycle -> [[0,1,2],[2,0,1],[1,2,0]]
    g = graphgen.from_edges(3, [(0, 1), (1, 2), (2, 0)])
    got, order = _collect(_graph(g), [0, 1, 2], chunk=2)
    assert order == [(0, 2), (2, 1)]
    M = np.stack([got[i] for i in range(3)])
    assert M.tolist() == [[0, 1, 2], [2, 0, 1], [1, 2, 0]]


def test_edgeless_rows():
    # edgeless n=3 -> every row unreached except d(s, s) = 0 (reading Q4)
    g = graphgen.from_edges(3, [])
    got, _ = _collect(_graph(g), [0, 1, 2], chunk=256)
    for s in range(3):
        exp = np.full(3, UNR, np.uint32)
        exp[s] = 0
        assert np.array_equal(got[s], exp)


def test_random_digraph_64_matches_floyd_warshall():
    # n=64 random digraph -> matrix equals the oracle row by row
    g = graphgen.er(64, 256, 5)
    fw = oracle.floyd_warshall(g.n, g.row_ptr, g.col)
    got, _ = _collect(_graph(g), list(range(64)), chunk=7)
    M = np.stack([got[i] for i in range(64)])
    assert np.array_equal(M, fw)


def test_ragged_pieces_kron12():
    # 700 sources in pieces of 300 (two full 256-source passes + partial ones per piece), with
    # repeated sources; every row vs the FIFO-BFS oracle
    g = graphgen.kron(12, 16, 12)
    G = _graph(g)
    src = list(g.sample_sources(690, seed=4)) + [3, 3, 0, g.n - 1] * 2 + [5, 7]
    got, order = _collect(G, src, chunk=300)
    assert [o[0] for o in order] == [0, 300, 600] and sum(o[1] for o in order) == len(src)
    for i, s in enumerate(src):
        assert np.array_equal(got[i], oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(s))[0]), (i, s)


def test_sink_stop_and_errors():
    g = graphgen.kron(10, 16, 10)
    G = _graph(g)
    seen = []

    def stop_after_first(first, rows):
        seen.append(first)
        return False

    with pytest.raises(dawn.DawnError) as ei:
        dawn.apsp_rows(G, list(range(600)), stop_after_first, chunk=256)
    assert ei.value.status == 1 and seen == [0]
    with pytest.raises(dawn.DawnError) as ei:
        dawn.apsp_rows(G, [0, g.n], lambda f, r: None)
    assert ei.value.status == 2  # DAWN_ERR_BOUNDS before any work
    # dense outputs above the configured limit are refused
    G.set_tuning(dense_max_entries=10 * g.n)
    with pytest.raises(dawn.DawnError) as ei:
        dawn.msssp(G, list(range(10)), dist=True, records=False)
    assert ei.value.status == 4
    d, _ = dawn.msssp(G, list(range(9)), dist=True, records=False)  # below the limit: fine
    assert np.array_equal(d[3].cpu().numpy().view(np.uint32),
                          oracle.bfs_fifo(g.n, g.row_ptr, g.col, 3)[0])
    with pytest.raises(dawn.DawnError) as ei:
        dawn.apsp_rows(G, list(range(20)), lambda f, r: None, chunk=16)
    assert ei.value.status == 4
    got, _ = _collect(G, list(range(20)), chunk=9)  # pieces under the limit stream fine
    assert all(np.array_equal(got[i], oracle.bfs_fifo(g.n, g.row_ptr, g.col, i)[0]) for i in range(20))
    torch.cuda.synchronize()


def test_dist_u8_compaction():
    # dawn_dist_u8: 1-byte rows (255 = unreached / overflow with the flag), ragged lengths
    g = graphgen.kron(11, 16, 11)
    G = _graph(g)
    for s in g.sample_sources(3, seed=1):
        d = dawn.sssp(G, int(s))
        u8, fl = dawn.dist_u8(d)
        exp = oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(s))[0]
        assert np.array_equal(u8.cpu().numpy(), np.where(exp == UNR, 255, exp).astype(np.uint8))
        assert int(fl[0]) == 0
    x = torch.tensor([0, 1, 254, 255, 256, -1, 7], dtype=torch.int32, device="cuda")  # n % 4 = 3
    u8, fl = dawn.dist_u8(x)
    assert u8.cpu().tolist() == [0, 1, 254, 255, 255, 255, 7] and int(fl[0]) == 1
    u8, fl = dawn.dist_u8(torch.tensor([3, -1, 2, 9], dtype=torch.int32, device="cuda"))
    assert u8.cpu().tolist() == [3, 255, 2, 9] and int(fl[0]) == 0
    with pytest.raises(dawn.DawnError):
        dawn.dist_u8(torch.zeros(9, dtype=torch.int32, device="cuda")[1:])  # misaligned


def test_dist_u4_compaction():
    # dawn_dist_u4: 4-bit rows, two per byte (15 = unreached / overflow with the flag); every
    # tail length 1..17 (the 8-entry vector body plus the per-byte tail, odd counts padded)
    g = graphgen.kron(11, 16, 11)
    G = _graph(g)
    for s in g.sample_sources(3, seed=1):
        d = dawn.sssp(G, int(s))
        u4, fl = dawn.dist_u4(d)
        exp = oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(s))[0]
        assert int(exp[exp != UNR].max()) < 15 and int(fl[0]) == 0
        assert np.array_equal(dawn.unpack_u4(u4.cpu().numpy(), g.n), exp)
    rng = np.random.default_rng(5)
    for cnt in range(1, 18):
        v = rng.integers(0, 15, cnt).astype(np.int64)
        v[rng.random(cnt) < 0.3] = -1
        x = torch.from_numpy(v.astype(np.int32)).cuda()
        u4, fl = dawn.dist_u4(x)
        assert u4.numel() == (cnt + 1) // 2 and int(fl[0]) == 0
        exp = np.where(v < 0, UNR, v).astype(np.uint32)
        assert np.array_equal(dawn.unpack_u4(u4.cpu().numpy(), cnt), exp), cnt
        if cnt % 2:
            assert int(u4[-1].item()) >> 4 == 15                       # pad nibble
    u4, fl = dawn.dist_u4(torch.tensor([14, 15, 16, -1, 3], dtype=torch.int32, device="cuda"))
    assert u4.cpu().tolist() == [14 | (15 << 4), 15 | (15 << 4), 3 | (15 << 4)] and int(fl[0]) == 1
    with pytest.raises(dawn.DawnError):
        dawn.dist_u4(torch.zeros(9, dtype=torch.int32, device="cuda")[1:])  # misaligned
    torch.cuda.synchronize()
