"""Host side of the partitioned single-source path on CPU, world_size-2
gloo: every rank builds its partition with the host builder of libdawn.so (dawn_part_build) and
the ranks check together that the partitions cover the graph exactly (each arc held once, by
the owner of its target, in both groupings; own out-degrees), then run the binding's frontier
exchange (part_exchange: the per-level all-gather) on CPU tensors and decode the gathered
bitmap with the kernels' index rule."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import graphgen
import paper_2208_04514_b200 as dawn


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _HostPart:  # the exchange buffers of a rank, on the host (no device / workspace)
    def __init__(self, n, world, rank):
        self.n, self.world, self.rank = n, world, rank
        self.lo, self.hi = dawn.part_range(n, world, rank)
        self.B = dawn.part_range(n, world, 0)[1]  # block size (rank 0 owns a full block)
        self.slice_words = 4 + self.B // 32
        self.send = torch.zeros(self.slice_words, dtype=torch.int32)
        self.recv = torch.zeros(self.slice_words * world, dtype=torch.int32)


def _worker(rank, world, port, out_dir, name):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = graphgen.kron(10, 16, 10) if name == "kron" else graphgen.er(1000, 8000, 1)
    P = dawn.part_build(g.row_ptr, g.col, world, rank)
    # arcs of this rank as global (source, target) from both groupings
    src_o = np.repeat(np.arange(g.n), np.diff(P["out_rp"]))
    a_out = np.stack([src_o, P["out_col"].astype(np.int64) + P["lo"]], 1)
    tgt_i = np.repeat(np.arange(P["hi"] - P["lo"]), np.diff(P["in_rp"])) + P["lo"]
    a_in = np.stack([P["in_col"].astype(np.int64), tgt_i], 1)
    np.save(os.path.join(out_dir, f"{name}_out_{rank}.npy"), a_out)
    np.save(os.path.join(out_dir, f"{name}_in_{rank}.npy"), a_in)
    np.save(os.path.join(out_dir, f"{name}_deg_{rank}.npy"), P["deg"])
    # the frontier exchange: rank r marks its owned vertices v with v % 3 == r % 3
    hp = _HostPart(g.n, world, rank)
    words = hp.send[4:].numpy().view(np.uint32)
    for v in range(hp.lo, hp.hi):
        if v % 3 == rank % 3:
            t = v - hp.lo
            words[t >> 5] |= np.uint32(1 << (t & 31))
    hp.send[0] = int(sum(1 for v in range(hp.lo, hp.hi) if v % 3 == rank % 3))
    dawn.part_exchange(hp)
    rv = hp.recv.numpy().view(np.uint32)
    got = [v for v in range(g.n)
           if (rv[(v // hp.B) * hp.slice_words + 4 + (v % hp.B) // 32] >> ((v % hp.B) & 31)) & 1]
    exp = [v for v in range(g.n) if v % 3 == (dawn.part_range(g.n, world, 0)[0] * 0 +
                                              next(r for r in range(world)
                                                   if dawn.part_range(g.n, world, r)[0] <= v <
                                                   dawn.part_range(g.n, world, r)[1])) % 3]
    assert got == exp, rank
    assert sum(int(rv[q * hp.slice_words]) for q in range(world)) == len(exp)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["kron", "er"])
def test_partition_world2_gloo(tmp_path, name):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path), name), nprocs=world,
                       join=True, start_method="spawn")
    g = graphgen.kron(10, 16, 10) if name == "kron" else graphgen.er(1000, 8000, 1)
    exp = np.stack([np.repeat(np.arange(g.n), np.diff(g.row_ptr)), g.col.astype(np.int64)], 1)
    key = lambda a: np.sort(a[:, 0] * g.n + a[:, 1])
    for grp in ("out", "in"):
        allarcs = np.concatenate([np.load(tmp_path / f"{name}_{grp}_{r}.npy") for r in range(world)])
        assert np.array_equal(key(allarcs), key(exp)), grp  # every arc exactly once
    for r in range(world):
        lo, hi = dawn.part_range(g.n, world, r)
        a = np.load(tmp_path / f"{name}_out_{r}.npy")
        assert ((a[:, 1] >= lo) & (a[:, 1] < hi)).all()  # held by the owner of its target
        assert np.array_equal(np.load(tmp_path / f"{name}_deg_{r}.npy"),
                              np.diff(g.row_ptr)[lo:hi].astype(np.uint32))


def test_partition_ranges_and_errors():
    for n, W in [(1, 1), (40, 4), (1000, 3), (1 << 20, 8)]:
        r = [dawn.part_range(n, W, k) for k in range(W)]
        assert r[0][0] == 0 and r[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
        assert all((hi - lo) % 32 == 0 for lo, hi in r[:-1] if hi < n)
    with pytest.raises(dawn.DawnError):
        dawn.part_range(10, 2, 2)
    bad = np.array([0, 1, 2], np.int64)
    with pytest.raises(dawn.DawnError) as ei:
        dawn.part_build(bad, np.array([1, 5], np.int32), 1, 0)  # col out of range
    assert ei.value.status == 6
