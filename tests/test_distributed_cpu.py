"""The N>1 APSP path on CPU: world_size-2 gloo processes each take their shard of the source
list (dawn_apsp_shard, host-only logic of libdawn.so), compute the shard's records with the
oracle, and reassemble them with the binding's gather_records (the single all-gather of the
APSP path).  The result must equal the single-process oracle records byte for
byte, for several source counts including partial batches."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import graphgen
import oracle
import paper_2208_04514_b200 as dawn


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, k, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = graphgen.kron(10, 8, 3)
    verts, _ = g.largest_wcc()
    srcs = np.resize(verts, k)  # k may exceed S_wcc: repeated sources are allowed
    mine = dawn.apsp_shard(k, rank, world)
    recs = oracle.records(g.n, g.row_ptr, g.col, srcs[mine], threads=2)
    local = torch.from_numpy(recs.view(np.int64).reshape(-1, 4).copy())
    full = dawn.gather_records(local, k, world)
    if rank == 0:
        np.save(os.path.join(out_dir, f"full_{k}.npy"), full.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("k", [1, 255, 256, 600, 1030])
def test_apsp_gather_world2_gloo(tmp_path, k):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), k, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    full = np.load(tmp_path / f"full_{k}.npy")
    g = graphgen.kron(10, 8, 3)
    verts, _ = g.largest_wcc()
    exp = oracle.records(g.n, g.row_ptr, g.col, np.resize(verts, k), threads=4)
    assert full.tobytes() == exp.tobytes()
    got = full.view(oracle.REC_DTYPE).reshape(-1)
    assert np.array_equal(got["source"], np.resize(verts, k).astype(np.uint32))
