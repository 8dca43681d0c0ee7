"""The APSP path through a real NCCL process group (PAPER E11-E12 L303-308: the
sources are independent, so they shard; NCCL carries only the 32-byte records).  One process
per visible GPU (world = torch.cuda.device_count(): 1 on the single-GPU test box, N on an
N-GPU box): every rank runs dawn_apsp on its shard on its own GPU and the binding's
gather_records does the one all-gather over NCCL; rank 0 compares the gathered records with the
oracle byte for byte, and the gathered set is identical for every world size (determinism
across W, the SPEC S:L456 idea applied to GPU count)."""
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

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    g = graphgen.kron(13, 16, 13)
    G = dawn.Graph(g.row_ptr, g.col, True)
    verts, _ = dawn.largest_wcc(G)
    for k in (len(verts), 700, 256, 1):
        srcs = verts[:k]
        full = dawn.apsp(G, srcs, rank, world)             # shard + NCCL all-gather
        torch.cuda.synchronize()
        if rank == 0:
            np.save(os.path.join(out_dir, f"nccl_{k}.npy"), full.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_apsp_nccl_all_visible_gpus(tmp_path):
    world = torch.cuda.device_count()
    assert world >= 1
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    g = graphgen.kron(13, 16, 13)
    verts, _ = oracle.largest_wcc(g.n, g.row_ptr, g.col)
    for k in (len(verts), 700, 256, 1):
        full = np.load(tmp_path / f"nccl_{k}.npy")
        exp = oracle.records(g.n, g.row_ptr, g.col, verts[:k])
        assert full.tobytes() == exp.tobytes(), (world, k)


def _part_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    g = graphgen.kron(13, 16, 13)
    pg = dawn.PartGraph(dawn.part_build(g.row_ptr, g.col, world, rank), world, rank, device=dev)
    for i, s in enumerate(g.sample_sources(3, seed=5)):
        for v in ("auto", "push", "pull"):
            d = dawn.part_sssp(pg, int(s), v)              # one NCCL all-gather per level
            torch.cuda.synchronize()
            np.save(os.path.join(out_dir, f"part_{rank}_{i}_{v}.npy"), d.cpu().numpy())
            f = dawn.part_sssp_fused(pg, int(s), v)        # fused: peer stores over IPC mappings
            torch.cuda.synchronize()
            np.save(os.path.join(out_dir, f"fused_{rank}_{i}_{v}.npy"), f.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_partitioned_sssp_nccl_all_visible_gpus(tmp_path):
    # NEXT-3 through torch.distributed / NCCL: each rank holds only the arcs into its vertex
    # range; the gathered distance slices equal the oracle
    world = torch.cuda.device_count()
    mp.start_processes(_part_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    g = graphgen.kron(13, 16, 13)
    for i, s in enumerate(g.sample_sources(3, seed=5)):
        exp, _ = oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(s))
        for v in ("auto", "push", "pull"):
            for tag in ("part", "fused"):
                got = np.concatenate([np.load(tmp_path / f"{tag}_{r}_{i}_{v}.npy")[: dawn.part_range(g.n, world, r)[1] - dawn.part_range(g.n, world, r)[0]]
                                      for r in range(world)]).view(np.uint32)
                assert np.array_equal(got, exp), (tag, world, s, v)


def _fused_ipc_worker(rank, world, port, out_dir):
    # two processes on ONE device: the exchange buffers are shared through CUDA IPC
    # (torch.multiprocessing's tensor sharing, handles over a gloo group) exactly as across GPUs,
    # and the two persistent kernels signal each other with system-scope atomics; the device
    # time-slices the two contexts, so this checks the protocol, not the speed
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = graphgen.kron(10, 8, 10)
    pg = dawn.PartGraph(dawn.part_build(g.row_ptr, g.col, world, rank), world, rank,
                        device=torch.device("cuda", 0))
    for i, s in enumerate(g.sample_sources(2, seed=3)):
        d = dawn.part_sssp_fused(pg, int(s))
        torch.cuda.synchronize()
        np.save(os.path.join(out_dir, f"ipc_{rank}_{i}.npy"), d.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_fused_exchange_across_processes_ipc(tmp_path):
    world = 2
    ctx = mp.start_processes(_fused_ipc_worker, args=(world, _free_port(), str(tmp_path)),
                             nprocs=world, join=False, start_method="spawn")
    import time
    deadline = time.time() + 240
    while not ctx.join(timeout=5):
        if time.time() > deadline:
            for p in ctx.processes:
                p.kill()
            pytest.fail("fused exchange across processes did not finish in 240 s")
    g = graphgen.kron(10, 8, 10)
    for i, s in enumerate(g.sample_sources(2, seed=3)):
        exp, _ = oracle.bfs_fifo(g.n, g.row_ptr, g.col, int(s))
        got = np.concatenate([np.load(tmp_path / f"ipc_{r}_{i}.npy")[: dawn.part_range(g.n, world, r)[1] - dawn.part_range(g.n, world, r)[0]]
                              for r in range(world)]).view(np.uint32)
        assert np.array_equal(got, exp), (i, int(s))
