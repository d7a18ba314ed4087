"""Multi-rank host logic on CPU (world_size 2, gloo): the group sharding bench.py
uses and the gray all-reduce it ends with.  Each rank runs the CPU
oracle on its own group shard and the ranks sum their gray outputs with
torch.distributed.all_reduce — this must equal the single-rank result, exactly
as the NCCL all-reduce of the GPU path does on the device."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank: int, world: int, port: int, cfg: tuple, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from bench import shard_groups
        prob = synth.config(*cfg)
        g0, g1 = shard_groups(prob.G, world, rank)
        part = torch.from_numpy(oracle.sweep(prob.group_slice(g0, g1), nthreads=1))
        dist.all_reduce(part, op=dist.ReduceOp.SUM)
        # broadcast of an NCCL-id-like blob, as bench.py does for sweep_nccl_unique_id
        blob = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(blob, src=0)
        q.put((rank, (g0, g1), part.numpy(), blob[0] == bytes(range(128))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg", [(2, (4, 24, 6)), (2, (5, 12, 5)), (3, (2, 64, 7))])
def test_sharded_gray_allreduce_equals_full(world, cfg):
    import oracle
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    shards = [r[1] for r in res]
    # contiguous, disjoint, covering
    assert shards[0][0] == 0 and shards[-1][1] == synth.config(*cfg).G
    for a, b in zip(shards, shards[1:]):
        assert a[1] == b[0]
    full = oracle.sweep(synth.config(*cfg), nthreads=1)
    for _, _, got, ok in res:
        assert ok
        assert np.abs(got - full).max() <= 1e-13 * np.abs(full).max()


def test_shard_groups_balance():
    from bench import shard_groups
    for G in (1, 7, 32, 64, 65):
        for ws in (1, 2, 3, 4, 8):
            parts = [shard_groups(G, ws, r) for r in range(ws)]
            sizes = [b - a for a, b in parts]
            assert sum(sizes) == G and max(sizes) - min(sizes) <= 1
            assert parts[0][0] == 0 and all(parts[i][1] == parts[i + 1][0] for i in range(ws - 1))


# ------------------------------------------------------------------ the product, 2 ranks on one GPU
def _gpu_worker(rank: int, world: int, port: int, cfg: tuple, q):
    """One rank of a group-sharded run through the product (libsweep via the binding): the
    rank sweeps its group shard on cuda:0 (nranks = 1 inside the library: NCCL cannot put two
    ranks on one device) and the ranks sum the gray outputs with gloo, as the NCCL all-reduce
    of a multi-GPU run does on the device."""
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        import paper_2504_21784_b200 as pk
        from bench import shard_groups
        prob = synth.config(*cfg)
        g0, g1 = shard_groups(prob.G, world, rank)
        shard = prob.group_slice(g0, g1)
        out = pk.run_problem(shard, device=0)
        part = torch.from_numpy(out)
        dist.all_reduce(part, op=dist.ReduceOp.SUM)
        q.put((rank, part.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,cfg", [(2, (5, 16, 8)), (2, (4, 20, 6)), (2, (2, 128, 9))])
def test_product_sharded_two_ranks_one_gpu(world, cfg):
    import torch
    import oracle
    import synth
    from tests.parity import assert_parity
    import paper_2504_21784_b200 as pk
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device on a -m gpu run")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    prob = synth.config(*cfg)
    full = pk.run_problem(prob, device=0)
    ref = oracle.sweep(prob)
    for _, got in res:
        # sharded sum = one-rank result (to rounding of the different group partition) = oracle
        assert np.abs(got - full).max() <= 1e-13 * np.abs(full).max()
        assert_parity(got, ref, prob.dim, prob.nx, prob.ny, prob.p)
