"""Multi-process (world_size 2, gloo, CPU) coverage of bench.py's N>1 logic: replicas are
independent, so the only cross-rank operations are the barrier and the max/sum of the
timing scalars; the reference arm runs on rank 0 only."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms, units = bench.reduce_timing(100.0 + 50.0 * rank, 1000.0 * (rank + 1), world, "cpu")
    dist.barrier()
    # the reference arm: only rank 0 does work
    class A:
        config, warmup, steps, gpus = 1, 0, 0, world
    bench.run_reference(A(), rank, world) if rank != 0 else None
    out[rank] = (ms, units)
    dist.destroy_process_group()


def test_reduce_timing_world2_gloo():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for r in range(2):
        ms, units = out[r]
        assert ms == 150.0               # max over ranks
        assert units == 3000.0           # sum over ranks


def test_reduce_timing_single_rank_passthrough():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.reduce_timing(12.5, 7.0, 1) == (12.5, 7.0)
