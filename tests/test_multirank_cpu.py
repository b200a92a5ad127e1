"""World-size-2 gloo test (CPU) of the multi-rank host logic of bench.py: the max-over-ranks device
time and the summed unknown-iterations that define the whole-job value."""
import os
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import bench
    t = bench.max_over_ranks(1.0 + rank, ws)
    s = bench.sum_over_ranks(10.0 * (rank + 1), ws)
    bench.barrier(ws)
    out[rank] = (t, s)
    dist.destroy_process_group()


def test_rank_reductions_gloo():
    ws = 2
    port = 29500 + os.getpid() % 1000
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(ws, port, out), nprocs=ws, join=True)
    for r in range(ws):
        assert out[r] == (2.0, 30.0)
