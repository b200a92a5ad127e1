"""Multi-rank host logic on CPU (gloo): bench.py's max-over-ranks device time and summed
unknown-iterations, and the slab bookkeeping of the sharded 3D solver (rsfde_team_partition: x1 slabs,
x2 slabs, all-to-all block layout) exercised by a real all-to-all transpose of a seeded grid between
world_size 2 and 4 processes."""
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


def _transpose_worker(rank, ws, port, n, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    sys.path.insert(0, ROOT)
    import numpy as np
    from paper_2404_10221_b200.solver import team_partition
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    n1, n2, n3 = n
    part = team_partition(n, ws, rank)
    s, s2, blk = part["s"], part["s2"], part["block"]
    allp = [None] * ws
    dist.all_gather_object(allp, part)
    G = np.random.default_rng(7).uniform(-1, 1, (n1, n2, n3))          # the same global grid on every rank
    # layout A: this rank's x1 slab, padded to s planes (the pad plane of the last rank stays zero)
    A = np.zeros((s, n2, n3))
    A[:part["x1_count"]] = G[part["x1_lo"]:part["x1_lo"] + part["x1_count"]]
    # send block r' = [x2l < s2][x3][x1l < s] of the x2 range of rank r' (pack_AT_kernel's layout)
    send = np.zeros((ws, s2, n3, s))
    for rp in range(ws):
        lo = rp * s2
        hi = min(lo + s2, n2)
        if hi > lo:
            send[rp, :hi - lo] = np.transpose(A[:, lo:hi, :], (1, 2, 0))
    assert send[0].size == blk
    recv = torch.empty(ws * blk, dtype=torch.float64)
    dist.all_to_all_single(recv, torch.from_numpy(send.reshape(-1)))
    # layout T = [x2l < s2][x3][x1 < ws s] (unpack_AT_kernel's layout; x1 = r'' s + x1l)
    R = recv.numpy().reshape(ws, s2, n3, s)
    T = np.transpose(R, (1, 2, 0, 3)).reshape(s2, n3, ws * s)
    ref = np.zeros((s2, n3, ws * s))
    ref[:part["x2_count"], :, :n1] = np.transpose(G[:, part["x2_lo"]:part["x2_lo"] + part["x2_count"], :], (1, 2, 0))
    out[rank] = (allp, bool(np.array_equal(T, ref)))
    dist.destroy_process_group()


@pytest.mark.parametrize("ws,n", [(2, (15, 7, 5)), (4, (15, 11, 3)), (2, (1, 1, 4))])
def test_slab_partition_and_alltoall_transpose_gloo(ws, n):
    port = 29600 + (os.getpid() + 17 * ws + n[1]) % 300
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_transpose_worker, args=(ws, port, n, out), nprocs=ws, join=True)
    parts = out[0][0]
    # x1 slabs tile [0, n1) in rank order, x2 slabs tile [0, n2); every rank agrees
    assert [p["x1_lo"] for p in parts] == [r * parts[0]["s"] for r in range(ws)]
    assert sum(p["x1_count"] for p in parts) == n[0] and sum(p["x2_count"] for p in parts) == n[1]
    for r in range(ws):
        assert out[r][0] == parts
        assert out[r][1], f"rank {r}: transposed slab differs from the global transpose"


def _chunked_worker(rank, ws, port, n, req, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    sys.path.insert(0, ROOT)
    import numpy as np
    from paper_2404_10221_b200.solver import team_chunking, team_partition
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    n1, n2, n3 = n
    part = team_partition(n, ws, rank)
    ch = team_chunking(n, ws, req)
    s, s2, blk = part["s"], part["s2"], part["block"]
    nc, sc, piece = ch["nchunk"], ch["sc"], ch["piece"]
    G = np.random.default_rng(11).uniform(-1, 1, (n1, n2, n3))
    A = np.zeros((s, n2, n3))
    A[:part["x1_count"]] = G[part["x1_lo"]:part["x1_lo"] + part["x1_count"]]
    # send blocks [peer][chunk][x2l < s2][x3][x1l < sc]: sub-slab c = planes [c sc, (c+1) sc) of the slab
    send = np.zeros((ws, nc, s2, n3, sc))
    for rp in range(ws):
        lo, hi = rp * s2, min(rp * s2 + s2, n2)
        for c in range(nc):
            if hi > lo:
                send[rp, c, :hi - lo] = np.transpose(A[c * sc:(c + 1) * sc, lo:hi, :], (1, 2, 0))
    recv = np.zeros((ws, nc, s2, n3, sc))
    # one all-to-all per piece c (what the exchange stream does while sub-slab c+1 is computed)
    for c in range(nc):
        buf = torch.empty(ws * piece, dtype=torch.float64)
        dist.all_to_all_single(buf, torch.from_numpy(np.ascontiguousarray(send[:, c]).reshape(-1)))
        recv[:, c] = buf.numpy().reshape(ws, s2, n3, sc)
    # the x1 pencil (x2l, x3) = segments (r'', c) of sc planes: x1 = (r'' nc + c) sc + x1l
    T = np.transpose(recv, (2, 3, 0, 1, 4)).reshape(s2, n3, ws * nc * sc)
    ref = np.zeros((s2, n3, ws * s))
    ref[:part["x2_count"], :, :n1] = np.transpose(G[:, part["x2_lo"]:part["x2_lo"] + part["x2_count"], :], (1, 2, 0))
    out[rank] = (ch, blk, bool(np.array_equal(T, ref)))
    dist.destroy_process_group()


@pytest.mark.parametrize("ws,n,req,expect", [(2, (15, 7, 5), 4, (4, 2)), (2, (31, 3, 2), 8, (8, 2)),
                                             (4, (15, 11, 3), 4, (2, 2)), (2, (3, 1, 4), 4, (1, 2))])
def test_chunked_alltoall_pieces_gloo(ws, n, req, expect):
    # rsfde_team_chunking's piece layout [peer][chunk][x2l][x3][x1l < sc] exchanged piece by piece
    # reassembles every x1 pencil as the segments (peer, chunk) -- the layout the x1 pass reads with
    # seg_lg = log2(sc), seg_stride = piece
    port = 29900 + (os.getpid() + 13 * ws + n[0] + req) % 90
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_chunked_worker, args=(ws, port, n, req, out), nprocs=ws, join=True)
    for r in range(ws):
        ch, blk, ok = out[r]
        assert (ch["nchunk"], ch["sc"]) == expect
        assert ch["piece"] * ch["nchunk"] == blk
        assert ok, f"rank {r}: pencils reassembled from the pieces differ from the global transpose"
