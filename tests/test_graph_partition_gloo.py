"""CPU, world_size 2 over gloo: the 1D-partitioned BFS and PageRank exchanges (bench/graph.py
bfs_partitioned / pagerank_partitioned: per-level all-gather + OR of next-frontier bitmaps,
per-iteration all-gather of x slices) reproduce the single-device answers bit for bit.  Each
rank's compute is the CPU restatement (oracle/graph.py OracleBfsRank / OraclePagerankRank); the
GPU test (test_gpu_graph_partition.py) runs the same drivers over the kernels."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _graph(seed, V=1024, E=12000, transpose=False):
    rng = np.random.default_rng(seed)
    src = (rng.zipf(1.3, E) * 7919) % V
    dst = rng.integers(0, V, E)
    outdeg = np.bincount(src, minlength=V)
    if transpose:
        src, dst = dst, src
    order = np.lexsort((dst, src))
    src, dst = src[order], dst[order]
    row_ptr = np.zeros(V + 1, dtype=np.int64)
    row_ptr[1:] = np.cumsum(np.bincount(src, minlength=V))
    return row_ptr, dst.astype(np.int32), outdeg


def _allgather(world):
    def ag(t):
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return out
    return ag


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.graph import OracleBfsRank, OraclePagerankRank, bfs_levels, pagerank_f32
    from paper_2504_19365_b200.bench.graph import bfs_partitioned, pagerank_partitioned, partition_1d
    ok = True
    rp, col, _ = _graph(1)
    part = partition_1d(rp, world)[rank]
    for source in (0, 77, 513):
        r = OracleBfsRank(part, rp, col, len(rp) - 1, source)
        bfs_partitioned([r], _allgather(world))
        ok &= bool(np.array_equal(r.level.numpy(), bfs_levels(rp, col, source)))
    rT, cT, od = _graph(2, transpose=True)
    part = partition_1d(rT, world)[rank]
    pr = OraclePagerankRank(part, rT, cT, len(rT) - 1, od)
    pagerank_partitioned([pr], 10, _allgather(world))
    full = pagerank_f32(rT, cT, od, 10)
    ok &= bool(np.array_equal(pr.r.numpy(), full[part.v0:part.v1]))
    q.put((rank, ok))
    dist.destroy_process_group()


def test_partitioned_graph_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
