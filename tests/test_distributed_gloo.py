"""CPU, world_size 2 over gloo: the sharded DLRM exchange (TWRW plan -> data-parallel, one
unpadded all_to_all_single of the kernel's output rows) delivers every rank exactly the global
pooled embeddings of its sample slice.  Each rank's send buffer is the CPU restatement of K5's
output bytes (pool_rank_reference: fp32 whole tables, fp64 row-wise partials at the kernel's
offsets) — the layout the GPU test checks the kernel against."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.embbag import embbag_rows_reference
from paper_2504_19365_b200.bench.dlrm import exchange, make_batch, plan_shards, pool_rank_reference, table_rows

SEED, B, L, D = 11, 16, 5, 32


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows = table_rows(64 << 20, D, 26)
    plan = plan_shards(rows, world, D)
    full_idx = make_batch(SEED, 0, rows, B, L, 1.05, True)
    send = torch.from_numpy(pool_rank_reference(plan, rank, full_idx[:, plan.rank_tables(rank)], SEED))
    got = exchange(plan, send, rank, B)
    exp = embbag_rows_reference(SEED, full_idx, D)[rank * (B // world):(rank + 1) * (B // world)]
    q.put((rank, bool(np.array_equal(got.numpy(), exp))))
    dist.destroy_process_group()


def test_sharded_exchange_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
