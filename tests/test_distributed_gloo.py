"""CPU, world_size 2 over gloo: the sharded DLRM exchange (table-wise -> data-parallel, one
all_to_all) delivers every rank exactly the global pooled embeddings of its sample slice.  Each
rank pools its own tables with the CPU oracle (stand-in for its GPU's kernel)."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.embbag import embbag_reference
from paper_2504_19365_b200.bench.dlrm import exchange_pooled, layout, make_batch, shard_tables, table_rows

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
    groups, _ = shard_tables(rows, world)
    mine = groups[rank]
    idx = make_batch(SEED, 0, rows, B, L, 1.05, True, mine)
    key0, _ = layout(rows[mine], D)
    pooled = torch.from_numpy(embbag_reference(SEED, 0, key0, idx, D))
    got = exchange_pooled(pooled, groups, rank, world)
    # the global reference for this rank's samples, tables in global order
    full_idx = make_batch(SEED, 0, rows, B, L, 1.05, True)
    out = np.zeros((B, 26, D), dtype=np.float32)
    for g in range(world):
        k0, _ = layout(rows[groups[g]], D)
        out[:, groups[g]] = embbag_reference(SEED, 0, k0, full_idx[:, groups[g]], D)
    exp = out[rank * (B // world):(rank + 1) * (B // world)]
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
