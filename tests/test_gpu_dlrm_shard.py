"""GPU: sharded DLRM (BASELINE configs[4]) on one B200, rank by rank.

Every rank of a G-way TWRW plan (bench/dlrm.py plan_shards) gets its own context (cache, queue
pairs, service, engine, page store holding only its pieces) on cuda:0; K5 writes each rank's
pooled rows straight into its peer-major send buffer; the all_to_all_single is replayed on the
host (recv of rank p = block p of every rank's send buffer, in rank order) and combine() adds the
row-wise partials.  The exchanged result must equal the single-device oracle bit for bit.
Also: variable-length bags (offsets), out-of-range indices, and the kernel's byte layout."""

import numpy as np
import pytest
import torch

from oracle.embbag import embbag_offsets_reference, embbag_rows_reference
from paper_2504_19365_b200 import AgileSystem
from paper_2504_19365_b200.errors import OutOfRange
from paper_2504_19365_b200.bench.dlrm import (combine, fill_rank_store, make_batch, plan_shards,
                                              pool_rank_reference, table_rows)
from conftest import small_config

pytestmark = pytest.mark.gpu
SEED, B, L, D = 77, 64, 20, 128
DEV = torch.device("cuda", 0)


def _rank_system(pages, cache_frac=0.25):
    lines = max(256, int(pages * cache_frac) // 32 * 32)
    cfg = small_config(cache_lines=lines, ways=32, blocks=max(pages, 64), pairs=8, sq_depth=256, cq_depth=256,
                       engine_warps=8, warps=4)
    return AgileSystem(cfg, device=0)


def _pool_rank(plan, rank, idx, pd=0):
    descs, _, pages = plan.rank_layout(rank)
    with _rank_system(pages) as s:
        fill_rank_store(s, plan, rank, SEED)
        out = torch.full((B, plan.row_bytes(rank)), 0xAB, dtype=torch.uint8, device=DEV)
        cnt = torch.zeros(2, dtype=torch.int64, device=DEV)
        tabs = torch.from_numpy(descs.view(np.uint8).copy()).to(DEV)
        s.embbag_sharded(torch.from_numpy(idx).to(DEV), tabs, out, cnt, D, prefetch_distance=pd)
        s.sync(torch.cuda.current_stream(DEV).cuda_stream)
        return out.cpu(), cnt.cpu().numpy()


@pytest.mark.parametrize("G", [2, 4, 8])
def test_sharded_exchange_bit_exact(G):
    rows = table_rows(96 << 20, D, 26)          # 96 MiB of Criteo-shaped tables
    plan = plan_shards(rows, G, D)
    assert any(p.partial for ps in plan.pieces for p in ps), "plan should split the large tables"
    full = make_batch(SEED, 3, rows, B, L, 1.05, True)
    ref = embbag_rows_reference(SEED, full, D)
    sends, lookups = [], 0
    for r in range(G):
        idx = np.ascontiguousarray(full[:, plan.rank_tables(r)])
        out, cnt = _pool_rank(plan, r, idx, pd=r % 2)
        # the kernel's bytes are exactly the CPU restatement of the rank's output rows
        assert np.array_equal(out.numpy(), pool_rank_reference(plan, r, idx, SEED)), f"rank {r} layout"
        sends.append(out)
        lookups += int(cnt[0])
    assert lookups == B * 26 * L                # every lookup pooled exactly once, by one rank
    nl = B // G
    for p in range(G):
        recv = torch.cat([sends[q][p * nl:(p + 1) * nl].reshape(-1) for q in range(G)])
        got = combine(plan, recv, nl).numpy()
        assert np.array_equal(got, ref[p * nl:(p + 1) * nl]), f"rank {p} exchanged output differs"


def test_variable_length_bags(gpu_system):
    s = gpu_system(cache_lines=512, ways=32, blocks=1 << 12, pairs=8, sq_depth=256, cq_depth=256,
                   engine_warps=8, warps=4)
    rows = np.array([3000, 70, 9000], dtype=np.int64)
    plan = plan_shards(rows, 1, D)
    descs, first, pages = plan.rank_layout(0)
    fill_rank_store(s, plan, 0, SEED)
    rng = np.random.default_rng(5)
    Bv, T = 24, 3
    lens = rng.integers(0, 80, size=Bv * T)     # empty bags and bags of several 32-lookup chunks
    lens[:3] = [0, 32, 33]
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    tab_of = np.repeat(np.tile(plan.rank_tables(0), Bv), lens)
    flat = np.array([rng.integers(0, rows[t]) for t in tab_of], dtype=np.int64)
    out = torch.full((Bv, plan.row_bytes(0) // 4), float("nan"), dtype=torch.float32, device=DEV)
    cnt = torch.zeros(2, dtype=torch.int64, device=DEV)
    tabs = torch.from_numpy(descs.view(np.uint8).copy()).to(DEV)
    s.embbag_sharded(torch.from_numpy(flat).to(DEV), tabs, out, cnt, D, offsets=torch.from_numpy(offs).to(DEV), B=Bv)
    s.sync(torch.cuda.current_stream(DEV).cuda_stream)
    got = out.cpu().numpy().reshape(Bv, T, D)
    ref = embbag_offsets_reference(SEED, flat, offs, T, D, tables=plan.rank_tables(0))
    assert np.array_equal(got, ref)
    assert int(cnt[0].item()) == int(lens.sum())


def test_out_of_range_index_raises(gpu_system):
    s = gpu_system(cache_lines=256, ways=32, blocks=1 << 10)
    s.fill_store(0, seed=1, kind="f32")
    idx = torch.zeros((4, 2, 5), dtype=torch.int64, device=DEV)
    idx[3, 1, 2] = 500                          # table 1 has 500 rows: row 500 does not exist
    out = torch.empty((4, 2, D), dtype=torch.float32, device=DEV)
    cnt = torch.zeros(2, dtype=torch.int64, device=DEV)
    k0 = torch.tensor([0, 100], dtype=torch.int64, device=DEV)
    rows = torch.tensor([800, 500], dtype=torch.int64, device=DEV)
    with pytest.raises(OutOfRange):
        s.embbag(idx, k0, rows, out, cnt, prefetch_distance=0)
        s.sync(torch.cuda.current_stream(DEV).cuda_stream)
    idx[3, 1, 2] = -1
    s.reset()
    with pytest.raises(OutOfRange):
        s.embbag(idx, k0, rows, out, cnt, prefetch_distance=0)
        s.sync(torch.cuda.current_stream(DEV).cuda_stream)
