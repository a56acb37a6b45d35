"""GPU write path: AgileApi.async_write with eager write-back
(gpu_api.py:192-227, SoftwareCache._try_write / _install_locked / _allocate_locked,
software_cache.py:458-523): bytes land in the block's cache line, the device write starts at
once, and the line is READY again once durable.  Checked against the reference's own tests:
write -> evict -> device read (test_gpu_api.py:131-151), the device store round trip
(test_ssd_model.py:141-150) and the rand_write plateau parallelism * 4 KiB / write latency."""

import numpy as np
import pytest

from oracle import audit

pytestmark = pytest.mark.gpu


def _payloads(rng, n):
    return rng.integers(0, 256, size=(n, 4096), dtype=np.uint8)


def test_write_then_read_back_and_device_store(gpu_system):
    s = gpu_system(cache_lines=64, ways=16, blocks=1 << 12, pairs=4, engine_warps=4, warps=2)
    s.fill_store(0, seed=1)
    rng = np.random.default_rng(0)
    blk = rng.choice(4096, size=300, replace=False).astype(np.uint64)
    pay = _payloads(rng, len(blk))
    s.write_blocks(np.zeros(len(blk)), blk, pay)
    store = s.store_view(0)
    assert np.array_equal(store[blk.astype(np.int64)], pay)       # durable on the device
    # read back through the cache: 64 lines for 300 blocks -> hits on the last ones, misses
    # (device reads of the written bytes) on the rest
    _, _, pages = s.run_seq(np.zeros(len(blk)), blk, pages=True)
    assert np.array_equal(pages, pay)


def test_overwrite_resident_line(gpu_system):
    s = gpu_system(cache_lines=32, ways=32, blocks=256, pairs=2, engine_warps=4, warps=2)
    s.fill_store(0, seed=2)
    blk = np.arange(8, dtype=np.uint64)
    s.run_seq(np.zeros(8), blk)                                   # resident, READY
    rng = np.random.default_rng(1)
    pay = _payloads(rng, 8)
    hits0 = s.stats()["hits"]
    s.write_blocks(np.zeros(8), blk, pay)
    out, _, pages = s.run_seq(np.zeros(8), blk, pages=True)
    assert list(out) == [0] * 8                                   # still resident: hits
    assert np.array_equal(pages, pay)
    assert np.array_equal(s.store_view(0)[:8], pay)
    assert s.stats()["writebacks"] >= 8 and s.stats()["hits"] > hits0


def test_same_block_twice_in_one_warp_last_lane_wins(gpu_system):
    s = gpu_system(cache_lines=32, ways=32, blocks=256, pairs=2, engine_warps=4, warps=2)
    s.fill_store(0, seed=3)
    blk = np.array([5, 9, 5, 5], dtype=np.uint64)
    pay = _payloads(np.random.default_rng(2), 4)
    s.write_blocks(np.zeros(4), blk, pay)
    assert np.array_equal(s.store_view(0)[5], pay[3])
    assert np.array_equal(s.store_view(0)[9], pay[1])


def test_write_audits_exactly_once(gpu_system):
    """Traced concurrent writes: every WRITE command enqueued, issued, fetched, completed and
    released exactly once; cache states follow the reference's transitions."""
    s = gpu_system(cache_lines=128, ways=16, blocks=1 << 12, pairs=4, sq_depth=8, cq_depth=8,
                   engine_warps=4, warps=2, trace=True)
    s.fill_store(0, seed=4)
    rng = np.random.default_rng(3)
    blk = rng.choice(4096, size=1000, replace=False).astype(np.uint64)
    s.write_blocks(np.zeros(len(blk)), blk, _payloads(rng, len(blk)))
    recs = s.events().records
    q = audit.queue_protocol(recs)
    assert q["enqueues"] == len(blk)
    assert q["fetches"] == q["completions"] == q["releases"] == q["issues"] == q["enqueues"]
    audit.cache_states(recs)
    assert sum(1 for r in recs if r[2] == "cache" and r[3] == "install") == len(blk)


def test_rand_write_model_plateau(gpu_system):
    """Closed-loop writers in model mode saturate parallelism * 4 KiB / write_latency
    (2.2 GB/s at the reference defaults: 16 channels, 29,789 ns)."""
    s = gpu_system(pairs=8, sq_depth=256, cq_depth=256, cache_lines=4096, ways=32, blocks=1 << 16,
                   emulation="model", engine_warps=16, warps=4)
    s.fill_store(0, seed=5)
    r = s.run_loop(512, warmup_ns=2_000_000, measure_ns=20_000_000, write=True)
    gbps = r["completions"] * 4096 / r["window_ns"]
    ceiling = 16 * 4096 / 29789
    assert ceiling * 0.95 <= gbps <= ceiling * 1.02, (gbps, ceiling)   # window-edge completions


def test_write_evict_then_device_read(gpu_system):
    """test_gpu_api.py:131-151: write a block, evict it, read it back — the read misses and
    returns the written bytes from the device."""
    s = gpu_system(cache_lines=64, ways=16, blocks=1024, pairs=2, engine_warps=4, warps=2)
    s.fill_store(0, seed=7)
    blk = np.array([3, 77, 500], dtype=np.uint64)
    pay = _payloads(np.random.default_rng(8), 3)
    s.write_blocks(np.zeros(3), blk, pay)
    assert list(s.evict_blocks(np.zeros(3), blk)) == [0, 0, 0]           # RESET
    assert list(s.evict_blocks(np.zeros(3), blk)) == [2, 2, 2]           # no longer resident
    out, _, pages = s.run_seq(np.zeros(3), blk, pages=True)
    assert list(out) == [1, 1, 1]                                         # misses: device reads
    assert np.array_equal(pages, pay)
