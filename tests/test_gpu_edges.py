"""GPU edge cases the reference's tests exercise: empty inputs, out-of-range blocks and devices,
extreme queue geometry (depth 2 and 65536), configuration errors, duplicate keys in one warp."""

import numpy as np
import pytest
import torch

from oracle.cache import clock_sequence
from oracle.pages import page_bytes
from paper_2504_19365_b200 import AgileSystem
from paper_2504_19365_b200.errors import OutOfRange
from conftest import small_config

pytestmark = pytest.mark.gpu


def test_empty_inputs_are_no_ops(gpu_system):
    s = gpu_system(cache_lines=64, ways=16, blocks=256)
    z32, z64 = np.zeros(0, np.uint32), np.zeros(0, np.uint64)
    out, vic, _ = s.run_seq(z32, z64)
    assert len(out) == 0 and len(vic) == 0
    assert len(s.evict_blocks(z32, z64)) == 0
    s.write_blocks(z32, z64, np.zeros((0, 4096), np.uint8))
    assert len(s.array_get(0, np.zeros(0, np.uint64))) == 0
    st = s.stats()
    assert st["misses"] == st["hits"] == st["fills"] == 0


def test_out_of_range_block_and_device(gpu_system):
    s = gpu_system(num_devices=2, cache_lines=64, ways=16, blocks=128)
    with pytest.raises(OutOfRange):
        s.run_seq(np.zeros(1), np.array([128]))            # ssd_model.py:24 / gpu_api.py:122-126
    with pytest.raises(OutOfRange):
        s.run_seq(np.array([2]), np.array([0]))            # no device 2
    out, _, _ = s.run_seq(np.array([1]), np.array([127]))  # the last block of the last device
    assert list(out) == [1]


@pytest.mark.parametrize("depth", [2, 65536])
def test_extreme_queue_depths(gpu_system, depth):
    s = gpu_system(pairs=1, sq_depth=depth, cq_depth=depth, cache_lines=64, ways=16, blocks=512)
    s.fill_store(0, seed=3)
    blk = np.random.default_rng(depth).integers(0, 512, size=300)
    out, vic, pages = s.run_seq(np.zeros_like(blk), blk, pages=True)
    eo, _ = clock_sequence([(0, int(b)) for b in blk], 64, 16)
    assert ["hit" if o == 0 else "miss" for o in out] == eo
    assert np.array_equal(pages, page_bytes(3, 0, blk))


@pytest.mark.parametrize("key,value", [("queues.sq_depth", 48), ("queues.cq_depth", 1), ("cache.ways", 24),
                                       ("cache.policy", "lru"), ("cache.busy_choice", "spin"),
                                       ("engine.copy", "dma"), ("share_table.buckets", 3)])
def test_bad_geometry_is_a_config_error(key, value):
    cfg = small_config(cache_lines=64)
    sec, name = key.split(".")
    setattr(getattr(cfg, sec), name, value)
    if key == "share_table.buckets":
        cfg.share_table.enabled = True
    with pytest.raises(ValueError):
        AgileSystem(cfg, device=0)


def test_duplicate_keys_in_one_warp_read_once(gpu_system):
    """32 lanes asking for 4 distinct blocks: every lane gets its element, 4 device reads."""
    s = gpu_system(cache_lines=64, ways=16, blocks=256, trace=True)
    s.fill_store(0, seed=12)
    idx = np.repeat(np.array([5, 9, 200, 33], dtype=np.uint64) * 1024 + 7, 8)
    got = s.array_get(0, idx, 4)
    pb = page_bytes(12, 0, idx // 1024)
    exp = [int.from_bytes(pb[i, 28:32].tobytes(), "little") for i in range(len(idx))]
    assert [int(x) for x in got] == exp
    from oracle import audit
    assert audit.count_device_ops(s.events().records, "READ") == 4
