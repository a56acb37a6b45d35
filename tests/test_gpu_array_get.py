"""GPU parity: AgileApi.array_get (gpu_api.py:250-278) through the cache, every element width,
non-zero offsets, hits and misses, vs the page-content oracle; reference error behaviour."""

import numpy as np
import pytest

from oracle.pages import page_bytes
from paper_2504_19365_b200.errors import OutOfRange

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("elem", [1, 2, 4, 8, 16, 64, 4096])
def test_array_get_matches_pages(gpu_system, elem):
    s = gpu_system(cache_lines=64, ways=16, blocks=512, pairs=4)
    s.fill_store(0, seed=21)
    per = 4096 // elem
    rng = np.random.default_rng(elem)
    idx = rng.integers(0, 512 * per, size=1500).astype(np.uint64)   # 512 blocks over 64 lines: misses + hits
    got = s.array_get(0, idx, elem)
    blk = (idx * elem) // 4096
    off = (idx * elem) % 4096
    pages = page_bytes(21, 0, blk)
    exp = [int.from_bytes(pages[i, off[i]:off[i] + elem].tobytes(), "little") for i in range(len(idx))]
    assert [int(x) for x in got] == exp
    # scalar form (reference signature: one element per call)
    i0 = int(idx[7])
    assert s.array_get(0, i0, elem) == exp[7]


def test_array_get_errors(gpu_system):
    s = gpu_system(cache_lines=16, ways=16, blocks=64)
    with pytest.raises(ValueError):
        s.array_get(0, 0, 3)           # element size must divide the block size
    with pytest.raises(OutOfRange):
        s.array_get(0, 64 * 1024, 4)   # block 64 of a 64-block device
    assert s.array_get(0, 64 * 1024 - 1, 4) == 0   # last element of the (zeroed) context-owned store
