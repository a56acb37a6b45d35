"""CPU: the C port of the embedding-bag path (oracle/agile_oracle.c — the reference arm and the
cpu_baseline of bench.py) pinned against the Python oracles: pooled values bit-exact with
embbag_rows_reference / embbag_reference, and single-threaded hit / miss / eviction counts equal
to the serialized set-associative clock oracle (oracle/cache.py, itself pinned to the reference
simulator's plug-in sequences in tests/golden)."""

import numpy as np
import pytest

from oracle.cache import clock_sequence
from oracle.cpu import CpuEmbeddingCache
from oracle.embbag import embbag_reference, embbag_rows_reference
from paper_2504_19365_b200.bench.dlrm import layout
from paper_2504_19365_b200.errors import OutOfRange


@pytest.mark.parametrize("lines,ways", [(256, 16), (512, 32), (64, 8)])
def test_c_port_row_keyed_matches_oracles(lines, ways):
    rng = np.random.default_rng(lines)
    rows = np.array([5000, 300, 9000], dtype=np.int64)
    key0, _ = layout(rows, 128)
    idx = np.stack([rng.integers(0, rows[t], size=(32, 20)) for t in range(3)], axis=1).astype(np.int64)
    cc = CpuEmbeddingCache(lines, ways, 7, row_dim=128)
    out = cc.embbag(idx, key0, rows, 128, threads=1)
    assert np.array_equal(out, embbag_rows_reference(7, idx, 128))
    seq = [(0, int(key0[t]) + int(idx[b, t, l]) // 8) for b in range(32) for t in range(3) for l in range(20)]
    outcomes, victims = clock_sequence(seq, lines, ways)
    st = cc.stats()
    assert st["hits"] == outcomes.count("hit") and st["misses"] == outcomes.count("miss")
    assert st["evictions"] == len(victims)
    cc.close()


def test_c_port_page_keyed_and_threads():
    rng = np.random.default_rng(3)
    rows = np.array([2000, 64], dtype=np.int64)
    key0, _ = layout(rows, 64)
    idx = np.stack([rng.integers(0, rows[t], size=(40, 7)) for t in range(2)], axis=1).astype(np.int64)
    cc = CpuEmbeddingCache(1024, 32, 5)
    assert np.array_equal(cc.embbag(idx, key0, rows, 64, threads=4), embbag_reference(5, 0, key0, idx, 64))
    idx[0, 1, 0] = 64
    with pytest.raises(OutOfRange):
        cc.embbag(idx, key0, rows, 64, threads=2)
