"""CPU: DLRM host-side layout, index generation and sharding (the inputs every GPU rank builds)."""

import numpy as np

from paper_2504_19365_b200.bench.dlrm import (build_shard, layout, make_batch, shard_tables, table_rows,
                                              zipf_rows)


def test_table_rows_criteo_shape_and_budget():
    rows = table_rows(64 << 30)
    assert len(rows) == 26 and rows.min() >= 1
    total = rows.sum() * 128 * 4
    assert 0.97 * (64 << 30) < total <= (64 << 30)
    assert rows[2] > 1000 * rows[8]          # skew kept: a few tables hold most rows


def test_layout_is_contiguous_pages():
    rows = np.array([8, 9, 1, 16])
    key0, pages = layout(rows, 128)
    assert list(key0) == [0, 1, 3, 4] and pages == 6


def test_zipf_rows_bounded_and_skewed():
    rng = np.random.default_rng(0)
    r = zipf_rows(rng, 1000, 20000, 1.05, scatter=False)
    assert r.min() >= 0 and r.max() < 1000
    assert (r == 0).mean() > 0.05           # heavy head
    s = zipf_rows(np.random.default_rng(0), 1000, 20000, 1.05, scatter=True)
    assert sorted(np.unique(s).tolist()) != sorted(np.unique(r).tolist()) or (s != r).any()
    assert s.min() >= 0 and s.max() < 1000


def test_make_batch_rank_slices_equal_global():
    rows = table_rows(1 << 30)
    full = make_batch(3, 5, rows, 64, 20, 1.05, True)
    groups, _ = shard_tables(rows, 4)
    for g in groups:
        assert np.array_equal(make_batch(3, 5, rows, 64, 20, 1.05, True, g), full[:, g])
    assert (full < rows[None, :, None]).all()


def test_shard_tables_balanced():
    rows = table_rows(8 << 30)
    for G in (2, 4, 8):
        groups, owner = shard_tables(rows, G)
        assert sorted(np.concatenate(groups).tolist()) == list(range(26))
        load = [rows[g].sum() for g in groups]
        assert max(load) <= rows.max() + sum(load) / G
        sh = build_shard(rows, groups[0], 128)
        assert sh.pages == layout(rows[groups[0]], 128)[1]
