"""GPU port of the reference's coherence equivalence tests (tests/test_coherence.py:68-171):
concurrent tasks read and write a few blocks through the share table (share_table.py) and the
cache's MODIFIED lines; the device event log (install / write_commit / observe records, in an
order consistent with every commit) is replayed against the sequential oracle, and the flushed
device must end at each block's last committed value.  Same plans as the reference (its seeded
generator), same desk geometry (tests/conftest.py small_config)."""

import random

import numpy as np
import pytest

from conftest import small_config
from paper_2504_19365_b200 import AgileSystem, TraceRecorder

pytestmark = pytest.mark.gpu


def _plans(seed, n_tasks, n_blocks, ops_per_task):
    # test_coherence.py:27-33: one seeded generator, plans drawn task by task
    rng = random.Random(f"{seed}:coherence")
    plans = [[(rng.choice(("read", "write")), rng.randrange(n_blocks), rng.randrange(0, 4000))
              for _ in range(ops_per_task)] for _ in range(n_tasks)]
    op = np.array([[1 if o == "write" else 0 for o, _, _ in p] for p in plans], dtype=np.uint8)
    blk = np.array([[b for _, b, _ in p] for p in plans], dtype=np.uint32)
    think = np.array([[t for _, _, t in p] for p in plans], dtype=np.uint32)
    return op, blk, think


def replay_check(records, n_blocks):
    """test_coherence.py:62-77: every observe sees the last commit before it."""
    last = {b: 0 for b in range(n_blocks)}
    bad = []
    for t, who, module, action, det in records:
        if (module, action) in (("cache", "install"), ("api", "write_commit")):
            last[det[1]] = det[2]
        elif (module, action) == ("test", "observe"):
            if det[2] != last[det[1]]:
                bad.append((t, det[1], det[2], last[det[1]]))
    return bad


def final_state_check(s, records, n_blocks):
    last = {b: 0 for b in range(n_blocks)}
    for t, who, module, action, det in records:
        if (module, action) in (("cache", "install"), ("api", "write_commit")):
            last[det[1]] = det[2]
    view = s.store_view(0).reshape(-1, 4096)
    return [(b, int(view[b, :8].view(np.uint64)[0]), last[b]) for b in range(n_blocks)
            if int(view[b, :8].view(np.uint64)[0]) != last[b]]


def _run(seed, table_on, n_tasks=4, n_blocks=4, ops=8, cache_lines=32, blocks=64):
    cfg = small_config(pairs=2, cache_lines=cache_lines, blocks=blocks, warps=2, seed=seed)
    cfg.share_table.enabled = table_on
    s = AgileSystem(cfg, recorder=TraceRecorder(), device=0)
    op, blk, think = _plans(seed, n_tasks, n_blocks, ops)
    seen, flushed = s.run_coherence(op, blk, think)
    recs = s.events().records
    return s, recs, seen, flushed


def test_share_table_runs_match_sequential_oracle_sample():
    for seed in range(24):
        s, recs, _, _ = _run(seed, True)
        try:
            assert replay_check(recs, 4) == [], f"seed {seed}: stale reads"
            assert final_state_check(s, recs, 4) == [], f"seed {seed}: device state"
            assert s.share_live() == 0
        finally:
            s.close()


def test_writeback_completeness_holds_even_without_the_table():
    for seed in range(12):
        s, recs, _, _ = _run(seed, False)
        try:
            assert final_state_check(s, recs, 4) == [], f"seed {seed}"
        finally:
            s.close()


@pytest.mark.parametrize("table_on", [True, False])
def test_coherence_under_eviction_pressure(table_on):
    """More blocks than cache lines: MODIFIED lines are written back on eviction (WB_EVICT) before
    their line is reused; observes and the final device still replay the commit order."""
    for seed in range(6):
        s, recs, _, flushed = _run(seed, table_on, n_tasks=8, n_blocks=48, ops=12, cache_lines=8, blocks=64)
        try:
            if table_on:
                assert replay_check(recs, 48) == [], f"seed {seed}"
                assert s.share_live() == 0
            assert final_state_check(s, recs, 48) == [], f"seed {seed}"
        finally:
            s.close()


def _hazard(seed, table_on):
    # test_coherence.py:112-141: a direct-buffer read racing a cache-path write on block 0
    rng = random.Random(f"{seed}:hazard")
    d_read = rng.randrange(1, 60_000)
    d_write = rng.randrange(1, 60_000)
    cfg = small_config(pairs=1, cache_lines=16, blocks=16, warps=1, seed=seed)
    cfg.share_table.enabled = table_on
    with AgileSystem(cfg, recorder=TraceRecorder(), device=0) as s:
        op = np.array([[2], [1]], dtype=np.uint8)
        blk = np.zeros((2, 1), dtype=np.uint32)
        think = np.array([[d_read], [d_write]], dtype=np.uint32)
        s.run_coherence(op, blk, think)
        return replay_check(s.events().records, 1)


def test_disabled_table_exhibits_the_raw_hazard():
    assert [sd for sd in range(40) if _hazard(sd, False)], "no seed exhibited a stale read without the table"


def test_enabled_table_masks_the_hazard_on_every_seed():
    for seed in range(40):
        assert _hazard(seed, True) == [], f"seed {seed}"
