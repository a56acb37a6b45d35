"""GPU: debug_locks — the device restatement of the reference's DeadlockDetector
(lock_chain.py:70-121) reports planted wait-for cycles instead of spinning into the watchdog
(reference tests/test_lock_chain.py:26-47 two-task cycle, 40-47 self re-acquire, 84-95 planted
rings), and stays silent on the normal protocol (every other GPU test runs with debug_locks on,
the reference default)."""

import pytest

from paper_2504_19365_b200 import AgileSystem, TraceRecorder
from paper_2504_19365_b200.errors import LockCycle
from conftest import small_config

pytestmark = pytest.mark.gpu


def _sys(debug=True):
    cfg = small_config(cache_lines=64, ways=8, blocks=256)
    cfg.debug_locks = debug
    return AgileSystem(cfg, recorder=TraceRecorder(), device=0)


@pytest.mark.parametrize("n", [2, 3, 5, 8])
def test_planted_ring_is_reported(n):
    with _sys() as s:
        with pytest.raises(LockCycle):
            s.lock_cycle_demo(n, 0)
        rep = s.events().by_action("lock", "deadlock")
        assert rep, "no deadlock record"
        _, _, _, _, det = rep[0]
        assert det[1] == n                           # cycle length = ring size
        assert set(det[2:2 + min(n, 4)]) <= set(range(n))   # the ring's set locks


def test_self_reacquire_is_a_one_cycle():
    with _sys() as s:
        with pytest.raises(LockCycle):
            s.lock_cycle_demo(1, 1)
        _, _, _, _, det = s.events().by_action("lock", "deadlock")[0]
        assert det[0] == 0 and det[1] == 1 and det[2] == 0   # [L0, L0]


@pytest.mark.parametrize("write", [False, True])
def test_pending_buffer_raises_buffer_busy(write):
    """AgileApi._fresh_barrier (gpu_api.py:132-137): a second transfer on a buffer whose first is
    still pending raises BufferBusy (model-mode device: the first read takes ~18 us)."""
    from paper_2504_19365_b200.errors import BufferBusy
    cfg = small_config(cache_lines=64, ways=8, blocks=256, emulation="model")
    with AgileSystem(cfg, device=0) as s:
        with pytest.raises(BufferBusy):
            s.buffer_busy_demo(write)
