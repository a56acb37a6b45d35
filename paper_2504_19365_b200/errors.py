"""Exception types of the reference, raised from device-side error words of the B200 path.

Names and bases follow the reference so callers' ``except`` clauses keep working:
ProtocolViolation (nvme_queue.py:23), UnknownCid (agile_service.py:27), OutOfRange
(ssd_model.py:24), IllegalState (software_cache.py:26), LivelockSuspected (sim_core.py:23),
BufferBusy (gpu_api.py:21).
"""

from __future__ import annotations


class AgileError(RuntimeError):
    """Base for failures reported by the native library."""


class ProtocolViolation(AgileError):
    """An illegal queue-state transition was attempted."""


class UnknownCid(ProtocolViolation):
    """A completion arrived with no matching in-flight command."""


class OutOfRange(ValueError):
    """Block index beyond the device's capacity."""


class IllegalState(AgileError):
    """A line transition that the state machine forbids."""


class LivelockSuspected(AgileError):
    """The device watchdog saw no progress within the budget."""


class LockCycle(LivelockSuspected):
    """debug_locks found a wait-for cycle (the DeadlockDetector report, lock_chain.py:70-121)."""


class BufferBusy(AgileError):
    """Buffer reused while its previous transfer is still pending."""


class NativeUnavailable(AgileError):
    """The CUDA extension is missing or no GPU is visible (there is no CPU fallback)."""


CODE_TO_EXC = {
    -1: AgileError,
    -2: ValueError,
    -3: ValueError,
    -101: ProtocolViolation,
    -102: UnknownCid,
    -103: OutOfRange,
    -104: IllegalState,
    -105: LivelockSuspected,
    -106: BufferBusy,
    -107: LockCycle,
}
