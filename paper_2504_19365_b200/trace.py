"""Trace recorder and the K10 device event-log renderer.

``TraceRecorder`` keeps the reference's structured records ``(time, who, module, action,
details)`` and its text form ``<time_ns> <task> <module> <action> <details>`` (reference
``sim_core.py:162-191``).  ``render_event_log`` turns the 64-byte device records written by the
kernels' ``log_ev`` into exactly those tuples (same module/action names and detail arities), so
the reference's trace audits run unchanged over a GPU run.
"""

from __future__ import annotations

import numpy as np

MODULES = ("nvme", "ssd", "svc", "cache", "api", "table", "test", "lock")
ACTIONS = ("enqueue", "sqe_updated", "sqe_issued", "doorbell", "sqe_release", "head",
           "fetch", "complete", "cqe_post", "cqe_stall",
           "window_ring", "drain_ring", "stop", "start", "cqe_process",
           "state", "miss", "hit", "attach", "evict_reset", "drain", "async_read", "prefetch", "install",
           "write_commit", "observe", "register", "share", "release", "modified", "propagate", "duty_transfer",
           "evict_wb", "write_intent", "deadlock")
STATES = ("INVALID", "BUSY", "READY", "MODIFIED")
OPS = ("READ", "WRITE")
ARITY = {"enqueue": 6, "sqe_updated": 2, "sqe_issued": 3, "doorbell": 4, "sqe_release": 3,
         "head": 2, "fetch": 4, "complete": 5, "cqe_post": 4, "cqe_stall": 3,
         "window_ring": 3, "drain_ring": 3, "stop": 0, "start": 1, "cqe_process": 4,
         "state": 5, "miss": 2, "hit": 2, "attach": 2, "evict_reset": 3, "drain": 2,
         "async_read": 2, "prefetch": 2, "install": 3,
         "write_commit": 3, "observe": 3, "register": 2, "share": 4, "release": 3, "modified": 2, "propagate": 2,
         "duty_transfer": 3, "evict_wb": 3, "write_intent": 2, "deadlock": 6}
SHARE_STATES = ("Exclusive", "Shared", "Modified")

RECORD = np.dtype([("t", "<u8"), ("who", "<u4"), ("modact", "<u4"), ("a", "<u8", (6,))])


class TraceRecorder:
    """Collects (time, who, module, action, details) tuples."""

    __slots__ = ("records",)

    def __init__(self):
        self.records = []

    def emit(self, t, who, module, action, details):
        self.records.append((t, who, module, action, details))

    def lines(self):
        for t, who, module, action, details in self.records:
            tail = " ".join(str(d) for d in details)
            yield f"{t} {who} {module} {action} {tail}".rstrip()

    def text(self) -> str:
        return "\n".join(self.lines()) + "\n"

    def dump(self, path) -> None:
        with open(path, "w") as fh:
            for line in self.lines():
                fh.write(line + "\n")

    def by_action(self, module, action):
        return [r for r in self.records if r[2] == module and r[3] == action]


def _who(code: int) -> str:
    role, idx = code >> 30, code & ((1 << 30) - 1)
    return ("u", "svc", "dev", "host")[role] + str(idx)


def render_event_log(raw: bytes | np.ndarray, recorder: TraceRecorder | None = None) -> TraceRecorder:
    """Decode device records (in log order, which respects causality) into reference tuples."""
    rec = recorder if recorder is not None else TraceRecorder()
    arr = np.frombuffer(raw, dtype=RECORD) if not isinstance(raw, np.ndarray) else raw.view(RECORD)
    if len(arr) == 0:
        return rec
    t0 = int(arr["t"].min())
    for r in arr:
        mod = MODULES[int(r["modact"]) & 0xFF]
        act = ACTIONS[int(r["modact"]) >> 8]
        a = [int(x) for x in r["a"]]
        n = ARITY[act]
        det = a[:n]
        if act == "enqueue":
            det[3] = OPS[det[3]]
        elif act == "complete":
            det[3] = OPS[det[3]]
        elif act == "state":
            det[1] = STATES[det[1]]
            det[2] = STATES[det[2]]
        elif act == "share":
            det[3] = SHARE_STATES[det[3]]
        rec.emit(int(r["t"]) - t0, _who(int(r["who"])), mod, act, tuple(det))
    return rec
