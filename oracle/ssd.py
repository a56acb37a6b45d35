"""Device timing oracle (test infrastructure only): the reference SSD's FIFO channel model
(ssd_model.py:28-58, 151-206) restated as a tiny event computation for commands that all reach
the device at given times.  start_k = earliest free channel (FIFO backlog), completion =
start + service, channel held for occupancy (= service unless per_channel_rate is set)."""

from __future__ import annotations

import heapq


def completion_times(arrivals, parallelism: int, service_ns: int, per_channel_rate: float = 0.0):
    occ = max(1, int(1e9 / per_channel_rate)) if per_channel_rate else service_ns
    free = [0] * parallelism
    heapq.heapify(free)
    out = []
    for a in arrivals:
        f = heapq.heappop(free)
        start = max(a, f)
        heapq.heappush(free, start + occ)
        out.append(start + service_ns)
    return out


def plateau_gbps(parallelism: int, service_ns: int, block: int = 4096) -> float:
    """Saturated device rate: parallelism * block / service (config.py:29-31, ssd_model.py:33-36)."""
    return parallelism * block / service_ns


def cq_window_rings(n: int, window: int = 32):
    """One CQ, n completions consumed in order: full windows ring, the residue drains at stop
    (agile_service.py:147-171, 224-236)."""
    return {"steady": n // window, "drain": 1 if n % window else 0, "drain_sizes": [n % window] if n % window else []}
