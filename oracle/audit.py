"""Trace-invariant audits over (t, who, module, action, details) records — test infrastructure.

Restates the reference's audits (audit.py:25-175) so that GPU event logs rendered by
``paper_2504_19365_b200.trace.render_event_log`` are checked against the same invariants:
exactly-once queue pipeline and CID uniqueness (audit.py:25-78), 32-entry CQ windows with drain
rings only after stop (81-101), allowed cache-state closure (104-123), single in-flight fill per
block (126-145), and device read/write counts (148-175).
"""

from __future__ import annotations

from collections import Counter, defaultdict

ALLOWED = {("INVALID", "BUSY"), ("BUSY", "READY"), ("READY", "MODIFIED"),
           ("MODIFIED", "BUSY"), ("BUSY", "INVALID"), ("READY", "INVALID")}


def queue_protocol(records) -> dict:
    """enqueue = issued = fetch = complete = release per SQ; a CID is issued again only after
    its release; doorbells strictly increase without gaps, each step <= depth."""
    per = defaultdict(Counter)
    live = defaultdict(set)
    last_db = {}
    for t, _who, mod, act, d in records:
        if mod == "nvme":
            if act == "enqueue":
                per[d[0]]["enqueue"] += 1
            elif act == "sqe_issued":
                sq, _slot, cid = d
                per[sq]["issued"] += 1
                if cid in live[sq]:
                    raise AssertionError(f"t={t}: cid {cid} already in flight on sq{sq}")
                live[sq].add(cid)
            elif act == "sqe_release":
                sq, _slot, cid = d
                per[sq]["release"] += 1
                if cid not in live[sq]:
                    raise AssertionError(f"t={t}: release of unknown cid {cid} on sq{sq}")
                live[sq].remove(cid)
            elif act == "doorbell":
                sq, old, new, depth = d
                per[sq]["doorbell"] += 1
                if old != last_db.get(sq, 0):
                    raise AssertionError(f"t={t}: doorbell gap on sq{sq}")
                if not new > old:
                    raise AssertionError(f"t={t}: doorbell not increasing on sq{sq}")
                if new - old > depth:
                    raise AssertionError(f"t={t}: doorbell jumped a lap on sq{sq}")
                last_db[sq] = new
        elif mod == "ssd" and act in ("fetch", "complete"):
            per[d[1]][act] += 1
    totals = Counter()
    for sq, c in per.items():
        for stage in ("issued", "fetch", "complete", "release"):
            if c[stage] != c["enqueue"]:
                raise AssertionError(f"sq{sq}: {stage} {c[stage]} != enqueues {c['enqueue']}")
        if live[sq]:
            raise AssertionError(f"sq{sq}: cids leaked {sorted(live[sq])}")
        totals.update(c)
    return {"enqueues": totals["enqueue"], "issues": totals["issued"], "fetches": totals["fetch"],
            "completions": totals["complete"], "releases": totals["release"],
            "doorbells": totals["doorbell"], "per_sq": {k: dict(v) for k, v in per.items()}}


def cq_windows(records, window: int = 32) -> dict:
    stop_seen = False
    steady = drained = 0
    for t, _who, mod, act, d in records:
        if mod != "svc":
            continue
        if act == "stop":
            stop_seen = True
        elif act == "window_ring":
            if d[2] - d[1] != window:
                raise AssertionError(f"t={t}: steady ring advanced {d[2] - d[1]}")
            steady += 1
        elif act == "drain_ring":
            if not 1 <= d[2] - d[1] < window:
                raise AssertionError(f"t={t}: drain ring advanced {d[2] - d[1]}")
            if not stop_seen:
                raise AssertionError(f"t={t}: drain ring before stop")
            drained += 1
    return {"steady_rings": steady, "drain_rings": drained}


def cache_states(records) -> int:
    n = 0
    for t, _who, mod, act, d in records:
        if mod == "cache" and act == "state":
            if (d[1], d[2]) not in ALLOWED:
                raise AssertionError(f"t={t}: illegal cache transition {d[1]} -> {d[2]}")
            n += 1
    return n


def single_fill(records) -> int:
    open_reads = Counter()
    fills = 0
    for t, _who, mod, act, d in records:
        if mod == "nvme" and act == "enqueue" and d[3] == "READ":
            key = (d[4], d[5])
            if open_reads[key]:
                raise AssertionError(f"t={t}: second concurrent fill for {key}")
            open_reads[key] += 1
            fills += 1
        elif mod == "ssd" and act == "complete" and d[3] == "READ":
            open_reads[(d[0], d[4])] -= 1
    return fills


def count_device_ops(records, op: str, dev=None, blk=None) -> int:
    n = 0
    for _t, _who, mod, act, d in records:
        if mod == "ssd" and act == "complete" and d[3] == op:
            if (dev is None or d[0] == dev) and (blk is None or d[4] == blk):
                n += 1
    return n
