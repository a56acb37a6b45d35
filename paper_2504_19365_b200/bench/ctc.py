"""Compute/communication overlap sweep on the B200 path (reference bench/ctc.py:1-111).

Same protocol as the reference: a zero-compute synchronous run calibrates communication per
epoch; each target ratio sets compute = round(ratio * comm_per_epoch) ns; synchronous mode
reads -> waits -> epoch barrier -> computes, asynchronous mode issues epoch e+1's reads before
waiting on epoch e.  Times are real device nanoseconds (%globaltimer) instead of simulated ones.
Tasks are GPU threads (the paper runs 1,024 threads in one block).
"""

from __future__ import annotations

import copy

import numpy as np

from . import BenchResult, ideal_speedup
from ..system import AgileSystem, make_key
from ..trace import TraceRecorder


def _block_for(cfg, epoch, task_idx, i):
    """Per-epoch blocks are sequential and unique (bench/ctc.py:21-24): every read misses."""
    per_epoch = cfg.tasks * cfg.reads_per_task
    return (epoch * per_epoch + task_idx * cfg.reads_per_task + i) % cfg.system.device.num_blocks


def request_keys(cfg) -> np.ndarray:
    e = np.arange(cfg.epochs).reshape(-1, 1, 1)
    t = np.arange(cfg.tasks).reshape(1, -1, 1)
    i = np.arange(cfg.reads_per_task).reshape(1, 1, -1)
    per_epoch = cfg.tasks * cfg.reads_per_task
    blk = (e * per_epoch + t * cfg.reads_per_task + i) % cfg.system.device.num_blocks
    return make_key(np.zeros_like(blk), blk)


def _run_mode(system, cfg, keys, mode, compute_ns):
    system.reset()
    r = system.run_reads(keys, cfg.tasks, cfg.reads_per_task, cfg.epochs, mode == "async", compute_ns)
    return r["t_ns"]


def run_ctc_sweep(cfg, trace: bool = False) -> BenchResult:
    result = BenchResult(header=["ctc", "t_sync_ns", "t_async_ns", "speedup", "ideal"], rows=[], info={})
    recorder = TraceRecorder() if trace else None
    system = AgileSystem(copy.deepcopy(cfg.system), recorder=recorder)
    keys = request_keys(cfg)
    try:
        base = _run_mode(system, cfg, keys, "sync", 0)
        comm_per_epoch = base / cfg.epochs
        result.info["comm_per_epoch_ns"] = comm_per_epoch
        for target in cfg.ctc_points:
            compute_ns = int(round(target * comm_per_epoch))
            t_sync = _run_mode(system, cfg, keys, "sync", compute_ns)
            t_async = _run_mode(system, cfg, keys, "async", compute_ns)
            compute_total = compute_ns * cfg.epochs
            measured = compute_total / max(1, t_sync - compute_total)
            result.rows.append((round(measured, 6), t_sync, t_async, round(t_sync / t_async, 6),
                                round(ideal_speedup(measured), 6)))
        if trace:
            result.traces.append(("ctc_sweep", system.events()))
        result.info["stats"] = system.stats()
    finally:
        system.close()
    return result
