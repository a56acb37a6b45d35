"""4 KiB random read/write bandwidth vs in-flight count (reference bench/bandwidth.py:1-90).

Each requester keeps exactly one command outstanding; requester idx issues
dev = (idx + j) % d, blk = (j * conc + idx) % num_blocks; bandwidth is sampled between the
warm-up and end checkpoints (real nanoseconds on the B200)."""

from __future__ import annotations

import copy

from . import BenchResult
from ..system import AgileSystem
from ..trace import TraceRecorder


def _measure_point(cfg, conc: int, write: bool, trace: bool):
    system_cfg = copy.deepcopy(cfg.system)
    # keep every in-flight command on its own line, with headroom (bench/bandwidth.py:49-50)
    system_cfg.cache.lines = max(system_cfg.cache.lines, 4 * conc)
    system_cfg.cache.bytes = 0
    w = system_cfg.cache.ways or system_cfg.cache.lines
    system_cfg.cache.lines = -(-system_cfg.cache.lines // w) * w
    recorder = TraceRecorder() if trace else None
    system = AgileSystem(system_cfg, recorder=recorder)
    try:
        r = system.run_loop(conc, cfg.warmup_ns, cfg.measure_ns, write=write)
        gbps = r["completions"] * system.block_size / r["window_ns"]
        rec = system.events() if trace else None
    finally:
        system.close()
    return rec, gbps


def run_rand_rw(cfg, write: bool = False, trace: bool = False) -> BenchResult:
    result = BenchResult(header=["concurrent_requests", "num_devices", "gb_per_s"], rows=[], info={})
    d = cfg.system.num_devices
    for conc in cfg.concurrency_points:
        rec, gbps = _measure_point(cfg, conc, write, trace)
        result.rows.append((conc, d, round(gbps, 6)))
        if trace:
            result.traces.append((f"conc{conc}", rec))
    return result


def run_rand_read(cfg, trace: bool = False) -> BenchResult:
    return run_rand_rw(cfg, write=False, trace=trace)


def run_rand_write(cfg, trace: bool = False) -> BenchResult:
    return run_rand_rw(cfg, write=True, trace=trace)
