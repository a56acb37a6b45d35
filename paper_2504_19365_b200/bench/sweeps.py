"""Queue-geometry and cache-size sweeps over the synthetic gather (reference bench/sweeps.py).

The gather sets are drawn exactly as the reference draws them (random.Random(f"{seed}:gather")
.sample over block_pool, bench/sweeps.py:22-32), so both paths gather the same blocks; one warp =
32 tasks in lockstep (warp_size=32); compute per epoch = gathers * compute_ns_per_gather."""

from __future__ import annotations

import copy
import random

import numpy as np

from . import BenchResult
from ..system import AgileSystem, make_key


def gather_sets(cfg):
    need = cfg.tasks * cfg.epochs * cfg.gathers_per_epoch
    if need > cfg.block_pool:
        raise ValueError("block_pool smaller than the total gather count")
    draw = random.Random(f"{cfg.system.seed}:gather").sample(range(cfg.block_pool), need)
    return np.array(draw, dtype=np.int64).reshape(cfg.tasks, cfg.epochs, cfg.gathers_per_epoch)


def _run(cfg, system_cfg, mode, blocks):
    system_cfg = copy.deepcopy(system_cfg)
    system_cfg.device.num_blocks = max(system_cfg.device.num_blocks, cfg.block_pool)
    w = system_cfg.cache.ways or system_cfg.cache.lines
    if system_cfg.cache.lines % w:
        system_cfg.cache.ways = 0 if system_cfg.cache.lines < 32 else 32
        system_cfg.cache.lines = -(-system_cfg.cache.lines // 32) * 32 if system_cfg.cache.lines >= 32 else system_cfg.cache.lines
    system = AgileSystem(system_cfg)
    try:
        keys = make_key(np.zeros_like(blocks), blocks)
        r = system.run_gather(keys, cfg.tasks, cfg.epochs, cfg.gathers_per_epoch, mode == "async",
                              cfg.gathers_per_epoch * cfg.compute_ns_per_gather)
    finally:
        system.close()
    return r["t_ns"]


def run_queue_sweep(cfg, trace: bool = False) -> BenchResult:
    result = BenchResult(header=["queue_pairs", "queue_depth", "t_sync_ns", "t_async_ns", "speedup"], rows=[], info={})
    blocks = gather_sets(cfg)
    for qp in cfg.queue_pair_points:
        sc = copy.deepcopy(cfg.system)
        sc.queues.pairs_per_device = qp
        sc.queues.sq_depth = 64
        sc.queues.cq_depth = 64
        sc.cache.lines = max(sc.cache.lines, 4 * cfg.tasks * cfg.gathers_per_epoch)
        t_s = _run(cfg, sc, "sync", blocks)
        t_a = _run(cfg, sc, "async", blocks)
        result.rows.append((qp, 64, t_s, t_a, round(t_s / t_a, 6)))
    return result


def run_cache_sweep(cfg, trace: bool = False) -> BenchResult:
    result = BenchResult(header=["cache_lines", "cache_bytes", "t_sync_ns", "t_async_ns", "speedup"], rows=[], info={})
    blocks = gather_sets(cfg)
    for lines in cfg.cache_line_points:
        sc = copy.deepcopy(cfg.system)
        sc.cache.lines = lines
        sc.cache.bytes = 0
        t_s = _run(cfg, sc, "sync", blocks)
        t_a = _run(cfg, sc, "async", blocks)
        result.rows.append((lines, lines * cfg.system.device.block_size, t_s, t_a, round(t_s / t_a, 6)))
    return result
