"""Generate golden fixtures by running the REFERENCE simulator itself (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden.json and tests/golden/store.img.  The reference cannot travel to the
GPU box; these committed outputs pin the oracle (tests/test_oracle_golden.py) and, through it,
the CUDA path.  Each fixture names the reference test / survey recipe it reproduces.
"""

from __future__ import annotations

import json
import os
import random
import sys

REF = os.environ.get("AGILE_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from agile_sim.config import SystemConfig, TimingSpec  # noqa: E402
from agile_sim.lock_chain import AgileLockChain  # noqa: E402
from agile_sim.nvme_queue import (FILL, CommandContext, CompletionQueue, NvmeCommand,  # noqa: E402
                                  Opcode, SubmissionQueue, attempt_enqueue)
from agile_sim.sim_core import SimTask, Simulator, TraceRecorder  # noqa: E402
from agile_sim.software_cache import CachePolicy  # noqa: E402
from agile_sim.ssd_model import BlockStore, LatencyModel, SsdDevice  # noqa: E402
from agile_sim.system import AgileSystem  # noqa: E402
from agile_sim import audit  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def small_config(pairs=2, sq_depth=64, cq_depth=64, cache_lines=64, blocks=4096, warps=2, seed=0):
    # tests/conftest.py:17-32
    cfg = SystemConfig()
    cfg.queues.pairs_per_device = pairs
    cfg.queues.sq_depth = sq_depth
    cfg.queues.cq_depth = cq_depth
    cfg.cache.lines = cache_lines
    cfg.device.num_blocks = blocks
    cfg.service.warps = warps
    cfg.seed = seed
    return cfg


class SetAssocClock(CachePolicy):
    """SURVEY A.2 plug-in (builder-written; never modifies the reference)."""
    busy_eviction_choice = "wait"

    def __init__(self, sets):
        self.S = sets

    def bind(self, n):
        self.W = n // self.S
        self.hand = [0] * self.S
        self.ref = [0] * n

    def set_of(self, key):
        dev, blk = key
        x = ((blk & 0xFFFFFFFF) * 0x9E3779B9 + (blk >> 32) * 0x85EBCA77 + dev * 0xC2B2AE35) & 0xFFFFFFFF
        return (x * self.S) >> 32                     # oracle/cache.py:set_of (Fibonacci hashing)

    def on_hit(self, i):
        self.ref[i] = 1

    def on_insert(self, i):
        self.ref[i] = 1

    def map(self, cache, key, tries=0):
        s = self.set_of(key)
        base = s * self.W
        for _ in range(2 * self.W):
            w = self.hand[s]
            idx = base + w
            self.hand[s] = (w + 1) % self.W
            if not cache.lines[idx].available_as_victim():
                continue
            if self.ref[idx]:
                self.ref[idx] = 0
                continue
            return idx
        return None


def serialized_run(stream, lines, sets=None, blocks=256, with_bytes=False, seed_pages=None, policy=None):
    """A.1: one task, async_read + wait per request, full stack.  policy = (name, busy_choice)
    selects the reference's own plug-in through the config (system.py:23-31)."""
    cfg = small_config(pairs=2, cache_lines=lines, blocks=blocks, warps=2)
    if policy is not None:
        cfg.cache.policy, cfg.cache.busy_choice = policy
    system = AgileSystem(cfg, recorder=TraceRecorder())
    if sets is not None:
        p = SetAssocClock(sets)
        system.cache.policy = p
        p.bind(len(system.cache.lines))
    if seed_pages is not None:
        for b, payload in seed_pages.items():
            system.devices[0].store.write_block(b, payload)
    api = system.api
    got = []

    def prog(task, chain):
        buf = api.make_buf()
        for b in stream:
            yield from api.async_read(0, b, buf, chain)
            yield from api.wait(buf, chain)
            if with_bytes:
                got.append(bytes(buf.data[:16]).hex())

    system.run_workload([prog])
    system.assert_hygiene()
    recs = system.recorder.records
    outcomes = []
    for r in recs:
        if r[2] == "cache" and r[3] in ("hit", "miss"):
            outcomes.append(r[3])
    victims = [r[4][2] for r in recs if r[2] == "cache" and r[3] == "evict_reset"]
    q = audit.audit_queue_protocol(recs)
    w = audit.audit_cq_windows(recs)
    return {"outcomes": outcomes, "victims": victims, "hits": system.cache.hits,
            "misses": system.cache.misses, "enqueues": q.enqueues, "steady_rings": w["steady_rings"],
            "drain_rings": w["drain_rings"], "bytes16": got}


def device_timing():
    """tests/test_ssd_model.py:83-97, 167-182 closed forms, re-run on the reference."""
    out = {}

    def rig(par, base, rate=None, n=2):
        sim = Simulator(recorder=TraceRecorder())
        timing = TimingSpec(cmd_write_ns=0, doorbell_publish_ns=0, fetch_ns=0)
        store = BlockStore(64, block_size=8)
        lat = LatencyModel(read_base_ns=base, write_base_ns=base, per_channel_rate=rate)
        dev = SsdDevice(sim, 0, store, lat, par, timing)
        cq = CompletionQueue(sim, 0, 0, 16, doorbell_sink=dev.on_cq_doorbell)
        sq = SubmissionQueue(sim, 0, 0, 0, 16, timing, doorbell_sink=dev.on_sq_doorbell)
        dev.bind_queue_pair(sq, cq)
        chain = AgileLockChain(SimTask(0, "t0", "user_thread"))

        class S:
            data = bytearray(8)
        for blk in range(n):
            cmd = NvmeCommand(Opcode.READ, None, 0, blk, dest=S(), nbytes=8)
            gen = attempt_enqueue(sq, cmd, CommandContext(kind=FILL, dev_idx=0, blk_idx=blk), chain)
            try:
                next(gen)
            except StopIteration:
                pass
        sim.run_until_quiescent()
        return [r[0] for r in sim.recorder.by_action("ssd", "complete")]
    out["serial"] = rig(1, 10_000, n=2)
    out["eight_wide"] = rig(8, 10_000, n=8)
    out["pipelined"] = rig(1, 10_000, rate=1e6, n=4)
    return out


def windows(n):
    """tests/test_agile_service.py:53-73,178-185: completions vs ring counts."""
    system = AgileSystem(small_config(pairs=1, sq_depth=64, cq_depth=64, cache_lines=64, warps=1),
                         recorder=TraceRecorder())
    api = system.api

    def prog(task, chain):
        bufs = [api.make_buf() for _ in range(n)]
        for i in range(n):
            yield from api.async_read(0, i, bufs[i], chain)
        for b in bufs:
            yield from api.wait(b, chain)

    system.run_workload([prog])
    recs = system.recorder.records
    w = audit.audit_cq_windows(recs)
    drains = [r[4][2] - r[4][1] for r in recs if r[3] == "drain_ring"]
    return {"n": n, "steady": w["steady_rings"], "drain": w["drain_rings"], "drain_sizes": drains}


def main():
    g = {}
    rng = random.Random(1234)
    stream = [rng.randrange(64) for _ in range(2000)]
    g["a1_full_stack"] = {"stream": stream, "lines": 16, **serialized_run(stream, 16)}
    rng = random.Random(7)
    stream7 = [rng.randrange(256) for _ in range(3000)]
    g["a2_setassoc"] = {}
    for S in (1, 2, 4, 8):
        r = serialized_run(stream7, 32, sets=S, blocks=512)
        g["a2_setassoc"][str(S)] = {"outcomes": r["outcomes"], "victims": r["victims"]}
    g["a2_stream"] = stream7
    # the reference's ModuloPolicy (software_cache.py:129-143) through cache.policy = modulo
    g["a3_modulo"] = {}
    for lines in (16, 32):
        for busy in ("wait", "find_another"):
            r = serialized_run(stream7, lines, blocks=512, policy=("modulo", busy))
            g["a3_modulo"][f"{lines}_{busy}"] = {"outcomes": r["outcomes"], "victims": r["victims"]}
    # tests/test_software_cache.py:195-210 small streams through the reference test oracle
    sys.path.insert(0, os.path.join(os.path.dirname(REF), "tests"))
    from test_software_cache import _reference_clock
    g["ref_clock"] = [{"stream": s, "evictions": _reference_clock(4, s)}
                      for s in ([1, 2, 3, 4, 5], [1, 2, 3, 4, 2, 5, 6], [1, 2, 1, 3, 4, 5, 1, 6, 7, 8, 2, 9])]
    g["device_timing"] = device_timing()
    g["windows"] = [windows(n) for n in (5, 32, 40)]
    # page bytes through the full stack: written blocks come back bit-exact
    pages = {b: bytes([(b * 37 + i) & 0xFF for i in range(4096)]) for b in range(0, 200, 7)}
    r = serialized_run(list(range(0, 200, 7)) * 2, 16, with_bytes=True, seed_pages=pages)
    g["page_bytes"] = {"blocks": list(range(0, 200, 7)) * 2, "prefix16": r["bytes16"]}
    # raw image written by the reference BlockStore
    st = BlockStore(8, block_size=4096)
    st.write_block(0, b"a" * 4096)
    st.write_block(5, bytes(range(256)) * 16)
    st.save_image(os.path.join(HERE, "store.img"))
    g["image"] = {"num_blocks": 8, "written": [0, 5]}
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(g, fh)
    print("wrote", os.path.join(HERE, "golden.json"), {k: (len(v) if hasattr(v, '__len__') else v) for k, v in g.items()})


if __name__ == "__main__":
    main()


def config_golden():
    """config.py:220-230 rendering of the default tree + override/cast behaviour."""
    from agile_sim.config import ExperimentConfig, apply_overrides, config_text
    out = {"default_text": config_text(ExperimentConfig())}
    cfg = ExperimentConfig()
    apply_overrides(cfg, {"seed": "7", "device.jitter": "uniform", "cache.bytes": "65536",
                          "ctc_points": "0,0.5,1", "concurrency_points": "1,2", "debug_locks": "off",
                          "share_table.enabled": "yes", "tasks": "5", "device.per_channel_rate": "1e6"})
    out["override_text"] = config_text(cfg)
    bad = []
    for k in ("cache.nope", "nope", "device", "system.seed"):
        try:
            apply_overrides(ExperimentConfig(), {k: "1"})
            bad.append((k, "accepted"))
        except KeyError:
            bad.append((k, "KeyError"))
    out["bad_keys"] = bad
    return out


if __name__ == "__main__" and os.environ.get("AGILE_GOLDEN_CONFIG", "1") == "1":
    path = os.path.join(HERE, "golden.json")
    g = json.load(open(path))
    g["config"] = config_golden()
    json.dump(g, open(path, "w"))
    print("added config golden")
