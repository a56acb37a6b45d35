import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box)")


def small_config(**kw):
    """Desk geometry mirroring the reference's tests/conftest.py:17-32 (+ B200 keys)."""
    from paper_2504_19365_b200 import SystemConfig
    cfg = SystemConfig()
    cfg.num_devices = kw.pop("num_devices", 1)
    cfg.queues.pairs_per_device = kw.pop("pairs", 2)
    cfg.queues.sq_depth = kw.pop("sq_depth", 64)
    cfg.queues.cq_depth = kw.pop("cq_depth", 64)
    cfg.cache.lines = kw.pop("cache_lines", 64)
    cfg.cache.ways = kw.pop("ways", 0)
    cfg.device.num_blocks = kw.pop("blocks", 4096)
    cfg.device.emulation = kw.pop("emulation", "link")
    cfg.service.warps = kw.pop("warps", 2)
    cfg.engine.warps = kw.pop("engine_warps", 4)
    cfg.seed = kw.pop("seed", 0)
    cfg.cache.policy = kw.pop("policy", "clock")
    cfg.cache.busy_choice = kw.pop("busy_choice", "wait")
    for k, v in kw.items():
        setattr(cfg, k, v)
    return cfg


@pytest.fixture
def gpu_system():
    from paper_2504_19365_b200 import AgileSystem, TraceRecorder
    made = []

    def make(trace=False, **kw):
        s = AgileSystem(small_config(**kw), recorder=TraceRecorder() if trace else None, device=0)
        made.append(s)
        return s
    yield make
    for s in made:
        s.close()
