"""CPU: the config tree and key = value format behave like the reference's (config.py:151-230)."""

import json
import os

import pytest

from paper_2504_19365_b200.config import (ExperimentConfig, SystemConfig, apply_overrides, config_text,
                                          parse_config_file)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))["config"]
B200_KEYS = ("device.emulation", "cache.ways", "engine.warps", "engine.side_warps", "engine.copy", "service.side_warps", "backend",
             "dlrm_", "graph_", "pagerank_")


def _ref_lines(text):
    return [l for l in text.splitlines() if l]


def _ours_filtered(text):
    return [l for l in text.splitlines() if l and not any(l.startswith(k) for k in B200_KEYS)]


def test_default_text_matches_reference():
    assert _ours_filtered(config_text(ExperimentConfig())) == _ref_lines(GOLD["default_text"])


def test_overrides_cast_like_reference():
    cfg = ExperimentConfig()
    apply_overrides(cfg, {"seed": "7", "device.jitter": "uniform", "cache.bytes": "65536",
                          "ctc_points": "0,0.5,1", "concurrency_points": "1,2", "debug_locks": "off",
                          "share_table.enabled": "yes", "tasks": "5", "device.per_channel_rate": "1e6"})
    assert _ours_filtered(config_text(cfg)) == _ref_lines(GOLD["override_text"])
    assert cfg.system.cache.resolved_lines(4096) == 16


@pytest.mark.parametrize("key,what", [tuple(x) for x in GOLD["bad_keys"]])
def test_unknown_keys_rejected_like_reference(key, what):
    if what == "KeyError":
        with pytest.raises(KeyError):
            apply_overrides(ExperimentConfig(), {key: "1"})


def test_b200_keys_and_file_format(tmp_path):
    p = tmp_path / "c.cfg"
    p.write_text("# comment\nseed = 3\ncache.ways = 16  # inline\ndevice.emulation = link\nengine.warps=8\n")
    cfg = apply_overrides(ExperimentConfig(), parse_config_file(p))
    assert (cfg.seed, cfg.system.cache.ways, cfg.system.device.emulation, cfg.system.engine.warps) == (3, 16, "link", 8)
    bad = tmp_path / "bad.cfg"
    bad.write_text("novalue\n")
    with pytest.raises(ValueError):
        parse_config_file(bad)
    with pytest.raises(ValueError):
        apply_overrides(ExperimentConfig(), {"debug_locks": "maybe"})


def test_system_text_is_what_the_c_abi_reads():
    t = config_text(SystemConfig())
    assert "cache.ways = 32" in t and "queues.sq_depth = 256" in t and not t.startswith("experiment")
