"""CPU: the oracle against fixtures produced by running the reference simulator itself
(tests/golden/make_golden.py)."""

import json
import os

import numpy as np
import pytest

from oracle import audit
from oracle.cache import clock_sequence, modulo_sequence, reference_clock
from oracle.pages import load_image, page_bytes, page_floats, page_words, save_image
from oracle.ssd import completion_times, cq_window_rings, plateau_gbps

HERE = os.path.dirname(__file__)
GOLD = json.load(open(os.path.join(HERE, "golden", "golden.json")))


def test_full_stack_serialized_sequence():
    g = GOLD["a1_full_stack"]
    o, v = clock_sequence([(0, b) for b in g["stream"]], g["lines"])
    assert o == g["outcomes"]
    assert [k[1] for _, k in v] == g["victims"]
    assert o.count("hit") == g["hits"] and o.count("miss") == g["misses"]


@pytest.mark.parametrize("sets", ["1", "2", "4", "8"])
def test_set_associative_plugin_sequences(sets):
    r = GOLD["a2_setassoc"][sets]
    o, v = clock_sequence([(0, b) for b in GOLD["a2_stream"]], 32, 32 // int(sets))
    assert o == r["outcomes"]
    assert [k[1] for _, k in v] == r["victims"]


@pytest.mark.parametrize("case", ["16_wait", "16_find_another", "32_wait", "32_find_another"])
def test_modulo_policy_sequences(case):
    """The reference's own ModuloPolicy (cache.policy = modulo, software_cache.py:129-143)."""
    r = GOLD["a3_modulo"][case]
    lines = int(case.split("_")[0])
    o, v = modulo_sequence([(0, b) for b in GOLD["a2_stream"]], lines, lines)
    assert o == r["outcomes"]
    assert [k[1] for _, k in v] == r["victims"]


def test_reference_test_oracle_streams():
    for case in GOLD["ref_clock"]:
        assert reference_clock(4, case["stream"]) == case["evictions"]


def test_device_timing_closed_forms():
    dt = GOLD["device_timing"]
    assert completion_times([0, 0], 1, 10_000) == dt["serial"]
    assert completion_times([0] * 8, 8, 10_000) == dt["eight_wide"]
    assert completion_times([0] * 4, 1, 10_000, per_channel_rate=1e6) == dt["pipelined"]
    assert abs(plateau_gbps(16, 17712) - 3.70) < 0.01


def test_cq_window_semantics():
    for w in GOLD["windows"]:
        r = cq_window_rings(w["n"])
        assert (r["steady"], r["drain"], r["drain_sizes"]) == (w["steady"], w["drain"], w["drain_sizes"])


def test_image_format_round_trip(tmp_path):
    img = os.path.join(HERE, "golden", "store.img")
    blocks = load_image(img, GOLD["image"]["num_blocks"])
    assert bytes(blocks[0]) == b"a" * 4096 and bytes(blocks[5]) == bytes(range(256)) * 16
    assert not blocks[3].any()
    out = tmp_path / "x.img"
    save_image(out, {0: bytes(blocks[0]), 5: bytes(blocks[5])})
    assert out.read_bytes() == open(img, "rb").read()


def test_page_words_are_deterministic_and_distinct():
    a = page_words(7, 0, [0, 1, 2])
    assert np.array_equal(a, page_words(7, 0, [0, 1, 2]))
    assert not np.array_equal(a[0], a[1])
    assert not np.array_equal(page_words(7, 1, [0]), page_words(7, 0, [0]))
    assert page_bytes(7, 0, [3]).shape == (1, 4096)
    f = page_floats(7, 0, [3])
    assert f.dtype == np.float32 and f.min() >= -1 and f.max() < 1


def test_audit_catches_violations():
    good = [(0, "u0", "nvme", "enqueue", (0, 0, 0, "READ", 0, 5)), (1, "u0", "nvme", "sqe_issued", (0, 0, 0)),
            (2, "u0", "nvme", "doorbell", (0, 0, 1, 4)), (3, "dev0", "ssd", "fetch", (0, 0, 0, 0)),
            (4, "dev0", "ssd", "complete", (0, 0, 0, "READ", 5)), (5, "svc0", "nvme", "sqe_release", (0, 0, 0))]
    assert audit.queue_protocol(good)["enqueues"] == 1
    assert audit.single_fill(good) == 1
    with pytest.raises(AssertionError):
        audit.queue_protocol(good[:-1])                       # cid leaked
    with pytest.raises(AssertionError):
        audit.queue_protocol(good + [(6, "u0", "nvme", "doorbell", (0, 2, 3, 4))])   # doorbell gap
    with pytest.raises(AssertionError):
        audit.cache_states([(0, "u", "cache", "state", (0, "INVALID", "READY", 0, 1))])
    with pytest.raises(AssertionError):
        audit.cq_windows([(0, "s", "svc", "drain_ring", (0, 0, 5))])                 # drain before stop
