"""GPU parity: serialized cache sequences, page bytes and trace audits vs the oracle/golden."""

import json
import os

import numpy as np
import pytest

from oracle import audit
from oracle.cache import clock_sequence, modulo_sequence
from oracle.pages import page_bytes

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
NOVIC = np.uint64(2**64 - 1)


def _victims(vic):
    return [int(v) & ((1 << 36) - 1) for v in vic if v != NOVIC]


def test_a1_full_stack_sequence_fully_associative(gpu_system):
    g = GOLD["a1_full_stack"]
    s = gpu_system(cache_lines=16, ways=0, blocks=256)
    out, vic, _ = s.run_seq(np.zeros(len(g["stream"])), g["stream"])
    assert ["hit" if o == 0 else "miss" for o in out] == g["outcomes"]
    assert _victims(vic) == g["victims"]
    st = s.stats()
    assert st["hits"] == g["hits"] and st["misses"] == g["misses"] == st["fills"]


@pytest.mark.parametrize("sets", [1, 2, 4, 8])
def test_a2_set_associative_sequences(gpu_system, sets):
    g = GOLD["a2_setassoc"][str(sets)]
    s = gpu_system(cache_lines=32, ways=32 // sets, blocks=512)
    out, vic, _ = s.run_seq(np.zeros(len(GOLD["a2_stream"])), GOLD["a2_stream"])
    assert ["hit" if o == 0 else "miss" for o in out] == g["outcomes"]
    assert _victims(vic) == g["victims"]


@pytest.mark.parametrize("case", ["16_wait", "16_find_another", "32_wait", "32_find_another"])
def test_a3_modulo_policy_sequences(gpu_system, case):
    """cache.policy = modulo with one set (ways = lines): the reference's ModuloPolicy exactly."""
    g = GOLD["a3_modulo"][case]
    lines, busy = int(case.split("_")[0]), case.split("_", 1)[1]
    s = gpu_system(cache_lines=lines, ways=lines, blocks=512, policy="modulo", busy_choice=busy)
    out, vic, _ = s.run_seq(np.zeros(len(GOLD["a2_stream"])), GOLD["a2_stream"])
    assert ["hit" if o == 0 else "miss" for o in out] == g["outcomes"]
    assert _victims(vic) == g["victims"]


@pytest.mark.parametrize("ways", [8, 32, 64])
def test_modulo_policy_set_associative_vs_oracle(gpu_system, ways):
    rng = np.random.default_rng(ways + 1)
    blk = rng.integers(0, 3000, size=3000)
    s = gpu_system(cache_lines=512, ways=ways, blocks=4096, pairs=4, policy="modulo", busy_choice="find_another")
    s.fill_store(0, seed=5)
    out, vic, pages = s.run_seq(np.zeros_like(blk), blk, pages=True)
    eo, ev = modulo_sequence([(0, int(b)) for b in blk], 512, ways)
    assert ["hit" if o == 0 else "miss" for o in out] == eo
    assert _victims(vic) == [k[1] for _, k in ev]
    assert np.array_equal(pages, page_bytes(5, 0, blk))


@pytest.mark.parametrize("ways", [4, 8, 16, 32])
def test_set_assoc_large_vs_oracle_with_bytes(gpu_system, ways):
    rng = np.random.default_rng(ways)
    blk = rng.integers(0, 3000, size=4000)
    s = gpu_system(cache_lines=512, ways=ways, blocks=4096, pairs=4)
    s.fill_store(0, seed=99)
    out, vic, pages = s.run_seq(np.zeros_like(blk), blk, pages=True)
    eo, ev = clock_sequence([(0, int(b)) for b in blk], 512, ways)
    assert ["hit" if o == 0 else "miss" for o in out] == eo
    assert _victims(vic) == [k[1] for _, k in ev]
    assert np.array_equal(pages, page_bytes(99, 0, blk))


def test_page_bytes_written_blocks_round_trip(gpu_system):
    g = GOLD["page_bytes"]
    s = gpu_system(cache_lines=16, ways=0, blocks=256)
    for b in set(g["blocks"]):
        s.devices[0].store.write_block(b, bytes([(b * 37 + i) & 0xFF for i in range(4096)]))
    _, _, pages = s.run_seq(np.zeros(len(g["blocks"])), g["blocks"], pages=True)
    assert [bytes(p[:16]).hex() for p in pages] == g["prefix16"]


def test_image_load_matches_reference_blockstore(gpu_system, tmp_path):
    s = gpu_system(cache_lines=16, ways=0, blocks=8)
    s.load_image(0, os.path.join(os.path.dirname(__file__), "golden", "store.img"))
    _, _, pages = s.run_seq(np.zeros(8), np.arange(8), pages=True)
    assert bytes(pages[0]) == b"a" * 4096
    assert bytes(pages[5]) == bytes(range(256)) * 16
    assert not pages[3].any() and not pages[7].any()
    p = tmp_path / "out.img"
    s.save_image(0, p)
    assert p.read_bytes() == open(os.path.join(os.path.dirname(__file__), "golden", "store.img"), "rb").read()


def test_trace_audits_on_serialized_run(gpu_system):
    g = GOLD["a1_full_stack"]
    s = gpu_system(cache_lines=16, ways=0, blocks=256, trace=True)
    s.run_seq(np.zeros(len(g["stream"])), g["stream"])
    recs = s.events().records
    q = audit.queue_protocol(recs)
    assert q["enqueues"] == g["enqueues"] == q["completions"] == q["releases"]
    w = audit.cq_windows(recs)
    assert (w["steady_rings"], w["drain_rings"]) == (g["steady_rings"], g["drain_rings"])
    assert audit.cache_states(recs) > 0
    assert audit.single_fill(recs) == g["misses"]
    victims = [r[4][2] for r in recs if r[2] == "cache" and r[3] == "evict_reset"]
    assert victims == g["victims"]
