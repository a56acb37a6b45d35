"""Serialized cache-sequence oracle (test infrastructure only).

Restates, for one task issuing ``async_read`` + ``wait`` per request, the reference
cache's observable sequence:
  * lookup through ``tag_index`` -> HIT sets the ref bit (software_cache.py:428-434, 103-107);
  * miss -> ``ClockPolicy.map`` victim (software_cache.py:109-126): the hand sweeps, skipping
    unavailable lines, clearing ref bits, returning the first line with ref 0; a READY victim is
    reset (evict_reset, software_cache.py:339-346) and the new block inserted with ref 1.
The set-associative generalisation is SURVEY A.2's plug-in with a Fibonacci set index:
set = ((blk * 0x9E3779B9 + (blk >> 32) * 0x85EBCA77 + dev * 0xC2B2AE35) mod 2^32) * S >> 32 (SURVEY A.2 used the low bits of a
32-bit multiplicative hash, which fold strided block ids onto a few sets), one hand per set, sweep
restricted to the set's ways.
With S = 1 it is the reference's built-in clock.  In serialized mode no line is ever BUSY at
access time, so every line is available to the sweep.
"""

from __future__ import annotations


def set_of(dev: int, blk: int, num_sets: int) -> int:
    """Fibonacci hashing: x = blk * 2^32/phi (+ high block bits and device) mod 2^32, scaled to
    [0, S) by a multiply-high.  Arithmetic progressions of block ids (sequential epochs, strided pages) land
    with near-minimal discrepancy, so sets fill evenly."""
    x = ((blk & 0xFFFFFFFF) * 0x9E3779B9 + (blk >> 32) * 0x85EBCA77 + dev * 0xC2B2AE35) & 0xFFFFFFFF
    return (x * num_sets) >> 32


def clock_sequence(accesses, lines: int, ways: int | None = None):
    """accesses: iterable of (dev, blk).  Returns (outcomes, victims): outcome 'hit'/'miss' per
    access; victims = list of (index_of_access, (dev, blk)) for every READY line evicted."""
    ways = lines if not ways else ways
    assert lines % ways == 0
    sets = lines // ways
    slot = [None] * lines
    ref = [0] * lines
    hand = [0] * sets
    where = {}
    outcomes, victims = [], []
    for i, key in enumerate(accesses):
        key = (int(key[0]), int(key[1]))
        li = where.get(key)
        if li is not None:
            ref[li] = 1
            outcomes.append("hit")
            continue
        outcomes.append("miss")
        s = set_of(key[0], key[1], sets)
        base = s * ways
        chosen = None
        for _ in range(2 * ways):
            w = hand[s]
            hand[s] = (w + 1) % ways
            if ref[base + w]:
                ref[base + w] = 0
                continue
            chosen = base + w
            break
        if chosen is None:   # unreachable in serialized mode (every line available)
            raise AssertionError("no victim")
        old = slot[chosen]
        if old is not None:
            victims.append((i, old))
            del where[old]
        slot[chosen] = key
        where[key] = chosen
        ref[chosen] = 1
    return outcomes, victims


def reference_clock(cache_size: int, accesses):
    """Independent hand-simulation of the reference's test oracle
    (tests/test_software_cache.py:164-185): eviction sequence of a fully associative clock."""
    _, v = clock_sequence([(0, b) for b in accesses], cache_size, cache_size)
    return [k[1] for _, k in v]


def modulo_sequence(accesses, lines: int, ways: int | None = None):
    """ModuloPolicy (software_cache.py:129-143) per set: a miss of (dev, blk) evicts way
    (dev * 7919 + blk) mod W of the key's set (set_of above; with one set, W = lines, this is the
    reference's direct-mapped placement over the whole cache).  Serialized mode: the home way is
    always available, so busy_eviction_choice never matters.  Same return shape as
    clock_sequence."""
    ways = lines if not ways else ways
    assert lines % ways == 0
    sets = lines // ways
    slot = [None] * lines
    where = {}
    outcomes, victims = [], []
    for i, key in enumerate(accesses):
        key = (int(key[0]), int(key[1]))
        if key in where:
            outcomes.append("hit")
            continue
        outcomes.append("miss")
        chosen = set_of(key[0], key[1], sets) * ways + (key[0] * 7919 + key[1]) % ways
        old = slot[chosen]
        if old is not None:
            victims.append((i, old))
            del where[old]
        slot[chosen] = key
        where[key] = chosen
    return outcomes, victims
