// agile_core.cuh — cache (K1), SQ submit (K2), completion service (K3), device engine (K4).
// All user-facing functions are warp-collective: every lane of the warp calls them, each lane
// carrying its own request (or none); the warp coalesces, probes and submits cooperatively.
#pragma once
#include <type_traits>
#include "agile_dev.cuh"
#undef SPIN_FILE_ID
#define SPIN_FILE_ID 1

// CTAs per SM the fused kernel's register budget targets (__launch_bounds__ min blocks)
#ifndef AGILE_MIN_CTAS
#define AGILE_MIN_CTAS 2
#endif

namespace agile {

constexpr u32 FULL = 0xffffffffu;
constexpr u32 NONE = 0xffffffffu;

// access outcomes (software_cache.py:37-41)
// R_WBEVICT: the chosen victim was MODIFIED; the claimant started its write-back (the line is
// BUSY with the OLD key until the write is durable, then INVALID) and must submit that WRITE
// (K_WB_EVICT) and retry (software_cache.py:348-353, 482-486)
enum : int { R_NONE = -1, R_HIT = 0, R_FILLING = 1, R_MISS = 2, R_RETRY = 3, R_WBEVICT = 4 };

struct Launch {
  u32 n_user_ctas;
  u32 pad;
};

// users_started bit set by an infra grid that gave up on a user grid that never started
constexpr u32 kInfraGaveUp = 0x80000000u;

// position of the n-th (0-based) set bit of m (n < popc(m))
__device__ __forceinline__ u32 nth_set_bit(u32 m, u32 n) {
  u32 pos = 0;
#pragma unroll
  for (int w = 16; w; w >>= 1) {
    const u32 lowmask = (1u << w) - 1u;
    const u32 lo = __popc(m & lowmask);
    if (n >= lo) { n -= lo; m >>= w; pos += w; }
    else m &= lowmask;
  }
  return pos;
}

// ======================================================================= K1: cache

// Probe one key (warp-uniform) across all ways of its set.  Relaxed loads; callers that act
// on the result re-validate (seqlock) or hold the set lock.
__device__ __forceinline__ bool probe_key_warp(const DevCtx& c, u64 key, u32& line, u64& word) {
  const u32 lane = lane_id();
  const u64 base = (u64)set_of(c, key) * c.ways;
  for (u32 w0 = 0; w0 < c.ways; w0 += 32) {
    const u32 w = w0 + lane;
    u64 tw = 0;
    bool m = false;
    if (w < c.ways) {
      tw = ld_relaxed(&c.tags[base + w]);
      m = tw_live(tw) && tw_key(tw) == key;
    }
    const u32 b = __ballot_sync(FULL, m);
    if (b) {
      const int src = __ffs(b) - 1;
      line = (u32)(base + w0 + src);
      word = __shfl_sync(FULL, tw, src);
      return true;
    }
  }
  return false;
}

// Batched warp-cooperative probe: every active lane carries a key; lanes are split into groups
// of W (one lane per way) and each group resolves one key per round with a ballot.  Returns per
// lane the matching (line, word) or line = NONE.  Used for W <= 32; larger W falls back to the
// per-key probe.
// bit 15 / bit 31 set where the low / high 16-bit half of w equals pat's (exact: the 15-bit add
// cannot carry into the next half)
__device__ __forceinline__ u32 sig_zero2(u32 w, u32 pat) {
  const u32 x = w ^ pat;
  return ~(((x & 0x7FFF7FFFu) + 0x7FFF7FFFu) | x) & 0x80008000u;
}
// bit 7 of each byte of y (bytes 0 or 0x80) -> a 4-bit mask (the multiply's partial products
// land on distinct bits, so nothing carries into bits 28..31)
__device__ __forceinline__ u32 byte_flags4(u32 y) { return (((y >> 7) & 0x01010101u) * 0x10204080u) >> 28; }
__device__ __forceinline__ u32 sig_match8(uint4 v, u32 pat) {
  // 8 x 16-bit signatures -> 8-bit match mask (way 2i = low half of word i), SWAR on the integer
  // pipe: 4 ops per word to flag equal halves, a byte permute to gather the 8 flags, one multiply
  // per 4 flags to pack them
  const u32 z0 = sig_zero2(v.x, pat), z1 = sig_zero2(v.y, pat), z2 = sig_zero2(v.z, pat), z3 = sig_zero2(v.w, pat);
  return byte_flags4(__byte_perm(z0, z1, 0x7531)) | (byte_flags4(__byte_perm(z2, z3, 0x7531)) << 4);
}

// Probe result of one lane (line = NONE: not resident)
struct ProbeRes { u64 word; u32 line; };

// Generic batched probe (W > 32, W not a multiple of 8): lanes are split into groups of W (one
// lane per way) and each group resolves one key per round with a ballot; W > 32 or W not a power
// of two go one key at a time.  Out of line: the hot paths (W a multiple of 8, <= 32) never carry
// its registers.
__device__ __noinline__ ProbeRes probe_lanes_generic(const DevCtx& c, bool active, u64 key) {
  ProbeRes res;
  res.line = NONE;
  res.word = 0;
  const u32 W = c.ways;
  const u32 lane = lane_id();
  const u32 act = __ballot_sync(FULL, active);
  if (!act) return res;
  if (W > 32 || (W & (W - 1))) {
    u32 todo = act;
    while (todo) {
      const int src = __ffs(todo) - 1;
      todo &= todo - 1;
      const u64 k = __shfl_sync(FULL, key, src);
      u32 l; u64 w;
      const bool f = probe_key_warp(c, k, l, w);
      if (lane == (u32)src && f) { res.line = l; res.word = w; }
    }
    return res;
  }
  const u32 G = 32 / W;                // keys per round
  const u32 g = lane / W, way = lane % W;
  const u32 nact = __popc(act);
  const u32 my_rank = __popc(act & lanemask_lt());
  const u32 rounds = (nact + G - 1) / G;
  const u32 gmask = (W == 32) ? FULL : ((1u << W) - 1);
  for (u32 r0 = 0; r0 < rounds; ++r0) {
    const u32 rank = r0 * G + g;
    const bool valid = rank < nact;
    const u32 src = valid ? nth_set_bit(act, rank) : 0u;
    const u64 k = __shfl_sync(FULL, key, src);
    u64 tw = 0, sb = 0;
    if (valid) {
      sb = (u64)set_of(c, k) * W;
      const u64 t = ld_relaxed(&c.tags[sb + way]);
      tw = (tw_live(t) && tw_key(t) == k) ? t : 0;
    }
    const u32 b = __ballot_sync(FULL, tw != 0);
    const bool mine = active && (my_rank / G) == r0;
    const u32 mg = my_rank % G;
    const u32 bits = (b >> (mg * W)) & gmask;
    const int hw = bits ? __ffs(bits) - 1 : 0;
    const u64 wv = __shfl_sync(FULL, tw, mg * W + hw);
    const u64 base = __shfl_sync(FULL, sb, mg * W + hw);
    if (mine && bits) { res.line = (u32)(base + hw); res.word = wv; }
  }
  return res;
}

// Lane-per-key probe.  For W a multiple of 8 and <= 32 (every production geometry) each active
// lane scans its own set's W 16-bit signatures (2W bytes, all loads in flight at once), then
// confirms candidate ways against the tag word.  kAcquire: the confirming load is an acquire
// (a READY word read here makes the line's bytes visible to the caller); false: relaxed, the
// caller orders its reads itself.  A signature lags its tag word only between a claim's CAS and
// the signature store; a probe that misses in that window takes the miss path, which re-probes
// the full tags under the set lock, so in-flight de-duplication is unaffected.  Warp-collective
// (the generic path needs every lane).
template <bool kAcquire = true>
__device__ __forceinline__ void probe_lanes(const DevCtx& c, bool active, u64 key, u32& line, u64& word) {
  line = NONE;
  word = 0;
  const u32 W = c.ways;
  if (W <= 32 && (W & 7u) == 0) {
    if (active) {
      const u64 base = (u64)set_of(c, key) * W;
      const uint4* sp = reinterpret_cast<const uint4*>(c.sig + base);
      const u32 pat = sig16(key) * 0x10001u;
      uint4 v[4];
#pragma unroll
      for (u32 q = 0; q < 4; ++q) v[q] = (q * 8 < W) ? __ldcg(sp + q) : make_uint4(0u, 0u, 0u, 0u);
      u32 m = 0;
#pragma unroll
      for (u32 q = 0; q < 4; ++q)
        if (q * 8 < W) m |= sig_match8(v[q], pat) << (8 * q);
      while (m) {
        const u32 wy = __ffs(m) - 1;
        m &= m - 1;
        const u64 t = kAcquire ? ld_acquire(&c.tags[base + wy]) : ld_relaxed(&c.tags[base + wy]);
        if (tw_live(t) && tw_key(t) == key) { line = (u32)(base + wy); word = t; break; }
      }
    }
    return;
  }
  const ProbeRes r = probe_lanes_generic(c, active, key);
  line = r.line;
  word = r.word;
}

// Clock victim choice over one set held under its lock (ClockPolicy.map semantics,
// software_cache.py:109-126, per set; SURVEY A.2 plug-in).  Lane w holds way w's word (W<=32).
// Returns victim way or -1; fills the swept-and-cleared way mask and the new hand.
__device__ __forceinline__ int clock_pick_vec(u32 W, u32 hand, u32 avail, u32 ref1, u32& cleared, u32& new_hand) {
  const u32 fullw = (W == 32) ? FULL : ((1u << W) - 1);
  auto rot = [&](u32 m) -> u32 { return hand ? (((m >> hand) | (m << (W - hand))) & fullw) : (m & fullw); };
  auto unrot = [&](u32 m) -> u32 { return hand ? (((m << hand) | (m >> (W - hand))) & fullw) : (m & fullw); };
  const u32 A = rot(avail), R = rot(ref1);
  const u32 Z = A & ~R;
  int p;
  u32 clr;
  if (Z) {
    p = __ffs(Z) - 1;
    clr = A & R & ((1u << p) - 1u);
  } else if (A) {
    p = __ffs(A) - 1;
    clr = A & R;
  } else {
    cleared = 0;
    new_hand = hand;
    return -1;
  }
  const int v = (int)((hand + (u32)p) % W);
  // the victim's own ref bit is re-set by on_insert (software_cache.py:106-107): never clear it
  cleared = unrot(clr) & ~(1u << v);
  new_hand = (u32)(v + 1) % W;
  return v;
}

// ModuloPolicy.map (software_cache.py:129-143) inside the key's set: try t maps to way
// (dev * 7919 + blk + t) mod W (with one set of W = lines ways this is the reference's direct-mapped
// modulo placement over the whole cache).  `avail` = ways that are not BUSY and not pinned.
// busy_eviction_choice (software_cache.py:366-371): "wait" takes the home way or nothing (the
// caller retries: the reference parks on that line's ready_wait); "find_another" walks t = 1, 2,
// .. to the first available way (none in W tries: every way busy -> any_free_wait).  No reference
// bits, no hand.
__device__ __forceinline__ int modulo_pick(const DevCtx& c, u64 key, u32 W, u32 avail) {
  const u32 h = (u32)(((u64)key_dev(key) * 7919ull + key_blk(key)) % W);
  if (!c.find_another) return ((avail >> h) & 1u) ? (int)h : -1;
  const u32 fullw = (W == 32) ? FULL : ((1u << W) - 1);
  const u32 r = h ? (((avail >> h) | (avail << (W - h))) & fullw) : (avail & fullw);
  if (!r) return -1;
  return (int)((h + (u32)(__ffs(r) - 1)) % W);
}

// Serial exact sweep for W > 32 (fully associative parity mode), run by one lane.
__device__ __forceinline__ int clock_pick_serial(const DevCtx& c, u64 base, u32 W, u32 hand, u32& new_hand,
                                                 u64* cleared_list, u32& ncleared, u32 max_cleared) {
  u32 h = hand;
  ncleared = 0;
  for (u32 scanned = 0; scanned < 2 * W; ++scanned) {
    const u32 idx = h;
    const u64 w = ld_relaxed(&c.tags[base + idx]);
    h = (idx + 1) % W;
    if (tw_state(w) == ST_BUSY || tw_pins(w)) continue;
    if (tw_ref(w)) {
      atomicAnd(&c.tags[base + idx], ~REF_BIT);
      continue;
    }
    new_hand = h;
    return (int)idx;
  }
  new_hand = hand;
  return -1;
}

// ModuloPolicy for W > 32, run by one lane (see modulo_pick)
__device__ __forceinline__ int modulo_pick_serial(const DevCtx& c, u64 base, u32 W, u64 key) {
  const u64 h = ((u64)key_dev(key) * 7919ull + key_blk(key)) % W;
  for (u32 t = 0; t < W; ++t) {
    const u32 idx = (u32)((h + t) % W);
    const u64 w = ld_relaxed(&c.tags[base + idx]);
    if (tw_state(w) != ST_BUSY && tw_pins(w) == 0) return (int)idx;
    if (!c.find_another) return -1;
  }
  return -1;
}

// ---------------------------------------------------------------- debug_locks: wait-for cycles
// The reference's DeadlockDetector (lock_chain.py:70-121), restated as a wait-for graph over device
// words: every lock (set locks, SQ doorbell locks, share-table bucket locks) publishes its holder
// thread, every thread publishes the lock it is failing to take; a failed attempt walks
// lock -> holder -> the lock that holder waits for -> ... and a path back to the caller is a cycle:
// it is logged ("lock", "deadlock") and the run aborts with the cycle instead of spinning into
// the watchdog.  Off (one predictable branch per lock operation) unless debug_locks is set.
__device__ __forceinline__ u32 lk_set_id(const DevCtx& c, u32 set) { (void)c; return set; }
__device__ __forceinline__ u32 lk_db_id(const DevCtx& c, u32 q) { return c.num_sets + q; }
__device__ __forceinline__ u32 lk_bucket_id(const DevCtx& c, u32 h) { return c.num_sets + c.num_qp + h; }
__device__ __forceinline__ u32 lk_me() { return blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ void lk_acquired(const DevCtx& c, u32 id) {
  if (!c.dbg_locks) return;
  const u32 me = lk_me();
  if (me >= c.dbg_threads) return;
  st_relaxed(&c.lk_holder[id], me + 1);
  st_relaxed(&c.lk_wait[me], 0u);
}
__device__ __forceinline__ void lk_released(const DevCtx& c, u32 id) {
  if (c.dbg_locks) st_relaxed(&c.lk_holder[id], 0u);
}
__device__ __forceinline__ void lk_stop_waiting(const DevCtx& c) {
  if (!c.dbg_locks) return;
  const u32 me = lk_me();
  if (me < c.dbg_threads) st_relaxed(&c.lk_wait[me], 0u);
}
__device__ __noinline__ bool lk_failed_slow(const DevCtx& c, u32 id, u32 who) {
  const u32 me = lk_me();
  if (me >= c.dbg_threads) return false;
  st_relaxed(&c.lk_wait[me], id + 1);
  u32 cur = id, path[4] = {NONE, NONE, NONE, NONE}, np = 0;
  for (u32 hop = 0; hop < 64; ++hop) {
    const u32 h = ld_relaxed(&c.lk_holder[cur]);
    if (h == 0) return false;
    if (np < 4) path[np] = cur;
    ++np;
    if (h - 1 == me) {
      // re-validate once (lock_chain.py:117-121): the first hop must still be held by the same thread
      if (ld_relaxed(&c.lk_holder[id]) == 0) return false;
      log_ev(c, who, M_LOCK, A_DEADLOCK, id, np, path[0], path[1], path[2], path[3]);
      set_error(c, E_LOCK_CYCLE, id, np);
      return true;
    }
    const u32 w = ld_relaxed(&c.lk_wait[h - 1]);
    if (w == 0) return false;
    cur = w - 1;
  }
  return false;
}
__device__ __forceinline__ bool lk_failed(const DevCtx& c, u32 id, u32 who) {
  return c.dbg_locks ? lk_failed_slow(c, id, who) : false;
}

__device__ __forceinline__ bool lock_set(const DevCtx& c, u32 set, u32 who = WHO_USER) {
  int ok = 1;
  if (lane_id() == 0) {
    Spin sp;
    while (atom_cas_acquire(&c.set_lock[set], 0u, 1u) != 0u) {
      lk_failed(c, lk_set_id(c, set), who);
      if (!sp.again(c, 256, __LINE__ + 100000 * SPIN_FILE_ID)) { ok = 0; break; }
    }
    if (ok) lk_acquired(c, lk_set_id(c, set));
    else lk_stop_waiting(c);
  }
  return __shfl_sync(FULL, ok, 0) != 0;
}
__device__ __forceinline__ void unlock_set(const DevCtx& c, u32 set) {
  __syncwarp();
  if (lane_id() == 0) { lk_released(c, lk_set_id(c, set)); st_release(&c.set_lock[set], 0u); }
}

// Pin a line found by a lock-free probe: CAS the pin count up by n (capped, so a hot page can
// never overflow the 10-bit field into the ref/state bits).  Returns the post-pin word, or 0 if
// the line no longer holds `key` or is at the cap (callers retry later through the miss path).
constexpr u32 kPinCap = 960;
__device__ __forceinline__ u64 pin_line(const DevCtx& c, u32 line, u64 key, u32 n) {
  u64 w = ld_relaxed(&c.tags[line]);
  while (true) {
    if (!tw_live(w) || tw_key(w) != key || tw_pins(w) + n > kPinCap) return 0;
    const u64 nw = w + (u64)n * PIN_ONE;
    const u64 prev = atomicCAS(&c.tags[line], w, nw);
    if (prev == w) return nw;
    w = prev;
  }
}

__device__ __forceinline__ void log_state(const DevCtx& c, u32 who, u32 line, u32 from, u32 to, u64 key) {
  log_ev(c, who, M_CACHE, A_STATE, line, from, to, key_dev(key), key_blk(key));
}

// Miss path for one key (warp-uniform), under the set lock: re-probe (in-flight dedup), else pick
// a clock victim, CAS it to BUSY(key) and return R_MISS with the line to fill.  pin_n pins are
// added atomically to the resulting line (async_read waiters).  victim_key gets the evicted READY
// key (evict_reset, software_cache.py:339-346) or ~0.
__device__ int claim_key_warp(const DevCtx& c, u64 key, u32 pin_n, u32 who, u32& line, u64& word, u64& victim_key) {
  const u32 lane = lane_id();
  const u32 set = set_of(c, key);
  const u64 base = (u64)set * c.ways;
  const u32 W = c.ways;
  victim_key = ~0ull;
  if (lane == 0) log_ev(c, who, M_CACHE, A_MISS, key_dev(key), key_blk(key));
  if (!lock_set(c, set, who)) return R_RETRY;
  for (int attempt = 0;; ++attempt) {
    if (aborted(c)) { unlock_set(c, set); return R_RETRY; }
    u32 l; u64 w;
    if (probe_key_warp(c, key, l, w)) {
      int kind = tw_state(w) == ST_BUSY ? R_FILLING : R_HIT;
      if (lane == 0) {
        if (pin_n) w = pin_line(c, l, key, pin_n);
        if (!w) {
          kind = R_RETRY;
        } else {
          if (kind == R_HIT && !tw_ref(w)) atomicOr(&c.tags[l], REF_BIT);
          kind = tw_state(w) == ST_BUSY ? R_FILLING : R_HIT;
        }
      }
      kind = __shfl_sync(FULL, kind, 0);
      w = __shfl_sync(FULL, w, 0);
      unlock_set(c, set);
      line = l; word = w;
      return kind;
    }
    int v;
    u32 new_hand;
    u64 old = 0;
    u32 cleared = 0;
    const u32 hand = ld_relaxed(&c.hand[set]);
    if (W <= 32) {
      u64 tw = 0;
      if (lane < W) tw = ld_relaxed(&c.tags[base + lane]);
      const u32 avail = __ballot_sync(FULL, lane < W && tw_state(tw) != ST_BUSY && tw_pins(tw) == 0);
      const u32 ref1 = __ballot_sync(FULL, lane < W && tw_ref(tw));
      if (c.policy == POL_MODULO) { v = modulo_pick(c, key, W, avail); new_hand = hand; }
      else v = clock_pick_vec(W, hand, avail, ref1, cleared, new_hand);
      if (v >= 0) old = __shfl_sync(FULL, tw, v);
    } else {
      int vv = -1;
      u32 nh = hand;
      u32 ncl = 0;
      if (lane == 0)
        vv = c.policy == POL_MODULO ? modulo_pick_serial(c, base, W, key)
                                    : clock_pick_serial(c, base, W, hand, nh, nullptr, ncl, 0);
      v = __shfl_sync(FULL, vv, 0);
      new_hand = __shfl_sync(FULL, nh, 0);
      if (v >= 0) old = ld_relaxed(&c.tags[base + v]);
    }
    if (v < 0) {  // every way busy/pinned: caller waits (any_free_wait, software_cache.py:364-365)
      unlock_set(c, set);
      return R_RETRY;
    }
    if (tw_state(old) == ST_MODIFIED) {
      // MODIFIED victim: write it back first (R_WBEVICT), claim the freed line on the retry
      const u64 nwb = tw_make(ST_BUSY, tw_key(old), tw_ver(old) + 1, false, 0);
      u64 pv = 0;
      if (lane == 0) {
        st_relaxed(&c.wl[base + v], ((u64)((tw_ver(old) + 1) & 0x1FFu)) << 55);
        pv = atom_cas_acqrel(&c.tags[base + v], old, nwb);
      }
      pv = __shfl_sync(FULL, pv, 0);
      if (pv != old) continue;
      if (lane == 0) {
        st_relaxed(&c.hand[set], new_hand);
        log_ev(c, who, M_CACHE, A_EVICT_WB, base + v, key_dev(tw_key(old)), key_blk(tw_key(old)));
        log_state(c, who, (u32)(base + v), ST_MODIFIED, ST_BUSY, tw_key(old));
      }
      unlock_set(c, set);
      victim_key = tw_key(old);
      line = (u32)(base + v);
      word = nwb;
      return R_WBEVICT;
    }
    const u64 nw = tw_make(ST_BUSY, key, tw_ver(old) + 1, true, pin_n);
    u64 prev = 0;
    if (lane == 0) {
      st_relaxed(&c.wl[base + v], ((u64)((tw_ver(old) + 1) & 0x1FFu)) << 55);   // open the waiter list
      prev = atom_cas_acqrel(&c.tags[base + v], old, nw);
    }
    prev = __shfl_sync(FULL, prev, 0);
    if (prev != old) continue;   // a hitter touched ref/pins: re-evaluate
    if (W <= 32 && lane < W && ((cleared >> lane) & 1u)) atomicAnd(&c.tags[base + lane], ~REF_BIT);
    if (lane == 0) {
      c.sig[base + v] = (unsigned short)sig16(key);   // probe hint (the tag word decides)
      st_relaxed(&c.hand[set], new_hand);
      const u32 ost = tw_state(old);
      if (ost == ST_READY || ost == ST_MODIFIED) {
        victim_key = tw_key(old);
        atomicAdd(&c.stats[S_RESETS], 1ull);
        log_ev(c, who, M_CACHE, A_EVICT_RESET, base + v, key_dev(victim_key), key_blk(victim_key));
        log_state(c, who, (u32)(base + v), ost, ST_INVALID, victim_key);
      }
      log_state(c, who, (u32)(base + v), ST_INVALID, ST_BUSY, key);
      atomicAdd(&c.stats[S_FILLS], 1ull);
    }
    victim_key = __shfl_sync(FULL, victim_key, 0);
    unlock_set(c, set);
    line = (u32)(base + v);
    word = nw;
    return R_MISS;
  }
}

// Lane-parallel miss path (W <= 32).  Lanes whose keys map to the same set form a group
// (__match_any_sync on the set index); the group's lowest lane takes the set lock ONCE per pass and
// every member then scans the set (all loads in flight at once, one round trip) and claims its own
// victim in lane order: member r replays the policy's picks of the members before it on the same
// scanned state (ClockPolicy.map called once per miss under the policy lock, software_cache.py:
// 109-126, 355-371 — so the order and the victims equal the reference's sequential claims) and
// CASes its victim to BUSY(key) in parallel with the others.  A whole group thus costs one lock
// round trip instead of one per member.  Same semantics per key as claim_key_warp: re-probe
// (in-flight dedup), victim by policy, MODIFIED victims written back first (R_WBEVICT).  The loop
// is convergent; a member whose CAS lost to a hitter retries next pass.  Returns per lane R_HIT /
// R_FILLING / R_MISS / R_RETRY / R_WBEVICT (R_NONE if !want).
__device__ int claim_lanes(const DevCtx& c, bool want, u64 key, u32 pin_n, u32 who, u32& line, u64& word,
                           u64& victim_key) {
  const u32 lane = lane_id();
  const u32 W = c.ways;
  int kind = R_NONE;
  victim_key = ~0ull;
  const u32 set = want ? set_of(c, key) : 0u;
  const u64 base = (u64)set * W;
  if (want) log_ev(c, who, M_CACHE, A_MISS, key_dev(key), key_blk(key));
  u32 pending = __ballot_sync(FULL, want);
  u32 fills = 0, resets = 0;
  Spin sp;
  while (pending) {
    const bool mine = (pending >> lane) & 1u;
    u32 grp = __match_any_sync(FULL, mine ? set : NONE);
    if (!mine) grp = 0;
    const u32 leader = grp ? (u32)(__ffs(grp) - 1) : lane;
    int got = 0;
    if (mine && lane == leader) {
      got = atom_cas_acquire(&c.set_lock[set], 0u, 1u) == 0u;
      if (got) lk_acquired(c, lk_set_id(c, set));
      else lk_failed(c, lk_set_id(c, set), who);
    }
    got = __shfl_sync(FULL, got, leader) && mine;
    bool settled = false;
    // ---- every member of a locked group scans the set (the same state for all of them)
    u32 avail = 0, ref1 = 0, hand = 0;
    int found = -1;
    u64 fw = 0;
    if (got) {
      hand = ld_relaxed(&c.hand[set]);
#pragma unroll
      for (u32 w0 = 0; w0 < 32; w0 += 8) {
        if (w0 >= W) break;
        ulonglong2 q[4];
#pragma unroll
        for (u32 j = 0; j < 4; ++j) {
          if (W & 1u) {   // odd ways: sets are not 16 B aligned
            const u32 a = w0 + 2 * j, b = a + 1;
            q[j] = make_ulonglong2(a < W ? ld_relaxed(&c.tags[base + a]) : 0ull,
                                   b < W ? ld_relaxed(&c.tags[base + b]) : 0ull);
          }
          else q[j] = (w0 + 2 * j < W) ? __ldcg(reinterpret_cast<const ulonglong2*>(c.tags + base + w0) + j)
                                       : make_ulonglong2(0ull, 0ull);
        }
#pragma unroll
        for (u32 j = 0; j < 8; ++j) {
          const u32 w = w0 + j;
          const u64 t = (j & 1u) ? q[j >> 1].y : q[j >> 1].x;
          if (w < W) {
            if (tw_live(t) && tw_key(t) == key) { found = (int)w; fw = t; }
            if (tw_state(t) != ST_BUSY && tw_pins(t) == 0) avail |= 1u << w;
            if (tw_ref(t)) ref1 |= 1u << w;
          }
        }
      }
    }
    // members that need a victim, in lane order; each replays the picks of the members of its own
    // group before it.  All groups replay in parallel, one member rank per step: in step r every
    // lane of a group computes the pick of its group's r-th member on the group's (replicated)
    // state, so a pass costs max-group-size picks instead of one per needing lane of the warp.
    const u32 needw = __ballot_sync(FULL, got && found < 0);
    int v = -1;
    u32 my_cleared = 0, nh = hand;
    {
      const u32 gneed = got ? (needw & grp) : 0u;
      const u32 myrank = __popc(gneed & lanemask_lt());
      const u32 gsz = __popc(gneed);
      u32 av = avail, rf = ref1, hd = hand;
      bool stop = false;
      for (u32 r = 0; __any_sync(FULL, r < gsz); ++r) {
        u64 kr = 0;
        if (c.policy == POL_MODULO)   // the key of the group's r-th member (warp-uniform branch)
          kr = __shfl_sync(FULL, key, r < gsz ? __fns(gneed, 0, (int)r + 1) : lane);
        if (r >= gsz || stop) continue;
        u32 cl = 0, h2 = hd;
        int pk;
        if (c.policy == POL_MODULO) {
          pk = modulo_pick(c, kr, W, av);
        } else {
          pk = clock_pick_vec(W, hd, av, rf, cl, h2);
        }
        if (myrank == r && found < 0) { v = pk; my_cleared = cl; nh = h2; }
        if (pk < 0) { stop = true; continue; }   // nothing left for this member or the ones after it
        av &= ~(1u << pk);                       // the victim turns BUSY
        rf = (rf & ~cl) | (1u << pk);            // swept bits cleared; on_insert sets the victim's
        hd = h2;
      }
    }
    if (got) {
      if (found >= 0) {
        u64 w2 = fw;
        if (pin_n) w2 = pin_line(c, (u32)(base + found), key, pin_n);
        if (w2) {
          kind = tw_state(w2) == ST_BUSY ? R_FILLING : R_HIT;
          if (kind == R_HIT && !tw_ref(w2)) atomicOr(&c.tags[base + found], REF_BIT);
          line = (u32)(base + found);
          word = w2;
        } else {
          kind = R_RETRY;   // pin count at its cap: come back later
        }
        settled = true;
      } else if (v < 0) {
        kind = R_RETRY;     // every way busy/pinned: wait (any_free_wait, software_cache.py:364-365)
        settled = true;
      } else {
        const u64 old = ld_relaxed(&c.tags[base + v]);
        if (tw_state(old) == ST_MODIFIED && tw_pins(old) == 0) {
          // MODIFIED victim: write it back first, claim the freed line on the retry
          const u64 nw = tw_make(ST_BUSY, tw_key(old), tw_ver(old) + 1, false, 0);
          st_relaxed(&c.wl[base + v], ((u64)((tw_ver(old) + 1) & 0x1FFu)) << 55);
          if (atom_cas_acqrel(&c.tags[base + v], old, nw) == old) {
            victim_key = tw_key(old);
            log_ev(c, who, M_CACHE, A_EVICT_WB, base + v, key_dev(victim_key), key_blk(victim_key));
            log_state(c, who, (u32)(base + v), ST_MODIFIED, ST_BUSY, victim_key);
            kind = R_WBEVICT;
            line = (u32)(base + v);
            word = nw;
            settled = true;
          }
        } else if (tw_state(old) != ST_BUSY && tw_pins(old) == 0) {
          const u64 nw = tw_make(ST_BUSY, key, tw_ver(old) + 1, true, pin_n);
          st_relaxed(&c.wl[base + v], ((u64)((tw_ver(old) + 1) & 0x1FFu)) << 55);   // open the waiter list
          if (atom_cas_acqrel(&c.tags[base + v], old, nw) == old) {
            c.sig[base + v] = (unsigned short)sig16(key);   // probe hint (the tag word decides)
            const u32 ost = tw_state(old);
            if (ost == ST_READY || ost == ST_MODIFIED) {
              victim_key = tw_key(old);
              ++resets;
              log_ev(c, who, M_CACHE, A_EVICT_RESET, base + v, key_dev(victim_key), key_blk(victim_key));
              log_state(c, who, (u32)(base + v), ost, ST_INVALID, victim_key);
            }
            log_state(c, who, (u32)(base + v), ST_INVALID, ST_BUSY, key);
            ++fills;
            kind = R_MISS;
            line = (u32)(base + v);
            word = nw;
            settled = true;
          }
        }
        // else: a hitter pinned/touched the victim between scan and CAS: re-evaluate next pass
        // the sweep of this member's pick cleared these reference bits (the reference's map)
        if (settled && c.policy != POL_MODULO)
          for (u32 m = my_cleared; m; m &= m - 1) atomicAnd(&c.tags[base + (__ffs(m) - 1)], ~REF_BIT);
      }
    }
    // the group's hand follows its last settled pick; the leader releases the lock after every
    // member's CAS (convergent point)
    const u32 setm = __ballot_sync(FULL, got && settled && v >= 0) & grp;
    const int lastp = setm ? 31 - __clz(setm) : -1;
    const u32 fin_hand = __shfl_sync(FULL, nh, lastp < 0 ? lane : (u32)lastp);
    __syncwarp();
    if (got && lane == leader) {
      if (lastp >= 0 && c.policy != POL_MODULO) st_relaxed(&c.hand[set], fin_hand);
      lk_released(c, lk_set_id(c, set));
      st_release(&c.set_lock[set], 0u);
    }
    const u32 progressed = __ballot_sync(FULL, got);
    pending &= ~__ballot_sync(FULL, settled);
    if (pending && !progressed) {
      if (!sp.again(c, 512, __LINE__ + 100000 * SPIN_FILE_ID)) {
        if ((pending >> lane) & 1u) kind = R_RETRY;
        break;
      }
    }
  }
  if (want) lk_stop_waiting(c);
  const u32 nf = __popc(__ballot_sync(FULL, fills != 0));
  const u32 nr = __popc(__ballot_sync(FULL, resets != 0));
  if (lane == 0) {
    if (nf) atomicAdd(&c.stats[S_FILLS], (u64)nf);
    if (nr) atomicAdd(&c.stats[S_RESETS], (u64)nr);
  }
  return kind;
}

__device__ __forceinline__ void unpin_line(const DevCtx& c, u32 line, u32 n) {
  atomicAdd(&c.tags[line], (u64)0 - (u64)n * PIN_ONE);
}

// ======================================================================= K2: SQ submit

__device__ __forceinline__ u32 sq_slot_index(const DevCtx& c, u32 q, u64 v) { return q * c.sq_depth + (u32)(v & (c.sq_depth - 1)); }

// Doorbell protocol (attempt_sqdb, nvme_queue.py:293-311): whoever wins the doorbell lock flips
// the contiguous UPDATED run after the published doorbell to ISSUED (64 entries per scan) and
// publishes once; everyone loops until the doorbell passed `target`.  Lock and doorbell share one
// word (doorbell << 1 | lock): the acquiring atomic OR returns the current doorbell and one release
// store publishes the new doorbell and unlocks (3 round trips fewer than lock word + doorbell word).
// `start`: first entry of the caller's own contiguous range [start, target) (all UPDATED by the
// calling warp before the call); when the published doorbell is exactly `start`, the lock holder
// flips its own range without scanning (one round trip less) and publishes `target`.
__device__ bool ring_doorbell_until(const DevCtx& c, u32 q, u64 target, u32 who, u64 start = ~0ull) {
  const u32 lane = lane_id();
  SqWords* s = &c.sqw[q];
  const u32 D = c.sq_depth;
  Spin sp;
  bool first = true;
  while (true) {
    // first pass: go straight for the lock (the caller just made entries UPDATED, so the
    // doorbell is almost never past them yet); afterwards check the doorbell before retrying
    if (!first) {
      const u64 db = ld_acquire(&s->dbl) >> 1;
      if (db >= target) {
        if (lane == 0) lk_stop_waiting(c);
        return true;
      }
    }
    first = false;
    int got = 0;
    u64 ow = 0;
    if (lane == 0) {
      ow = atom_or_acquire(&s->dbl, 1ull);
      got = (ow & 1ull) == 0;
      if (got) lk_acquired(c, lk_db_id(c, q));
      else lk_failed(c, lk_db_id(c, q), who);
    }
    got = __shfl_sync(FULL, got, 0);
    if (got) {
      const u64 old = __shfl_sync(FULL, ow, 0) >> 1;
      u64 v = old;
      const bool fast = old == start && target > start && target - start <= 32;
      if (fast) {
        // fast path: the range right after the doorbell is the caller's own (UPDATED by its
        // lanes before the warp barrier that precedes this call)
        const u64 vi = start + lane;
        if (vi < target) {
          if (atom_cas_acqrel(&c.sq_state[sq_slot_index(c, q, vi)], SQ_UPDATED, SQ_ISSUED) != SQ_UPDATED)
            set_error(c, E_PROTOCOL, q, vi);
          log_ev(c, who, M_NVME, A_SQE_ISSUED, q, vi & (D - 1), vi & (D - 1));
        }
        v = target;
      }
      while (!fast) {
        // 64 entries per round trip (two per lane): a full warp's submission (32 UPDATED
        // entries) is found and bounded in one scan instead of two
        const u64 vi0 = v + lane, vi1 = v + 32 + lane;
        const u32 idx0 = sq_slot_index(c, q, vi0), idx1 = sq_slot_index(c, q, vi1);
        bool upd0 = false, upd1 = false;
        if (vi0 < old + D) upd0 = ld_acquire(&c.sq_state[idx0]) == SQ_UPDATED;
        if (vi1 < old + D) upd1 = ld_acquire(&c.sq_state[idx1]) == SQ_UPDATED;
        const u32 b0 = __ballot_sync(FULL, upd0), b1 = __ballot_sync(FULL, upd1);
        const u32 prefix = (~b0) ? (u32)(__ffs(~b0) - 1) : ((~b1) ? 32u + (u32)(__ffs(~b1) - 1) : 64u);
#pragma unroll
        for (u32 h = 0; h < 2; ++h) {
          const u64 vi = h ? vi1 : vi0;
          if (32 * h + lane < prefix) {
            // per-lane acq_rel CAS: each lane's flip is itself a release (a relaxed store made
            // visible only through lane 0's doorbell release is not cumulative in practice — the
            // engine then saw the doorbell before the ISSUED word)
            if (atom_cas_acqrel(&c.sq_state[h ? idx1 : idx0], SQ_UPDATED, SQ_ISSUED) != SQ_UPDATED)
              set_error(c, E_PROTOCOL, q, vi);
            log_ev(c, who, M_NVME, A_SQE_ISSUED, q, vi & (D - 1), vi & (D - 1));
          }
        }
        v += prefix;
        if (prefix < 64) break;
      }
      __syncwarp();
      if (lane == 0) {
        if (v > old) {
          st_relaxed(&s->db_time, gtimer());
          log_ev(c, who, M_NVME, A_DOORBELL, q, old, v, D);
          atomicAdd(&c.stats[S_DOORBELLS], 1ull);
        }
        lk_released(c, lk_db_id(c, q));
        // publish + unlock: the doorbell is a release fence
        st_release(&s->dbl, v << 1);
      }
      __syncwarp();
      if (v >= target) {   // our own publish covered the caller's entries
        if (lane == 0) lk_stop_waiting(c);
        return true;
      }
      continue;
    }
    if (!sp.again(c, 256, __LINE__ + 100000 * SPIN_FILE_ID)) return false;
  }
}

// Warp-aggregated submission (submit_command/attempt_enqueue, nvme_queue.py:314-354).
// Lanes with `has` place one command each.  Lanes targeting the same device elect a leader
// (__match_any_sync) that reserves popc slots with a capacity-checked CAS on the SQ tail
// (tail - head <= depth - 1, nvme_queue.py:131-144); partial grants leave the remainder pending
// and the next round rotates to the following SQ; a full lap backs off until the service frees
// entries.  Returns false only when the run is aborting.
__device__ bool submit_warp(const DevCtx& c, bool has, u32 dev, u64 blk, u32 line, u32 kind, u32 op, u64 buf,
                            u64 key, u32 who, u32 sq_start) {
  const u32 lane = lane_id();
  const u32 D = c.sq_depth, P = c.pairs_per_device;
  u32 pending = __ballot_sync(FULL, has);
  u32 rot = 0;
  Spin sp;
  while (pending) {
    const bool mine = (pending >> lane) & 1u;
    u32 grp = __match_any_sync(FULL, mine ? dev : 0xffffffffu);
    if (!mine) grp = 0;
    const u32 rank = __popc(grp & lanemask_lt());
    const u32 n = __popc(grp);
    u32 q = 0, m = 0;
    u64 t = 0;
    if (mine && rank == 0) {
      for (u32 k = 0; k < P && m == 0; ++k) {
        const u32 qq = dev * P + (sq_start + rot + k) % P;
        SqWords* s = &c.sqw[qq];
        u64 tt = ld_relaxed(&s->tail);
        while (true) {
          const u64 hh = ld_acquire(&s->head);
          const u64 used = tt - hh;
          if (used >= (u64)(D - 1)) break;
          const u32 take = (u32)min((u64)n, (u64)(D - 1) - used);
          const u64 prev = atomicCAS(&s->tail, tt, tt + take);
          if (prev == tt) { q = qq; t = tt; m = take; break; }
          tt = prev;
        }
        if (m == 0) atomicAdd(&c.stats[S_SQ_FULL], 1ull);
      }
      if (m) atomicAdd(&c.pw->outstanding, (u64)m);
    }
    const u32 leader = grp ? (u32)(__ffs(grp) - 1) : lane;
    q = __shfl_sync(FULL, q, leader);
    t = __shfl_sync(FULL, t, leader);
    m = __shfl_sync(FULL, m, leader);
    const bool got = mine && rank < m;
    if (got) {
      const u64 v = t + rank;
      const u32 slot = (u32)(v & (D - 1));
      const u32 idx = q * D + slot;
      uint4* e = c.sqe + (u64)idx * 4;
      const u64 prp = kind == K_RAW ? buf : (u64)(uintptr_t)line_ptr(c, line);
      // 64 B NVMe SQE: CDW0 opcode|CID, NSID, PRP1 (dw6-7), SLBA (dw10-11), NLB (dw12, 0-based)
      e[0] = make_uint4((op == OP_READ ? 0x02u : 0x01u) | (slot << 16), dev + 1, 0u, 0u);
      e[1] = make_uint4(0u, 0u, (u32)prp, (u32)(prp >> 32));
      e[2] = make_uint4(0u, 0u, (u32)blk, (u32)(blk >> 32));
      e[3] = make_uint4(0u, 0u, 0u, 0u);
      CmdCtx* x = &c.cmd[idx];
      x->key = key;
      x->vidx = v;
      x->t_submit = gtimer();
      x->line = kind == K_RAW ? NONE : line;
      x->kind = kind;
      x->buf = buf;
      log_ev(c, who, M_NVME, A_ENQUEUE, q, slot, slot, op, dev, blk);
      // EMPTY -> UPDATED publishes the SQE and its context (release).  The reserved slot is EMPTY
      // by construction (tail - head <= depth - 1, head advances over released entries only);
      // debug runs verify it with a CAS (mark_updated, nvme_queue.py:160-162).
      if (c.trace) {
        if (atom_cas_acqrel(&c.sq_state[idx], SQ_EMPTY, SQ_UPDATED) != SQ_EMPTY)
          set_error(c, E_PROTOCOL, q, v);
      } else {
        st_release(&c.sq_state[idx], SQ_UPDATED);
      }
      log_ev(c, who, M_NVME, A_SQE_UPDATED, q, slot);
    }
    __syncwarp();
    u32 lead_b = __ballot_sync(FULL, mine && rank == 0 && m > 0);
    while (lead_b) {
      const int L = __ffs(lead_b) - 1;
      lead_b &= lead_b - 1;
      const u32 qL = __shfl_sync(FULL, q, L);
      const u64 endL = __shfl_sync(FULL, t + m, L);
      if (!ring_doorbell_until(c, qL, endL, who, __shfl_sync(FULL, t, L))) return false;
    }
    const u32 gb = __ballot_sync(FULL, got);
    if (lane == 0 && gb) atomicAdd(&c.stats[S_ENQUEUES], (u64)__popc(gb));
    pending &= ~gb;
    if (pending && !gb) {
      ++rot;
      if (!sp.again(c, 1024, __LINE__ + 100000 * SPIN_FILE_ID)) return false;
    }
  }
  return true;
}

// ======================================================================= user-side verbs
// (AgileApi, gpu_api.py:139-278; paper Listing 1 naming: prefetch / asyncRead / wait)

struct Req {        // per-lane result of an access
  u32 line;
  int kind;         // R_HIT / R_FILLING / R_MISS / R_NONE
  u64 word;
  u64 victim;       // key evicted by this miss (evict_reset) or ~0
};

// Warp-collective cache access, ONE attempt.  Lanes with the same key coalesce (__match_any_sync,
// lowest lane leads: warp_coalesce, gpu_api.py:40-54).  pin: every requesting lane of a resolved
// key holds one pin on the line (the leader adds them all); !pin: prefetch semantics.  Leaders
// whose set has no available victim get R_RETRY (so do their followers): callers retry after
// releasing every pin they hold — no pin is ever held across a claim or a retry, so a full cache
// cannot deadlock (hold-and-wait).
__device__ Req access_warp(const DevCtx& c, bool active, u64 key, bool pin, u32 who, u32 sq_start,
                           bool drop_followers) {
  const u32 lane = lane_id();
  Req r;
  r.line = NONE; r.kind = R_NONE; r.word = 0; r.victim = ~0ull;
  if (active) {   // AgileApi._check_block (gpu_api.py:122-126): OutOfRange before the cache is touched
    const u32 dv = key_dev(key);
    if (dv >= c.num_devices || key_blk(key) >= c.store_blocks[dv]) {
      set_error(c, E_OUT_OF_RANGE, dv, key_blk(key));
      active = false;
    }
  }
  u32 grp = __match_any_sync(FULL, active ? key : ~0ull);
  if (!active) grp = 0;
  const bool leader = active && (grp & lanemask_lt()) == 0;
  const u32 gsize = __popc(grp);
  const u32 lead_lane = grp ? (u32)(__ffs(grp) - 1) : lane;
  // lock-free probe for every leader
  u32 l; u64 w;
  probe_lanes(c, leader, key, l, w);
  bool resolved = false;
  if (leader && l != NONE) {
    u64 pw = w;
    if (pin) pw = pin_line(c, l, key, gsize);
    if (pw) {
      r.line = l;
      r.word = pw;
      r.kind = tw_state(pw) == ST_BUSY ? R_FILLING : R_HIT;
      if (r.kind == R_HIT && !tw_ref(pw)) atomicOr(&c.tags[l], REF_BIT);   // on_hit
      resolved = true;
    }
  }
  // misses: lane-parallel claims under per-set locks (W <= 32); one key at a time otherwise
  const u32 mb = __ballot_sync(FULL, leader && !resolved);
  bool need_submit = false, need_wb = false;
  u32 wb_line = NONE;
  u64 wb_key = 0;
  if (mb) {
    if (c.ways <= 32) {
      u32 cl = NONE; u64 cw = 0, vk = ~0ull;
      const bool wl = (mb >> lane) & 1u;
      const int kind = claim_lanes(c, wl, key, pin ? gsize : 0u, who, cl, cw, vk);
      if (wl) {
        if (kind == R_RETRY || kind == R_NONE) r.kind = R_RETRY;
        else if (kind == R_WBEVICT) { r.kind = R_RETRY; need_wb = true; wb_line = cl; wb_key = vk; }
        else { r.line = cl; r.word = cw; r.kind = kind; r.victim = vk; need_submit = kind == R_MISS; }
      }
    } else {
      u32 m2 = mb;
      while (m2) {
        const int src = __ffs(m2) - 1;
        m2 &= m2 - 1;
        const u64 k = __shfl_sync(FULL, key, src);
        const u32 pn = pin ? __shfl_sync(FULL, gsize, src) : 0u;
        u32 cl; u64 cw, vk;
        const int kind = claim_key_warp(c, k, pn, __shfl_sync(FULL, who, src), cl, cw, vk);
        if (lane == (u32)src) {
          if (kind == R_RETRY) r.kind = R_RETRY;
          else if (kind == R_WBEVICT) { r.kind = R_RETRY; need_wb = true; wb_line = cl; wb_key = vk; }
          else { r.line = cl; r.word = cw; r.kind = kind; r.victim = vk; need_submit = kind == R_MISS; }
        }
      }
    }
  }
  // submit fills and eviction write-backs (warp-aggregated)
  if (__any_sync(FULL, need_submit || need_wb)) {
    const bool sub = need_submit || need_wb;
    const u64 sk = need_wb ? wb_key : key;
    if (!submit_warp(c, sub, key_dev(sk), key_blk(sk), need_wb ? wb_line : r.line, need_wb ? K_WB_EVICT : K_FILL,
                     need_wb ? OP_WRITE : OP_READ, 0, sk, who, sq_start))
      if (sub) r.kind = R_NONE;
    const u32 nwb = __popc(__ballot_sync(FULL, need_wb));
    if (lane == 0 && nwb) atomicAdd(&c.stats[S_WRITEBACKS], (u64)nwb);
  }
  // accounting + trace
  u32 hits = 0, attaches = 0, misses = 0;
  if (leader) {
    if (r.kind == R_HIT) { hits = 1; log_ev(c, who, M_CACHE, A_HIT, key_dev(key), key_blk(key)); }
    else if (r.kind == R_MISS) misses = 1;
    else if (r.kind == R_FILLING) { attaches = 1; log_ev(c, who, M_CACHE, A_ATTACH, r.line, 1); }
  }
  // broadcast to followers
  const u32 bl = __shfl_sync(FULL, r.line, lead_lane);
  const int bk = __shfl_sync(FULL, r.kind, lead_lane);
  const u64 bw = __shfl_sync(FULL, r.word, lead_lane);
  if (active && !leader) {
    if (drop_followers) {
      r.line = NONE; r.kind = R_NONE;
    } else {
      r.line = bl; r.word = bw;
      r.kind = (bk == R_HIT || bk == R_RETRY || bk == R_NONE) ? bk : R_FILLING;
      if (r.kind == R_HIT) hits = 1;
      else if (r.kind == R_FILLING) { attaches = 1; log_ev(c, who, M_CACHE, A_ATTACH, r.line, 1); }
    }
  }
  const u32 h = __popc(__ballot_sync(FULL, hits != 0));
  const u32 a = __popc(__ballot_sync(FULL, attaches != 0));
  const u32 mm = __popc(__ballot_sync(FULL, misses != 0));
  if (lane == 0) {
    if (h) atomicAdd(&c.stats[S_HITS], (u64)h);
    if (a) atomicAdd(&c.stats[S_ATTACHES], (u64)a);
    if (mm) atomicAdd(&c.stats[S_MISSES], (u64)mm);
  }
  return r;
}

// Prefetch (AgileApi.prefetch, gpu_api.py:139-155): pull blocks toward the cache without waiting;
// duplicates die in the warp; lanes whose set is momentarily full retry (no pins are held).
__device__ void prefetch_warp(const DevCtx& c, bool active, u64 key, u32 who, u32 sq_start, bool best_effort) {
  bool want = active;
  Spin sp;
  while (__any_sync(FULL, want)) {
    const Req r = access_warp(c, want, key, false, who, sq_start, true);
    want = want && r.kind == R_RETRY;
    if (best_effort || !__any_sync(FULL, want)) break;
    if (!sp.again(c, 2048, __LINE__ + 100000 * SPIN_FILE_ID)) break;
  }
}

// ------------------------------------------------------------------ async_read waiter lists
// A lane's request is a WaitNode in device memory (its AgileBuf: destination + barrier word).
// Lines with a fill in flight carry a lock-free waiter stack `wl[line]` = [ver:9 | closed:1 |
// node>>4 : 54]; the claimant opens it for the new version, waiters push with a version-checked
// CAS, and the service closes it, copies the line into every waiter's buffer and clears their
// barriers before flipping the line READY (_drain_waiters, software_cache.py:563-570).  Nobody
// holds a line while waiting, exactly like the reference.
struct WaitNode {
  u64 next;     // packed next node
  u64 dst;      // 4 KiB destination
  u32 done;     // TransactionBarrier state: 0 PENDING, 1 DONE (agile_service.py:31-72)
  u32 pad;
  u64 t_issue;
};
constexpr int WL_VER_SHIFT = 55;
constexpr u64 WL_CLOSED = 1ull << 54;
constexpr u64 WL_PTR_MASK = (1ull << 54) - 1;
__device__ __forceinline__ u64 wl_open(u32 ver) { return (u64)(ver & 0x1FFu) << WL_VER_SHIFT; }
__device__ __forceinline__ u32 wl_ver(u64 w) { return (u32)(w >> WL_VER_SHIFT); }
__device__ __forceinline__ WaitNode* wl_node(u64 w) { return reinterpret_cast<WaitNode*>((w & WL_PTR_MASK) << 4); }

// push `node` on the line's stack for version `ver`; false if the list is closed (the fill is
// completing: the caller copies from the line itself) or belongs to another version
__device__ __forceinline__ bool wl_push(const DevCtx& c, u32 line, u32 ver, WaitNode* node) {
  u64 h = ld_acquire(&c.wl[line]);
  while (true) {
    if (wl_ver(h) != (ver & 0x1FFu) || (h & WL_CLOSED)) return false;
    node->next = h & WL_PTR_MASK;
    const u64 nw = wl_open(ver) | ((u64)(uintptr_t)node >> 4);
    const u64 prev = atom_cas_acqrel(&c.wl[line], h, nw);
    if (prev == h) return true;
    h = prev;
  }
}

// AgileApi._fresh_barrier (gpu_api.py:132-137): a buffer whose previous transfer is still pending
// (issued, barrier not DONE) cannot start another one -> BufferBusy.  WaitNodes start zeroed
// (t_issue 0: never used) at every run that hands them out.
__device__ __forceinline__ bool buffer_busy(const DevCtx& c, const WaitNode* node) {
  if (node->t_issue != 0 && ld_acquire(&node->done) == 0) {
    set_error(c, E_BUFFER_BUSY, (u64)(uintptr_t)node, node->t_issue);
    return true;
  }
  return false;
}

__device__ __forceinline__ void copy_page_warp(const uint4* src, uint4* dst) {
  const u32 lane = lane_id();
  uint4 v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = __ldcg(src + lane + 32 * k);
#pragma unroll
  for (int k = 0; k < 8; ++k) __stcg(dst + lane + 32 * k, v[k]);
}

// async_read (gpu_api.py:164-190), warp-collective: start filling each active lane's node->dst
// from `key`.  HIT: copied now.  MISS/FILLING: the node joins the line's waiter stack and the
// service delivers it.  Returns with no pin held.  Outcomes are counted by access_warp.
__device__ void async_read_warp(const DevCtx& c, bool active, u64 key, WaitNode* node, uint4* dst, u32 who,
                                u32 sq_start, int* outcome = nullptr, u64* victim = nullptr) {
  const u32 lane = lane_id();
  if (active && buffer_busy(c, node)) active = false;
  bool want = active;
  if (active) { node->dst = (u64)(uintptr_t)dst; node->done = 0; node->t_issue = gtimer(); }
  __syncwarp();
  Spin sp;
  while (__any_sync(FULL, want)) {
    const Req r = access_warp(c, want, key, true, who, sq_start, false);
    bool copy_now = false, pinned = false;
    if (want) {
      if (r.kind == R_RETRY) {
        // set full of busy/pinned lines: nothing held, try again
      } else if (r.kind == R_NONE) {
        want = false;   // aborting
      } else {
        pinned = true;
        if (outcome) *outcome = r.kind == R_HIT ? 0 : (r.kind == R_MISS ? 1 : 2);
        if (victim) *victim = r.victim;
        if (r.kind == R_HIT) copy_now = true;
        else if (!wl_push(c, r.line, tw_ver(r.word), node)) copy_now = true;   // fill completing
        want = false;
      }
    }
    // lanes copying themselves: wait for READY (the line is pinned and already completing), copy
    u32 cb = __ballot_sync(FULL, copy_now);
    Spin s2;
    while (cb) {
      bool ready = false;
      if ((cb >> lane) & 1u) {
        const u64 w = ld_acquire(&c.tags[r.line]);
        ready = tw_state(w) == ST_READY || tw_state(w) == ST_MODIFIED;
      }
      u32 rb = __ballot_sync(FULL, ready) & cb;
      __syncwarp();
      while (rb) {
        const int l0 = __ffs(rb) - 1;
        rb &= rb - 1;
        const uint4* src = reinterpret_cast<const uint4*>(line_ptr(c, __shfl_sync(FULL, r.line, l0)));
        WaitNode* nd = reinterpret_cast<WaitNode*>(__shfl_sync(FULL, (u64)(uintptr_t)node, l0));
        copy_page_warp(src, reinterpret_cast<uint4*>(nd->dst));
        __syncwarp();
        if (lane == (u32)l0) st_release(&nd->done, 1u);
        cb &= ~(1u << l0);
      }
      if (cb && !s2.again(c, 512, __LINE__ + 100000 * SPIN_FILE_ID)) break;
    }
    if (pinned) unpin_line(c, r.line, 1);
    if (__any_sync(FULL, want) && !sp.again(c, 2048, __LINE__ + 100000 * SPIN_FILE_ID)) break;
  }
}

// one poll pass over nodes: mask of lanes whose transfer is done (AgileApi.wait, gpu_api.py:233-248)
__device__ __forceinline__ u32 poll_nodes_warp(bool active, const WaitNode* node) {
  bool d = false;
  if (active) d = ld_acquire(&node->done) != 0;
  return __ballot_sync(FULL, d);
}

__device__ bool wait_nodes_warp(const DevCtx& c, bool active, const WaitNode* node) {
  u32 pending = __ballot_sync(FULL, active);
  Spin sp;
  while (pending) {
    pending &= ~poll_nodes_warp((pending >> lane_id()) & 1u, node);
    if (pending && !sp.again(c, 256, __LINE__ + 100000 * SPIN_FILE_ID)) return false;
  }
  return true;
}

// Wait (without pinning) until the line holds `key` READY.  Returns false if the line was
// reassigned meanwhile (caller re-accesses).
__device__ __forceinline__ bool wait_ready_lane(const DevCtx& c, u32 line, u64 key, Spin& sp, bool& alive) {
  const u64 w = ld_acquire(&c.tags[line]);
  if (!tw_live(w) || tw_key(w) != key) { alive = false; return false; }
  alive = true;
  return tw_state(w) == ST_READY || tw_state(w) == ST_MODIFIED;
}

template <int kSlice = 4>
__device__ void deliver_waiters_warp(const DevCtx& c, u64 cur, u32 line);

// Block write (SoftwareCache._try_write / _install_locked / _allocate_locked,
// software_cache.py:458-523), warp-collective: the 4 KiB at `src` land in the block's cache line.
//   eager (async_write, gpu_api.py:192-227; write_block, software_cache.py:221-235): a device write
//     (WB_KEEP) starts at once and the line is BUSY until it is durable, then READY
//     (complete_io); `node` is the durability handle, released by the service.
//   !eager (install_modified, software_cache.py:242-254: share-table data draining back): no device
//     write — the line is left MODIFIED; async_read waiters that attached meanwhile get the new bytes;
//     `node` is released on return.
// Resident READY/MODIFIED line with no pins: CAS -> BUSY, version + 1 (readers validating the old
// identity see the change).  Not resident: a victim is claimed like a fill; a MODIFIED victim is
// written back first (WB_EVICT) and the claim retried.  BUSY or pinned lines, and later lanes writing
// a block an earlier lane of the warp writes, retry (RETRY + ready_wait in the reference).  No pin
// is held.
// once: a single attempt (callers that re-check other state between attempts, the share table);
// returns true for lanes still pending.
__device__ bool write_block_warp(const DevCtx& c, bool active, u64 key, WaitNode* node, const uint4* src,
                                 u32 who, u32 sq_start, bool eager, bool once = false) {
  const u32 lane = lane_id();
  if (active) {
    const u32 dv = key_dev(key);
    if (dv >= c.num_devices || key_blk(key) >= c.store_blocks[dv]) {   // _check_block
      set_error(c, E_OUT_OF_RANGE, dv, key_blk(key));
      active = false;
    }
  }
  if (active && !once && buffer_busy(c, node)) active = false;
  if (active) { node->dst = 0; node->done = 0; node->t_issue = gtimer(); }
  __syncwarp();
  bool want = active;
  Spin sp;
  while (__any_sync(FULL, want)) {
    // same block twice in the warp: lowest lane first, the others next pass (program order)
    const u32 grp = __match_any_sync(FULL, want ? key : ~0ull);
    const u32 wb = __ballot_sync(FULL, want);
    const bool go = want && (grp & lanemask_lt() & wb) == 0;
    u32 line = NONE;
    u64 word = 0;
    probe_lanes(c, go, key, line, word);
    bool own = false;
    u32 ver = 0;
    if (go && line != NONE) {
      // resident: take it from READY/MODIFIED with no pins, under the set lock (victim claims
      // open waiter lists under the same lock, so no list opened here can be clobbered)
      const u32 set = line / c.ways;
      if (atom_cas_acquire(&c.set_lock[set], 0u, 1u) == 0u) {
        lk_acquired(c, lk_set_id(c, set));
        const u64 w = ld_relaxed(&c.tags[line]);
        const u32 st = tw_state(w);
        if (tw_live(w) && tw_key(w) == key && (st == ST_READY || st == ST_MODIFIED) && tw_pins(w) == 0) {
          ver = tw_ver(w) + 1;
          const u64 nw = tw_make(ST_BUSY, key, ver, true, 0);
          if (atom_cas_acqrel(&c.tags[line], w, nw) == w) {
            st_relaxed(&c.wl[line], ((u64)(ver & 0x1FFu)) << 55);   // open the waiter list
            own = true;
            log_ev(c, who, M_CACHE, A_HIT, key_dev(key), key_blk(key));
            log_state(c, who, line, st, ST_BUSY, key);
          }
        }
        lk_released(c, lk_set_id(c, set));
        st_release(&c.set_lock[set], 0u);
      } else {
        lk_failed(c, lk_set_id(c, set), who);
      }
    }
    const u32 mb = __ballot_sync(FULL, go && line == NONE);
    bool need_wb = false;
    u32 wb_line = NONE;
    u64 wb_key = 0;
    if (mb) {
      u32 cl = NONE; u64 cw = 0, vk = ~0ull;
      const bool wl = (mb >> lane) & 1u;
      if (c.ways <= 32) {
        const int kind = claim_lanes(c, wl, key, 0u, who, cl, cw, vk);
        if (wl && kind == R_MISS) { own = true; line = cl; word = cw; ver = tw_ver(cw); }
        if (wl && kind == R_WBEVICT) { need_wb = true; wb_line = cl; wb_key = vk; }
      } else {
        // generic geometry: one key at a time
        u32 m2 = mb;
        while (m2) {
          const int l = __ffs(m2) - 1;
          m2 &= m2 - 1;
          u32 l2; u64 w2, v2;
          const int k2 = claim_key_warp(c, __shfl_sync(FULL, key, l), 0u, __shfl_sync(FULL, who, l), l2, w2, v2);
          if (lane == (u32)l && k2 == R_MISS) { own = true; line = l2; word = w2; ver = tw_ver(w2); }
          if (lane == (u32)l && k2 == R_WBEVICT) { need_wb = true; wb_line = l2; wb_key = v2; }
        }
      }
    }
    // a MODIFIED victim's write-back: submitted now, the claim is retried once it is durable
    if (__any_sync(FULL, need_wb)) {
      if (!submit_warp(c, need_wb, key_dev(wb_key), key_blk(wb_key), wb_line, K_WB_EVICT, OP_WRITE, 0, wb_key, who,
                       sq_start))
        break;
      const u32 nwb = __popc(__ballot_sync(FULL, need_wb));
      if (lane == 0 && nwb) atomicAdd(&c.stats[S_WRITEBACKS], (u64)nwb);
    }
    // owners: register the durability handle (eager), land the bytes
    bool pushed = false;
    if (own && eager) pushed = wl_push(c, line, ver, node);
    u32 ob = __ballot_sync(FULL, own);
    while (ob) {
      const int l = __ffs(ob) - 1;
      ob &= ob - 1;
      const uint4* s0 = reinterpret_cast<const uint4*>(__shfl_sync(FULL, (u64)(uintptr_t)src, l));
      uint4* d0 = reinterpret_cast<uint4*>(line_ptr(c, __shfl_sync(FULL, line, l)));
      copy_page_warp(s0, d0);
    }
    __syncwarp();
    if (__any_sync(FULL, own)) {
      if (own) log_ev(c, who, M_CACHE, A_INSTALL, key_dev(key), key_blk(key), *reinterpret_cast<const u64*>(src));
      if (eager) {
        const u32 nwb = __popc(__ballot_sync(FULL, own));
        if (lane == 0) atomicAdd(&c.stats[S_WRITEBACKS], (u64)nwb);
        if (!submit_warp(c, own, key_dev(key), key_blk(key), line, K_WB_KEEP, OP_WRITE, 0, key, who, sq_start)) {
          if (own) want = false;
          break;
        }
      } else {
        // no device write: the bytes are visible, hand them to attached readers, then MODIFIED
        __threadfence();
        u64 wlh = 0;
        if (own) wlh = atom_exch_acqrel(&c.wl[line], ((u64)(ver & 0x1FFu) << 55) | WL_CLOSED);
        deliver_waiters_warp(c, own ? (wlh & WL_PTR_MASK) : 0ull, line);
        if (own) {
          atom_add_release(&c.tags[line], (u64)(ST_MODIFIED - ST_BUSY) << ST_SHIFT);   // BUSY -> MODIFIED
          log_state(c, who, line, ST_BUSY, ST_MODIFIED, key);
          st_release(&node->done, 1u);
        }
      }
    }
    if (own) {
      if (eager && !pushed) st_release(&node->done, 1u);   // cannot happen (the list was opened by us)
      want = false;
    }
    if (once) break;
    if (__any_sync(FULL, want) && !sp.again(c, 2048, __LINE__ + 100000 * SPIN_FILE_ID)) break;
  }
  if (active) lk_stop_waiting(c);
  return want;
}

__device__ __forceinline__ void async_write_warp(const DevCtx& c, bool active, u64 key, WaitNode* node,
                                                 const uint4* src, u32 who, u32 sq_start) {
  write_block_warp(c, active, key, node, src, who, sq_start, true);
}

// ======================================================================= K3: completion service

// uint4 per lane per waiter-copy step: 8 = every load of both pages in flight at once (the
// register-engine infra kernel, one CTA per SM), 4 = half the registers in two steps (the bulk-
// engine infra kernel at 128 registers, and user-side deliveries)

// Waiter delivery (_drain_waiters, software_cache.py:563-570), warp-collective: every lane with a
// closed waiter list (cur = its first node, 0 = none) of `line` copies the line into each waiting
// AgileBuf and releases its barrier.  Rounds: every lane loads its current node (destination and
// link: one round trip for the whole warp), the pages of all lanes' current nodes move kNP at a
// time (4 pages in flight per step with 8-uint4 slices — 128 registers of data, like the engine's
// page moves; 2 with 4-uint4 slices), then ONE fence and the barriers of the round are released.
// A window of single-waiter completions is thus delivered in one node round trip, ceil(n / kNP)
// page round trips and one fence.
template <int kSvcSlice>
__device__ void deliver_waiters_warp(const DevCtx& c, u64 cur, u32 line) {
  constexpr int kNP = kSvcSlice >= 8 ? 4 : 2;
  const u32 lane = lane_id();
  while (true) {
    const u32 all = __ballot_sync(FULL, cur != 0);
    if (!all) break;
    WaitNode* me = reinterpret_cast<WaitNode*>(cur << 4);
    {
      // a waiter list only ever links this run's WaitNodes: anything else is a corrupted list
      const u64 a = (u64)(uintptr_t)me;
      const bool bad = cur != 0 && (a < c.nodes_lo || a >= c.nodes_hi);
      if (__any_sync(FULL, bad)) {
        if (bad) { set_error(c, E_ILLEGAL_STATE, a, 0xD0000000ull | (u64)__LINE__); cur = 0; }
        continue;
      }
    }
    // dst == 0: a write's durability handle (async_write) — completion only, no copy.  The link
    // is read BEFORE the barrier is released: once DONE, the requester may reuse the node at once
    // (its next async_read re-links it into another line's list).
    u64 mydst = 0, mynext = 0;
    if (cur) { mydst = me->dst; mynext = me->next; }
    for (u32 rem = all; rem;) {
      int ln[kNP];
      const uint4* src[kNP];
      uint4* dst[kNP];
#pragma unroll
      for (int p = 0; p < kNP; ++p) {
        ln[p] = rem ? __ffs(rem) - 1 : -1;
        if (rem) rem &= rem - 1;
        const int sl = ln[p] < 0 ? ln[0] : ln[p];
        src[p] = reinterpret_cast<const uint4*>(line_ptr(c, __shfl_sync(FULL, line, sl)));
        const u64 d = __shfl_sync(FULL, mydst, sl);
        dst[p] = ln[p] < 0 ? nullptr : reinterpret_cast<uint4*>(d);
      }
#pragma unroll
      for (int h = 0; h < 8; h += kSvcSlice) {
        uint4 v[kNP][kSvcSlice];
#pragma unroll
        for (int p = 0; p < kNP; ++p)
          if (dst[p]) {
#pragma unroll
            for (int k = 0; k < kSvcSlice; ++k) v[p][k] = __ldcg(src[p] + lane + 32 * (h + k));
          }
#pragma unroll
        for (int p = 0; p < kNP; ++p)
          if (dst[p]) {
#pragma unroll
            for (int k = 0; k < kSvcSlice; ++k) __stcg(dst[p] + lane + 32 * (h + k), v[p][k]);
          }
      }
    }
    // release pattern for the whole round: every lane's page stores happen before the warp barrier
    // (bar.warp.sync orders memory among its participants), the fence after it is cumulative over
    // them, and each owning lane's DONE store follows that fence in its own program order — so a
    // requester whose acquire load sees DONE sees the page (one fence per round instead of an
    // st.release per barrier word, which serialised across the diverged owning lanes)
    __syncwarp();
    __threadfence();
    if (cur) { st_relaxed(&me->done, 1u); cur = mynext; }
  }
}


// SQ head advance over the completed prefix (_advance_head, nvme_queue.py:213-228), warp-
// collective for one SQ q (warp-uniform): 32 consecutive entries' completion words are checked in
// one round trip and the head moves over the whole done prefix with one CAS (a window of k
// completions costs one pass, not k dependent load + CAS pairs).
__device__ __forceinline__ void advance_head_warp(const DevCtx& c, u32 q, u32 who) {
  SqWords* s = &c.sqw[q];
  const u32 D = c.sq_depth;
  const u32 lane = lane_id();
  u64 h = 0;
  if (lane == 0) h = ld_acquire(&s->head);
  h = __shfl_sync(FULL, h, 0);
  bool moved = false;
  while (true) {
    const u64 e = h + lane;
    // depth < 32: lanes past the ring alias earlier slots whose word cannot equal e + 1
    const bool ok = ld_acquire(&c.sq_done_v[q * D + (u32)(e & (D - 1))]) == e + 1;
    const u32 b = __ballot_sync(FULL, ok);
    const u32 n = b == FULL ? 32u : (u32)(__ffs(~b) - 1);
    if (n == 0) break;
    u64 prev = 0;
    if (lane == 0) prev = atomicCAS(&s->head, h, h + n);
    prev = __shfl_sync(FULL, prev, 0);
    if (prev == h) {
      h += n;
      moved = true;
      if (n < 32) break;
    } else {
      h = prev;
    }
  }
  if (moved && lane == 0) log_ev(c, who, M_NVME, A_HEAD, q, h);
}

// One window pass over a CQ owned by the calling warp (cq_polling, agile_service.py:147-171 +
// process_cqe 173-199): 32 lanes validate 32 consecutive CQEs against the expected phase; each
// valid lane releases its SQE (first, so stuck producers move), then flips the cache line
// BUSY->READY with one release-add (fan-out: waiters poll the tag word), then the SQ head
// advances over the completed prefix.  Only a full window rings the CQ doorbell.  off/mask is the
// CQ's poll state, held in the owning lane's registers by service_main.
template <int kSlice>
__device__ u32 cq_window_pass(const DevCtx& c, u32 cq, u64& off, u32& mask, u32 who, u64& lat_acc, u32& rings) {
  const u32 lane = lane_id();
  const u32 window = c.cq_window;
  const u32 Dq = c.cq_depth;
  const u32 Ds = c.sq_depth;
  bool valid = false, cache = false;
  u32 sq = 0, slot = 0;
  CmdCtx x;
  x.line = NONE; x.t_submit = 0; x.key = 0;
  u64 wlh = 0;
  const u64 v = off + lane;
  if (lane < window && !((mask >> lane) & 1u)) {
    const u64 w = ld_acquire(reinterpret_cast<const u64*>(c.cqe + (u64)cq * Dq + (u32)(v & (Dq - 1))) + 1);
    const u32 phase = (u32)(w >> 48) & 1u;
    const u32 expect = 1u - (u32)((v / Dq) & 1u);   // lap 0 writes 1 (nvme_queue.py:262-264)
    if (phase == expect) {
      valid = true;
      sq = (u32)(w >> 16) & 0xffffu;
      slot = (u32)(w >> 32) & 0xffffu;   // CID == SQE slot
    }
  }
  if (valid) {
    const u32 idx = sq * Ds + slot;
    if (sq >= c.num_qp || slot >= Ds) {
      set_error(c, E_UNKNOWN_CID, cq, v);
      valid = false;
    } else {
      x = c.cmd[idx];
      if (x.line != NONE && x.line >= c.num_lines) {
        set_error(c, E_ILLEGAL_STATE, x.line, 0xC0000000ull | (u64)__LINE__);
        x.line = NONE;
      }
      const u32 os = atom_cas_acqrel(&c.sq_state[idx], SQ_ISSUED, SQ_EMPTY);
      atomicExch(&c.sq_done_v[idx], x.vidx + 1);
      cache = x.line != NONE && (x.kind == K_FILL || x.kind == K_WB_KEEP || x.kind == K_WB_EVICT);
      if (cache) {
        // close the waiter stack of this fill: setting the closed bit detaches the list (every
        // later push sees it closed and copies from the line itself; the next claim re-opens the
        // word for its version), so no tag read is needed to rebuild the word
        wlh = atom_or_acqrel(&c.wl[x.line], WL_CLOSED);
      }
      if (os != SQ_ISSUED) set_error(c, E_UNKNOWN_CID, sq, slot);
      log_ev(c, who, M_NVME, A_SQE_RELEASE, sq, slot, slot);
      log_ev(c, who, M_SVC, A_CQE_PROCESS, cq, v, slot, sq);
    }
  }
  __syncwarp();
  // drain waiters: copy the filled line into every waiting AgileBuf and clear its barrier while
  // the line is still BUSY (not evictable), then flip it READY (software_cache.py:538-541,563-570)
  deliver_waiters_warp<kSlice>(c, (valid && cache) ? (wlh & WL_PTR_MASK) : 0ull, x.line);
  if (valid && cache && x.kind != K_WB_EVICT) {
    const u64 ot = atom_add_release(&c.tags[x.line], 1ull << ST_SHIFT);   // BUSY -> READY
    if (tw_state(ot) != ST_BUSY) set_error(c, E_ILLEGAL_STATE, x.line, ot);
    log_state(c, who, x.line, ST_BUSY, ST_READY, x.key);
  } else if (valid && cache) {
    // eviction write-back durable (complete_io WB_EVICT, software_cache.py:538-553): the old key's
    // bytes are on the device; the line turns INVALID (version + 1, pins kept) for the claimant's retry
    u64 ot = ld_relaxed(&c.tags[x.line]);
    while (true) {
      if (tw_state(ot) != ST_BUSY) { set_error(c, E_ILLEGAL_STATE, x.line, ot); break; }
      const u64 nt = (ot & PIN_MASK) | tw_make(ST_INVALID, 0, tw_ver(ot) + 1, false, 0);
      const u64 pv = atom_cas_acqrel(&c.tags[x.line], ot, nt);
      if (pv == ot) break;
      ot = pv;
    }
    log_state(c, who, x.line, ST_BUSY, ST_INVALID, x.key);
  }
  if (valid) {
    lat_acc += gtimer() - x.t_submit;
    fence_sc();
  }
  __syncwarp();
  // head advance: one leader per SQ among completed lanes
  const u32 grp = __match_any_sync(FULL, valid ? sq : 0xffffffffu);
  for (u32 lb = __ballot_sync(FULL, valid && (grp & lanemask_lt()) == 0); lb; lb &= lb - 1)
    advance_head_warp(c, __shfl_sync(FULL, sq, __ffs(lb) - 1), who);
  const u32 vb = __ballot_sync(FULL, valid);
  mask |= vb;
  const u32 fullw = window == 32 ? FULL : ((1u << window) - 1u);
  if (mask == fullw) {
    if (lane == 0) {
      log_ev(c, who, M_SVC, A_WINDOW_RING, cq, off, off + window);
      st_release(&c.cqw[cq].host_db, off + window);   // ring only full windows
    }
    ++rings;
    off += window;
    mask = 0;
  }
  const u32 k = __popc(vb);
  if (k && lane == 0) atom_add_release(&c.pw->outstanding, (u64)0 - (u64)k);
  __syncwarp();
  return k;
}

__device__ void drain_partial_windows(const DevCtx& c, u32 who) {
  // _drain_partial_windows, agile_service.py:224-236 (lane-parallel over CQs)
  for (u32 cq0 = 0; cq0 < c.num_qp; cq0 += 32) {
    const u32 cq = cq0 + lane_id();
    if (cq < c.num_qp) {
      CqWords* cw = &c.cqw[cq];
      const u32 mask = ld_relaxed(&cw->poll_mask);
      if (mask) {
        const u32 k = (u32)(__ffs(~mask) - 1);
        if (mask != ((k == 32) ? FULL : ((1u << k) - 1u))) set_error(c, E_PROTOCOL, cq, mask);
        const u64 off = ld_relaxed(&cw->poll_offset);
        log_ev(c, who, M_SVC, A_DRAIN_RING, cq, off, off + k);
        st_release(&cw->host_db, off + k);
        st_relaxed(&cw->poll_offset, off + k);
        st_relaxed(&cw->poll_mask, 0u);
        atomicAdd(&c.stats[S_DRAIN_ENTRIES], (u64)k);
      }
    }
  }
}

// Service warps (AgileService._warp_program, agile_service.py:126-145).  Warp w serves CQs
// w, w+S, w+2S, ... — the reference's round-robin stride, made static so the poll state (offset,
// window mask) lives in the owning lane's registers and no claim word is needed.  Each pass one
// lane per CQ checks the next expected CQE's phase (one round trip for all owned CQs); only ready
// CQs get a window pass.  Idle passes back off poll_ns -> idle_max_ns.
constexpr u32 kMaxCqPerLane = 4;
template <int kSlice = 4>
__device__ void service_main(const DevCtx& c, const Launch& L, u32 sw) {
  const u32 lane = lane_id();
  const u32 who = WHO_SVC | sw;
  const u32 n = c.num_qp;
  const u32 S = c.service_warps;
  const u32 nown = n > sw ? (n - sw + S - 1) / S : 0;
  if (sw == 0 && lane == 0) log_ev(c, who, M_SVC, A_START, S);
  if (nown > 32 * kMaxCqPerLane) set_error(c, E_PROTOCOL, nown, 0);
  const u64 t_enter = gtimer();
  u64 off[kMaxCqPerLane];
  u32 msk[kMaxCqPerLane];
#pragma unroll
  for (u32 j = 0; j < kMaxCqPerLane; ++j) {
    const u32 k = lane + 32 * j;
    off[j] = 0; msk[j] = 0;
    if (k < nown) {
      const u32 cq = sw + k * S;
      off[j] = ld_relaxed(&c.cqw[cq].poll_offset);
      msk[j] = ld_relaxed(&c.cqw[cq].poll_mask);
    }
  }
  u32 idle = c.poll_ns;
  u64 lat = 0;
  u32 rings = 0, done = 0;
  const u32 Dq = c.cq_depth;
  while (true) {
    u32 got = 0;
#pragma unroll
    for (u32 j = 0; j < kMaxCqPerLane; ++j) {
      if (32 * j >= nown) break;
      const u32 k = lane + 32 * j;
      bool ready = false;
      if (k < nown) {
        const u32 cq = sw + k * S;
        const u64 nv = off[j] + __popc(msk[j]);   // valid CQEs arrive in order: the mask is a prefix
        const u64 w = ld_relaxed(reinterpret_cast<const u64*>(c.cqe + (u64)cq * Dq + (u32)(nv & (Dq - 1))) + 1);
        ready = (((u32)(w >> 48)) & 1u) == 1u - (u32)((nv / Dq) & 1u);
      }
      u32 rb = __ballot_sync(FULL, ready);
      while (rb) {
        const int l = __ffs(rb) - 1;
        rb &= rb - 1;
        u64 o = __shfl_sync(FULL, off[j], l);
        u32 m = __shfl_sync(FULL, msk[j], l);
        const u32 cq = sw + ((u32)l + 32 * j) * S;
        got += cq_window_pass<kSlice>(c, cq, o, m, who, lat, rings);
        if (lane == (u32)l) { off[j] = o; msk[j] = m; }
      }
    }
    done += got;
    if (got) {
      idle = c.poll_ns;
      continue;
    }
    int stop = 0;
    if (lane == 0) {
      const bool users = ld_acquire(&c.run->users_done) >= L.n_user_ctas;
      const u64 out = ld_acquire(&c.pw->outstanding);
      stop = (users && out == 0) || aborted(c);
      // the user grid never started (a kernel-serialising tool, or a launch that was not allowed
      // to overlap this grid): give up instead of waiting forever.  The CAS on users_started
      // orders the decision against every user CTA's start (a CTA that starts later reads the
      // give-up bit from its own atomicAdd and never waits on this grid).
      if (!stop && gtimer() - t_enter > c.user_start_ns && ld_relaxed(&c.run->users_started) == 0 &&
          atomicCAS(&c.run->users_started, 0u, kInfraGaveUp) == 0u) {
        if (!c.solo_ok) set_error(c, E_LIVELOCK, 0, __LINE__ + 100000 * SPIN_FILE_ID);
        stop = 1;
      }
      if (users && atomicCAS(&c.run->stop_logged, 0u, 1u) == 0u) log_ev(c, who, M_SVC, A_STOP);
    }
    if (__shfl_sync(FULL, stop, 0)) break;
    nap(idle);
    idle = min(idle * 2, c.idle_max_ns);
  }
  // persist the poll state for the drain and the next launch
#pragma unroll
  for (u32 j = 0; j < kMaxCqPerLane; ++j) {
    const u32 k = lane + 32 * j;
    if (k < nown) {
      const u32 cq = sw + k * S;
      st_relaxed(&c.cqw[cq].poll_offset, off[j]);
      st_relaxed(&c.cqw[cq].poll_mask, msk[j]);
    }
  }
  u64 lsum = lat;
#pragma unroll
  for (int o = 16; o; o >>= 1) lsum += __shfl_xor_sync(FULL, lsum, o);
  if (lane == 0) {
    if (done) {
      atomicAdd(&c.stats[S_COMPLETIONS], (u64)done);
      atomicAdd(&c.stats[S_BARRIER_COUNT], (u64)done);
      atomicAdd(&c.stats[S_BARRIER_NS], lsum);
    }
    if (rings) atomicAdd(&c.stats[S_WINDOWS], (u64)rings);
  }
  __threadfence();
  // the last warp out rings residual partial windows (agile_service.py:141-145)
  u32 order = 0;
  if (lane == 0) order = atomicAdd(&c.run->svc_exited, 1u);
  order = __shfl_sync(FULL, order, 0);
  if (order == S - 1) {
    __threadfence();
    drain_partial_windows(c, who);
    __syncwarp();
    if (lane == 0) st_release(&c.run->engine_stop, 1u);
  }
}

// ======================================================================= K4: device engine

__device__ __forceinline__ u64 splitmix64(u64 x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// LatencyModel.service_ns (ssd_model.py:45-53) for draw number `seq` of device `dev`
__device__ __forceinline__ u64 model_service_ns(const DevCtx& c, u32 op, u32 dev, u64 seq) {
  const u64 base = op == OP_READ ? c.model.read_ns : c.model.write_ns;
  if (c.model.jitter == 0 || c.model.jitter_ns == 0) return base;
  const u64 r = splitmix64(c.model.seed ^ ((u64)dev << 48) ^ seq);
  if (c.model.jitter == 1) return base + r % c.model.jitter_ns;
  const double u = ((r >> 11) + 0.5) * (1.0 / 9007199254740992.0);
  return base + (u64)(-log(u) * (double)c.model.jitter_ns);
}

// FIFO channel dispatch (_dispatch/_start/_free_channel, ssd_model.py:168-186) for every lane in
// `mask` whose command targets `dev`, in lane order: start at the earliest free channel no sooner
// than arrival; the channel is held for occupancy_ns.  One lock hold per (warp pass, device);
// channel free-times live in registers (lane i holds channels i, i+32, ...).
constexpr u32 kMaxChanPerLane = 8;   // parallelism <= 256
__device__ void model_schedule_batch(const DevCtx& c, u32 dev, u32 mask, u32 op, u64 arrival, u64& due) {
  const u32 lane = lane_id();
  const u32 P = c.model.parallelism;
  const u32 n = __popc(mask);
  int ok = 1;
  u64 seq0 = 0;
  if (lane == 0) {
    Spin sp;
    while (atom_cas_acquire(&c.dev_lock[dev], 0u, 1u) != 0u)
      if (!sp.again(c, 128, __LINE__ + 100000 * SPIN_FILE_ID)) { ok = 0; break; }
    if (ok && c.model.jitter && c.model.jitter_ns) seq0 = atomicAdd(&c.dev_seq[dev], (u64)n);
  }
  ok = __shfl_sync(FULL, ok, 0);
  seq0 = __shfl_sync(FULL, seq0, 0);
  if (!ok) { if ((mask >> lane) & 1u) due = 0; return; }
  u64* ch = c.chan_free + (u64)dev * P;
  u64 cf[kMaxChanPerLane];
#pragma unroll
  for (u32 k = 0; k < kMaxChanPerLane; ++k) {
    const u32 i = lane + 32 * k;
    cf[k] = i < P ? ld_relaxed(&ch[i]) : ~0ull;
  }
  u32 todo = mask;
  u32 rank = 0;
  while (todo) {
    const int l = __ffs(todo) - 1;
    todo &= todo - 1;
    const u64 arr = __shfl_sync(FULL, arrival, l);
    const u32 opl = __shfl_sync(FULL, op, l);
    const u64 svc = model_service_ns(c, opl, dev, seq0 + rank);
    ++rank;
    // warp argmin over channel free-times (ties -> lowest channel index)
    u64 best = ~0ull;
    u32 bi = 0;
#pragma unroll
    for (u32 k = 0; k < kMaxChanPerLane; ++k) {
      if (cf[k] < best) { best = cf[k]; bi = lane + 32 * k; }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const u64 ob = __shfl_xor_sync(FULL, best, o);
      const u32 oi = __shfl_xor_sync(FULL, bi, o);
      if (ob < best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    const u64 start = max(arr, best);
    const u64 occ = c.model.occupancy_ns ? c.model.occupancy_ns : svc;
#pragma unroll
    for (u32 k = 0; k < kMaxChanPerLane; ++k)
      if (lane + 32 * k == bi) cf[k] = start + occ;
    if (lane == (u32)l) due = start + svc;
  }
#pragma unroll
  for (u32 k = 0; k < kMaxChanPerLane; ++k) {
    const u32 i = lane + 32 * k;
    if (i < P) st_relaxed(&ch[i], cf[k]);
  }
  __syncwarp();
  if (lane == 0) st_release(&c.dev_lock[dev], 0u);
  __syncwarp();
}

// lane holding the smallest sequence number among lanes with `cand` (-1 if none)
__device__ __forceinline__ int oldest_lane(bool cand, u32 seq) {
  u32 best = cand ? seq : 0xffffffffu;
  int bl = cand ? (int)lane_id() : 32;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const u32 ob = __shfl_xor_sync(FULL, best, o);
    const int ol = __shfl_xor_sync(FULL, bl, o);
    if (ob < best || (ob == best && ol < bl)) { best = ob; bl = ol; }
  }
  return bl < 32 ? bl : -1;
}

// Constant service time (no jitter): FIFO dispatch to the earliest-free of P identical channels
// is round-robin in arrival order (starts are non-decreasing, so the channel that frees first is
// the one used P commands earlier).  Lock-free: a warp-aggregated ticket per device fixes the
// order, channel = ticket % P, and a per-channel turn word hands the channel from command k-P to
// command k.  Every lane with `want` gets its completion time in `due`.
__device__ void model_schedule_rr(const DevCtx& c, bool want, u32 dev, u32 op, u64 arrival, u64& due) {
  const u32 lane = lane_id();
  const u32 P = c.model.parallelism;
  u32 grp = __match_any_sync(FULL, want ? dev : 0xffffffffu);
  if (!want) grp = 0;
  const u32 rank = __popc(grp & lanemask_lt());
  u64 base = 0;
  if (want && rank == 0) base = atomicAdd(&c.dev_seq[dev], (u64)__popc(grp));
  base = __shfl_sync(FULL, base, want ? (u32)(__ffs(grp) - 1) : lane);
  const u64 ticket = base + rank;
  const u32 ch = (u32)(ticket % P);
  const u64 turn = ticket / P;
  const u64 svc = op == OP_READ ? c.model.read_ns : c.model.write_ns;
  const u64 occ = c.model.occupancy_ns ? c.model.occupancy_ns : svc;
  bool done = !want;
  Spin sp;
  while (__any_sync(FULL, !done)) {
    if (!done) {
      const u64 idx = (u64)dev * P + ch;
      if (ld_acquire(&c.chan_turn[idx]) == turn) {
        const u64 start = max(arrival, ld_relaxed(&c.chan_free[idx]));
        st_relaxed(&c.chan_free[idx], start + occ);
        st_release(&c.chan_turn[idx], turn + 1);
        due = start + svc;
        done = true;
      }
    }
    if (__any_sync(FULL, !done) && !sp.again(c, 64, __LINE__ + 100000 * SPIN_FILE_ID)) {
      if (!done) due = 0;
      break;
    }
  }
}

// pages one engine warp moves per pass, held in registers (32 per page per lane) while the pass
// posts completions and fetches new SQEs; the infra grid runs one CTA per SM, so 4 pages fit
#ifndef AGILE_ENGINE_PAGES
#define AGILE_ENGINE_PAGES 4
#endif
constexpr int kEnginePages = AGILE_ENGINE_PAGES;

// page stores of the engine: cache-streaming (evict-first in L2) so a stream of fills does not
// evict the working sets of kernels running beside it (AGILE_FILL_STORE=__stcg to compare)
#ifndef AGILE_FILL_STORE
#define AGILE_FILL_STORE __stcs
#endif

// Bulk-copy engine (split launch): a page moves host-pinned store -> shared memory through the
// TMA bulk-copy unit (cp.async.bulk ... mbarrier::complete_tx, UBLKCP in SASS), so the long host-
// link latency is covered by shared-memory slots instead of registers; the short HBM leg is a
// coalesced warp copy out of the slot.  kEngineSlots 4 KiB slots per engine warp.
#ifndef AGILE_ENGINE_SLOTS
#define AGILE_ENGINE_SLOTS 4
#endif
constexpr int kEngineSlots = AGILE_ENGINE_SLOTS;
constexpr u32 kInfraSmem = kCtaWarps * kEngineSlots * (kBlockBytes + 8);   // stages + mbarriers

__device__ __forceinline__ u32 smem_addr(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_test(u64* bar, u32 parity) {
  u32 done;
  asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(done) : "r"(smem_addr(bar)), "r"(parity) : "memory");
  return done != 0;
}
// one 4 KiB global -> shared bulk copy whose completion (bytes landed) flips `bar`
__device__ __forceinline__ void bulk_page_to_smem(void* dst_smem, const void* src, u64* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // earlier generic reads of the slot first
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 4096;" :: "r"(smem_addr(bar)) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];"
               :: "r"(smem_addr(dst_smem)), "l"(src), "r"(smem_addr(bar)) : "memory");
}

template <int kPages = kEnginePages, bool kBulk = false>
__device__ void engine_main(const DevCtx& c, u32 ew, uint8_t* slots = nullptr) {
  const u32 lane = lane_id();
  const u32 E = c.engine_warps;
  const u32 Ds = c.sq_depth, Dq = c.cq_depth;
  const u32 nq = c.num_qp > ew ? (c.num_qp - ew + E - 1) / E : 0;   // owned QPs: ew, ew+E, ...
  // one in-service command per lane: fetched (pv), data moved (pcp), completion due at pdue
  bool pv = false, pcp = false, plogged = false, pstalled = false;
  u32 pq = 0, pslot = 0, pop = 0, pdev = 0;
  u64 pdue = 0, pblk = 0, prp = 0;
  u32 rr = 0, pass = 0, seq = 0, pseq = 0;
  u32 idle = 32;
  u64 bytes_r = 0, bytes_w = 0;
  // bulk mode: slot s (< kEngineSlots) of this warp is tracked by lane s: busy, owner lane, phase
  bool pinf = false;                 // this lane's command has its page in a slot
  bool sbusy = false;
  u32 sowner = 0, spar = 0;
  uint8_t* stage = nullptr;
  u64* bars = nullptr;
  if constexpr (kBulk) {
    stage = slots + (u64)(threadIdx.x >> 5) * kEngineSlots * kBlockBytes;
    bars = reinterpret_cast<u64*>(slots + (u64)kCtaWarps * kEngineSlots * kBlockBytes) + (threadIdx.x >> 5) * kEngineSlots;
    if (lane < (u32)kEngineSlots) mbar_init(&bars[lane]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
  }
  while (true) {
    bool did = false;
    if constexpr (kBulk) {
      // ---- slots whose bytes landed: copy them out to HBM (or to the host store for writes)
      const bool sdone = lane < (u32)kEngineSlots && sbusy && mbar_test(&bars[lane], spar);
      u32 dm = __ballot_sync(FULL, sdone);
      if (dm) {
        did = true;
        u32 moved = 0;
        const u32 dm0 = dm;
        while (dm) {
          const int sl = __ffs(dm) - 1;
          dm &= dm - 1;
          const int ow = __shfl_sync(FULL, (int)sowner, sl);
          const u32 op = __shfl_sync(FULL, pop, ow);
          const u32 d = __shfl_sync(FULL, pdev, ow);
          const u64 b = __shfl_sync(FULL, pblk, ow);
          const u64 pr = __shfl_sync(FULL, prp, ow);
          uint4* dst = op == OP_READ ? reinterpret_cast<uint4*>(pr) : reinterpret_cast<uint4*>(c.store_w[d] + (b << kBlockShift));
          const uint4* src = reinterpret_cast<const uint4*>(stage + (u64)sl * kBlockBytes);
          uint4 v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = src[lane + 32 * k];
#pragma unroll
          for (int k = 0; k < 8; ++k) AGILE_FILL_STORE(dst + lane + 32 * k, v[k]);
          moved |= 1u << ow;
        }
        __threadfence();   // page bytes visible before the CQE release of these commands
        __syncwarp();
        if ((moved >> lane) & 1u) { pcp = true; pinf = false; }
        if ((dm0 >> lane) & 1u) { sbusy = false; spar ^= 1u; }
      }
      // ---- start bulk copies of the oldest fetched commands into free slots
      u32 freeslots = ~__ballot_sync(FULL, lane < (u32)kEngineSlots && sbusy) & ((1u << kEngineSlots) - 1u);
      u32 taken = 0;
      while (freeslots) {
        const int ow = oldest_lane(pv && !pcp && !pinf && !((taken >> lane) & 1u), pseq);
        if (ow < 0) break;
        did = true;
        const int sl = __ffs(freeslots) - 1;
        freeslots &= freeslots - 1;
        taken |= 1u << ow;
        const u32 op = __shfl_sync(FULL, pop, ow);
        const u32 d = __shfl_sync(FULL, pdev, ow);
        const u64 b = __shfl_sync(FULL, pblk, ow);
        const u64 pr = __shfl_sync(FULL, prp, ow);
        const void* src = op == OP_READ ? reinterpret_cast<const void*>(c.store[d] + (b << kBlockShift))
                                        : reinterpret_cast<const void*>(pr);
        if (lane == 0) bulk_page_to_smem(stage + (u64)sl * kBlockBytes, src, &bars[sl]);
        if (lane == (u32)ow) pinf = true;
        if (lane == (u32)sl) { sbusy = true; sowner = (u32)ow; }
      }
    }
    // ---- start moving the bytes of the two oldest fetched commands: the loads (host link
    //      latency) stay in flight while this pass posts completions and fetches new SQEs
    const u32 tocopy = kBulk ? 0u : __ballot_sync(FULL, pv && !pcp);
    int lk[kPages];
    uint4 v[kPages][8];
    uint4* tk[kPages];
#pragma unroll
    for (int p = 0; p < kPages; ++p) { lk[p] = -1; tk[p] = nullptr; }
    if (tocopy) {
      did = true;
      u32 taken = 0;   // lanes already picked this pass
#pragma unroll
      for (int p = 0; p < kPages; ++p) {
        // oldest first: no lane starves behind new fetches
        const int l = oldest_lane(pv && !pcp && !((taken >> lane) & 1u), pseq);
        lk[p] = l;
        if (l < 0) break;
        taken |= 1u << l;
        const u32 op = __shfl_sync(FULL, pop, l);
        const u32 d = __shfl_sync(FULL, pdev, l);
        const u64 b = __shfl_sync(FULL, pblk, l);
        const u64 pr = __shfl_sync(FULL, prp, l);
        const uint4* src = op == OP_READ ? reinterpret_cast<const uint4*>(c.store[d] + (b << kBlockShift))
                                         : reinterpret_cast<const uint4*>(pr);
        tk[p] = op == OP_READ ? reinterpret_cast<uint4*>(pr) : reinterpret_cast<uint4*>(c.store_w[d] + (b << kBlockShift));
#pragma unroll
        for (int k = 0; k < 8; ++k) v[p][k] = __ldcg(src + lane + 32 * k);
      }
    }
    const u64 now = gtimer();
    // ---- post due completions (device_post / stall, nvme_queue.py:266-279, ssd_model.py:200-206)
    const bool due = pv && pcp && pdue <= now;
    if (__ballot_sync(FULL, due)) {
      if (due && !plogged) {
        // the completion is reported at its model time (the bytes moved earlier)
        log_ev(c, WHO_DEV | pdev, M_SSD, A_COMPLETE, pdev, pq, pslot, pop, pblk);
        if (pop == OP_READ) bytes_r += kBlockBytes; else bytes_w += kBlockBytes;
        plogged = true;
      }
      u32 grp = __match_any_sync(FULL, due ? pq : 0xffffffffu);
      if (!due) grp = 0;
      const u32 rank = __popc(grp & lanemask_lt());
      const u32 n = __popc(grp);
      u64 tail = 0;
      u32 take = 0;
      if (due && rank == 0) {
        CqWords* cw = &c.cqw[pq];
        tail = cw->dev_tail;
        const u64 hdb = ld_acquire(&cw->host_db);
        const u64 room = (u64)Dq - (tail - hdb);
        take = (u32)min((u64)n, room);
        cw->dev_tail = tail + take;
      }
      const u32 leader = grp ? (u32)(__ffs(grp) - 1) : lane;
      tail = __shfl_sync(FULL, tail, leader);
      take = __shfl_sync(FULL, take, leader);
      if (due) {
        if (rank < take) {
          const u64 v = tail + rank;
          u64* cqe = reinterpret_cast<u64*>(c.cqe + (u64)pq * Dq + (u32)(v & (Dq - 1)));
          const u64 phase = 1ull - ((v / Dq) & 1ull);
          const u64 w1 = (u64)pq << 16 | (u64)pslot << 32 | phase << 48;   // SQID | CID | P
          cqe[0] = 0ull;
          st_release(cqe + 1, w1);
          log_ev(c, WHO_DEV | pdev, M_SSD, A_CQE_POST, pq, v, pslot, pq);
          pv = false;
          did = true;
        } else if (!pstalled) {
          log_ev(c, WHO_DEV | pdev, M_SSD, A_CQE_STALL, pq, pslot, pq);
          atomicAdd(&c.stats[S_CQE_STALLS], 1ull);
          pstalled = true;
        }
      }
    }
    // ---- fetch newly published SQEs into free lanes (on_sq_doorbell/_fetch, ssd_model.py:138-166);
    //      while bytes are still to be moved only every 4th pass pays the doorbell round trips
    const u32 freeb = __ballot_sync(FULL, !pv);
    u32 nfree = __popc(freeb);
    bool newcmd = false;
    ++pass;
    const u32 ncopy = __popc(__ballot_sync(FULL, pv && !pcp && !pinf));
    const bool fetch_now = ncopy < 8 || (pass & 3u) == 0;
    if (nfree && nq && fetch_now) {
      u32 assigned = 0;   // free lanes handed out in earlier chunks
      for (u32 b0 = 0; b0 < nq && nfree; b0 += 32) {
        const u32 k = b0 + lane;
        const bool own = k < nq;
        u32 q = 0;
        u64 f = 0, avail = 0;
        if (own) {
          q = ew + ((k + rr) % nq) * E;
          f = c.sqw[q].fetched;
          avail = (ld_acquire(&c.sqw[q].dbl) >> 1) - f;
        }
        const u32 a = (u32)min(avail, (u64)32);
        u32 pre = a;   // inclusive scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const u32 t = __shfl_up_sync(FULL, pre, o);
          if (lane >= (u32)o) pre += t;
        }
        pre -= a;   // exclusive
        const u32 take = pre >= nfree ? 0u : min(a, nfree - pre);
        if (take) c.sqw[q].fetched = f + take;
        u32 tot = take;
#pragma unroll
        for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(FULL, tot, o);
        if (!tot) continue;
        // distribute to free lanes in order
        const u32 fr = __popc(freeb & lanemask_lt());
        const bool isfree = !pv;
        for (u32 s = 0; s < 32; ++s) {
          const u32 ps = __shfl_sync(FULL, pre, s);
          const u32 ts = __shfl_sync(FULL, take, s);
          const u32 qs = __shfl_sync(FULL, q, s);
          const u64 fs = __shfl_sync(FULL, f, s);
          if (isfree && !newcmd && ts && fr >= assigned + ps && fr < assigned + ps + ts) {
            newcmd = true;
            pq = qs;
            const u64 v = fs + (fr - assigned - ps);
            pslot = (u32)(v & (Ds - 1));
          }
        }
        nfree -= tot;
        assigned += tot;
      }
      rr++;
    }
    const u32 nb = __ballot_sync(FULL, newcmd);
    if (nb) {
      did = true;
      u64 arrival = 0;
      if (newcmd) {
        const u32 idx = pq * Ds + pslot;
        if (ld_acquire(&c.sq_state[idx]) != SQ_ISSUED) set_error(c, E_PROTOCOL, pq, pslot);   // ssd_model.py:158-160
        const uint4* e = c.sqe + (u64)idx * 4;
        const uint4 e0 = e[0], e1 = e[1], e2 = e[2];
        pop = (e0.x & 0xffu) == 0x02u ? OP_READ : OP_WRITE;
        pdev = e0.y - 1;
        prp = (u64)e1.z | ((u64)e1.w << 32);
        pblk = (u64)e2.z | ((u64)e2.w << 32);
        if (pdev >= c.num_devices || pblk >= c.store_blocks[pdev]) {
          set_error(c, E_OUT_OF_RANGE, pdev, pblk);
          pdev = 0;
          pblk = 0;
        }
        {
          // the PRP of a cache command must be a line of this cache (raw commands carry
          // caller buffers and are not checked)
          const u64 lo = (u64)(uintptr_t)c.lines, hi = lo + ((u64)c.num_lines << kBlockShift);
          const CmdCtx& xc = c.cmd[idx];
          if (xc.line != NONE && (prp < lo || prp >= hi || ((prp - lo) & 4095u))) {
            set_error(c, E_ILLEGAL_STATE, prp, 0xE0000000ull | (u64)__LINE__);
            prp = lo;
          }
        }
        log_ev(c, WHO_DEV | pdev, M_SSD, A_FETCH, pdev, pq, pslot, pslot);
        arrival = ld_relaxed(&c.sqw[pq].db_time) + c.model.fetch_ns;
      }
      // completion time: link mode = as soon as the bytes moved; model mode replays the channels
      if (c.model.link_mode) {
        if (newcmd) pdue = 0;
      } else if (c.model.jitter == 0 || c.model.jitter_ns == 0) {
        model_schedule_rr(c, newcmd, pdev, pop, arrival, pdue);
      } else {
        u32 t2 = nb;
        while (t2) {
          const int l = __ffs(t2) - 1;
          const u32 dl = __shfl_sync(FULL, pdev, l);
          const u32 same = __ballot_sync(FULL, newcmd && pdev == dl) & t2;
          t2 &= ~same;
          model_schedule_batch(c, dl, same, pop, arrival, pdue);
        }
      }
      if (newcmd) {
        pv = true; pcp = false; plogged = false; pstalled = false;
        pseq = seq + __popc(nb & lanemask_lt());
      }
      seq += __popc(nb);
      if (lane == 0) atomicAdd(&c.stats[S_FETCHED], (u64)__popc(nb));
    }
    // ---- finish the page moves started at the top of the pass
    if (lk[0] >= 0) {
      u32 moved = 0;
#pragma unroll
      for (int p = 0; p < kPages; ++p) {
        if (lk[p] < 0) break;
#pragma unroll
        for (int k = 0; k < 8; ++k) AGILE_FILL_STORE(tk[p] + lane + 32 * k, v[p][k]);
        moved |= 1u << lk[p];
      }
      __threadfence();   // page bytes visible before the CQE release of these commands
      __syncwarp();
      if ((moved >> lane) & 1u) pcp = true;
    }
    // ---- exit once the service is done and nothing is in service
    const bool busy = __ballot_sync(FULL, pv) != 0;
    if (!busy) {
      int stop = 0;
      if (lane == 0) stop = ld_acquire(&c.run->engine_stop) != 0 || aborted(c);
      if (__shfl_sync(FULL, stop, 0)) break;
    } else if (aborted(c)) {
      break;
    }
    if (!did) {
      nap(idle);
      idle = min(idle * 2, 512u);
    } else {
      idle = 32;
    }
  }
  u64 br = bytes_r, bw = bytes_w;
#pragma unroll
  for (int o = 16; o; o >>= 1) { br += __shfl_xor_sync(FULL, br, o); bw += __shfl_xor_sync(FULL, bw, o); }
  if (lane == 0) {
    if (br) atomicAdd(&c.stats[S_BYTES_READ], br);
    if (bw) atomicAdd(&c.stats[S_BYTES_WRITTEN], bw);
  }
}

// ======================================================================= launch skeleton
// One AGILE run = two grids on one stream:
//   infra grid  [engine CTAs][service CTAs]  — register-rich (no spills in the engine/service),
//   user grid   the workload's CTAs           — its own register budget (UserMinCtas<Work>).
// The user grid is launched with programmatic stream serialization (PDL) and every infra CTA
// executes griddepcontrol.launch_dependents as its first instruction, so no user CTA starts
// before every engine and service CTA is resident: a spinning user waits only on CTAs that are
// already running (forward progress by construction; PAPER.md:811-819 puts the service in the
// first scheduled block for the same reason).  The user grid never calls griddepcontrol.wait.
// The last user CTA out waits for the infra CTAs to exit, so the next run on the stream (which
// resets the run words) cannot overlap this run's infra grid.

__device__ __forceinline__ void user_done(const DevCtx& c, u32 n_users) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const u32 n = atomicAdd(&c.run->users_done, 1u) + 1;
    if (n == n_users) {
      const u32 ninfra = c.n_engine_ctas + c.n_service_ctas;
      Spin sp;
      while (ld_acquire(&c.run->infra_exited) < ninfra)
        if (!sp.again(c, 1024, __LINE__ + 100000 * SPIN_FILE_ID)) break;
    }
  }
}

// kBulk: pages move through the TMA bulk-copy unit into shared-memory slots (the register budget
// no longer holds pages in flight); the infra grid's CTAs then fit beside user CTAs on their SMs
// Two infra kernels, picked per context (config engine.copy): kBulk = false moves pages through
// registers (4 per engine-warp pass; 236 registers, one infra CTA per SM: the infra SMs are the
// engine's alone, which keeps the miss path's latency lowest); kBulk = true moves them through the
// TMA bulk-copy unit into shared-memory slots (128 registers: two user CTAs fit beside each infra
// CTA, which gives hit-heavy runs ~8 % more user CTAs and the side-stream runs a smaller footprint)
template <bool kBulk>
__global__ void __launch_bounds__(kCtaThreads, kBulk ? 2 : 1)
    agile_infra_kernel(const __grid_constant__ DevCtx c, const Launch L) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(128) uint8_t infra_smem[];
  const u32 warp = threadIdx.x >> 5;
  if (blockIdx.x < c.n_engine_ctas) {
    const u32 ew = blockIdx.x * kCtaWarps + warp;
    if (ew < c.engine_warps) engine_main<kEnginePages, kBulk>(c, ew, infra_smem);
  } else {
    const u32 sw = (blockIdx.x - c.n_engine_ctas) * kCtaWarps + warp;
    if (sw < c.service_warps) service_main<kBulk ? 4 : 8>(c, L, sw);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(&c.run->infra_exited, 1u);
  }
}

// CTAs per SM a workload's user grid targets (its register budget): AGILE_MIN_CTAS unless the
// workload declares kMinCtas
template <class W, class = void>
struct UserMinCtas { static constexpr int v = AGILE_MIN_CTAS; };
template <class W>
struct UserMinCtas<W, std::void_t<decltype(W::kMinCtas)>> { static constexpr int v = W::kMinCtas; };

template <class Work>
// __grid_constant__: the device functions take the context and the workload by reference; without
// it every thread would copy both structs from the parameter bank into local memory at entry.
__global__ void __launch_bounds__(kCtaThreads, UserMinCtas<Work>::v)
    agile_user_kernel(const __grid_constant__ DevCtx c, const Launch L, const __grid_constant__ Work work) {
  __shared__ u32 s_solo;
  if (threadIdx.x == 0) {
    const u32 prev = atomicAdd(&c.run->users_started, 1u);
    s_solo = (prev & kInfraGaveUp) ? 1u : 0u;
    // the infra grid already left (this grid could not start beside it): outside profiling mode
    // that is an error; in profiling mode the workload runs alone (an all-hit replay needs no
    // engine or service; a miss then ends in the watchdog)
    if (s_solo && !c.solo_ok) set_error(c, E_LIVELOCK, 1, __LINE__ + 100000 * SPIN_FILE_ID);
  }
  __syncthreads();
  if (!s_solo || c.solo_ok) work.run(c, blockIdx.x, L.n_user_ctas);
  user_done(c, L.n_user_ctas);
}

// Fused single-grid launch (config `launch.mode = fused`): the roles are taken by arrival ticket —
// the first CTAs to start become the engine and the service — so users again wait only on
// resident CTAs.  One register budget for all roles (2 CTAs per SM, 2-page engine passes).  This
// is the mode a kernel-serialising profiler can capture (ncu replays one kernel at a time, which
// the two co-running grids of the split launch cannot survive); the split launch is the default.
template <class Work>
__global__ void __launch_bounds__(kCtaThreads, 2)
    agile_fused_kernel(const __grid_constant__ DevCtx c, const Launch L, const __grid_constant__ Work work) {
  __shared__ u32 s_ticket;
  if (threadIdx.x == 0) s_ticket = atomicAdd(&c.run->ticket, 1u);
  __syncthreads();
  u32 t = s_ticket;
  const u32 warp = threadIdx.x >> 5;
  if (t < c.n_engine_ctas + c.n_service_ctas) {
    if (t < c.n_engine_ctas) {
      const u32 ew = t * kCtaWarps + warp;
      if (ew < c.engine_warps) engine_main<2>(c, ew);
    } else {
      const u32 sw = (t - c.n_engine_ctas) * kCtaWarps + warp;
      if (sw < c.service_warps) service_main(c, L, sw);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&c.run->infra_exited, 1u);
    }
    return;
  }
  if (threadIdx.x == 0) atomicAdd(&c.run->users_started, 1u);
  work.run(c, t - c.n_engine_ctas - c.n_service_ctas, L.n_user_ctas);
  user_done(c, L.n_user_ctas);
}

}  // namespace agile
