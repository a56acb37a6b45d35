// agile_share.cuh — Share Table (share_table.py:52-200) and the table-aware API verbs
// (gpu_api.py:164-278 with self.table set): coherence of user-owned buffers.
//
// An open-addressed table in HBM maps a block key to the one live user buffer (WaitNode + its
// 4 KiB destination) holding that block; later requesters receive that buffer instead of a copy,
// with a reference count (refcount-collapsed MOESI: Exclusive / Shared / Modified).  The table
// outranks the software cache: reads and writes consult it first.  The last release of a Modified
// entry drains the buffer's bytes into the cache as a MODIFIED line (install_modified), which a
// flush or an eviction (WB_EVICT) later writes back.
//
// Concurrency: every operation on key k holds the lock of k's home bucket (share_table.py:66-68
// hash) for its table update only — never across a cache access or a wait (the reference's lock
// discipline).  Slots are claimed with a CAS on their key word, so keys of different home buckets
// never collide on a slot; a used slot only ever becomes a tombstone, never empty again, so probe
// chains stay intact.  Entry fields other than the key are read and written under the key's home
// lock.  Writes into a shared buffer happen under that lock too, so an observer holding it (the
// coherence test's observe instant) sees either the old or the new bytes, never a torn mix.
#pragma once
#include "agile_core.cuh"
#undef SPIN_FILE_ID
#define SPIN_FILE_ID 3

namespace agile {

struct ShareEntry {
  u64 key;      // SE_EMPTY, SE_TOMB, or key + 2
  u64 node;     // WaitNode* of the registered buffer
  u32 ref;      // reference count
  u32 state;    // SH_E / SH_S / SH_M, | SH_RETIRING while the last release propagates
  u32 owner;    // who registered (duty_transfer trace)
  u32 pad;
};
static_assert(sizeof(ShareEntry) == 32, "ShareEntry is 32 B");
constexpr u64 SE_EMPTY = 0, SE_TOMB = 1;
enum : u32 { SH_E = 0, SH_S = 1, SH_M = 2 };
constexpr u32 SH_RETIRING = 0x100;

__device__ __forceinline__ u32 st_home(const DevCtx& c, u64 key) {   // share_table.py:66-68
  const u64 h = ((u64)key_dev(key) * 0x9E3779B1ull) ^ (key_blk(key) * 0x85EBCA77ull);
  return (u32)(h & (c.st_buckets - 1));
}
__device__ __forceinline__ bool st_lock(const DevCtx& c, u32 h, u32 who = WHO_USER) {
  Spin sp;
  while (atom_cas_acquire(&c.st_lock[h], 0u, 1u) != 0u) {
    lk_failed(c, lk_bucket_id(c, h), who);
    if (!sp.again(c, 256, __LINE__ + 100000 * SPIN_FILE_ID)) { lk_stop_waiting(c); return false; }
  }
  lk_acquired(c, lk_bucket_id(c, h));
  return true;
}
__device__ __forceinline__ void st_unlock(const DevCtx& c, u32 h) {
  lk_released(c, lk_bucket_id(c, h));
  st_release(&c.st_lock[h], 0u);
}

// linear probe from the home bucket (share_table.py:70-86): the entry's slot or -1, with the first
// insertable slot (tombstone or empty) and the key word seen there
__device__ int st_find(const DevCtx& c, u64 key, u32& ins, u64& ins_seen) {
  const u32 mask = c.st_buckets - 1;
  u32 idx = st_home(c, key);
  ins = NONE;
  ins_seen = 0;
  for (u32 n = 0; n < c.st_buckets; ++n) {
    const u64 k = ld_relaxed(&c.st[idx].key);
    if (k == SE_EMPTY) {
      if (ins == NONE) { ins = idx; ins_seen = k; }
      return -1;
    }
    if (k == SE_TOMB) {
      if (ins == NONE) { ins = idx; ins_seen = k; }
    } else if (k == key + 2) {
      return (int)idx;
    }
    idx = (idx + 1) & mask;
  }
  return -1;
}

__device__ __forceinline__ void st_log_share(const DevCtx& c, u32 who, u64 key, const ShareEntry& e) {
  log_ev(c, who, M_TABLE, A_SHARE, key_dev(key), key_blk(key), e.ref, e.state & 0xFFu);
}

// lookup_or_register (share_table.py:90-121): returns the tracked buffer; registered = mine
// became the tracked buffer (Exclusive, the caller owns the fill).  Either way the caller holds
// one reference.  Per lane.
__device__ WaitNode* st_lookup_or_register(const DevCtx& c, u64 key, WaitNode* mine, u32 who, bool& registered) {
  registered = false;
  const u32 h = st_home(c, key);
  if (!st_lock(c, h)) return mine;
  WaitNode* res = mine;
  while (true) {
    u32 ins; u64 seen;
    const int f = st_find(c, key, ins, seen);
    if (f >= 0) {
      ShareEntry& e = c.st[f];
      e.ref += 1;
      e.state &= ~SH_RETIRING;
      if ((e.state & 0xFFu) == SH_E) e.state = SH_S;
      st_log_share(c, who, key, e);
      res = reinterpret_cast<WaitNode*>(e.node);
      break;
    }
    if (ins == NONE) { set_error(c, E_ILLEGAL_STATE, key, 0x5E000000ull | __LINE__); break; }   // table full
    if (atomicCAS(reinterpret_cast<unsigned long long*>(&c.st[ins].key), seen, key + 2) != seen) continue;
    ShareEntry& e = c.st[ins];
    e.node = (u64)(uintptr_t)mine;
    e.ref = 1;
    e.state = SH_E;
    e.owner = who;
    log_ev(c, who, M_TABLE, A_REGISTER, key_dev(key), key_blk(key));
    registered = true;
    break;
  }
  st_unlock(c, h);
  return res;
}

// acquire_if_present (share_table.py:123-142): a reference on an existing entry, else null
__device__ WaitNode* st_acquire_if_present(const DevCtx& c, u64 key, u32 who) {
  const u32 h = st_home(c, key);
  if (!st_lock(c, h)) return nullptr;
  u32 ins; u64 seen;
  const int f = st_find(c, key, ins, seen);
  WaitNode* res = nullptr;
  if (f >= 0) {
    ShareEntry& e = c.st[f];
    e.ref += 1;
    e.state &= ~SH_RETIRING;
    if ((e.state & 0xFFu) == SH_E) e.state = SH_S;
    st_log_share(c, who, key, e);
    res = reinterpret_cast<WaitNode*>(e.node);
  }
  st_unlock(c, h);
  return res;
}

// release (share_table.py:151-196), table part, per lane.  Returns 0 (references remain or the
// entry retired), 1 (last reference of a Modified entry: the buffer's bytes were snapshotted
// into `snap` under the lock; the caller installs them into the cache, then st_finish_release).
__device__ int st_release_begin(const DevCtx& c, u64 key, u32 who, uint4* snap, int& slot) {
  const u32 h = st_home(c, key);
  slot = -1;
  if (!st_lock(c, h)) return 0;
  u32 ins; u64 seen;
  const int f = st_find(c, key, ins, seen);
  if (f < 0) {   // NotRegistered
    st_unlock(c, h);
    set_error(c, E_ILLEGAL_STATE, key, 0x5E000000ull | __LINE__);
    return 0;
  }
  ShareEntry& e = c.st[f];
  if (e.ref == 0) {   // DoubleRelease
    st_unlock(c, h);
    set_error(c, E_ILLEGAL_STATE, key, 0x5E000000ull | __LINE__);
    return 0;
  }
  e.ref -= 1;
  log_ev(c, who, M_TABLE, A_RELEASE, key_dev(key), key_blk(key), e.ref);
  int rc = 0;
  if (e.ref == 0) {
    if ((e.state & 0xFFu) == SH_M) {
      e.state |= SH_RETIRING;
      const uint4* b = reinterpret_cast<const uint4*>(reinterpret_cast<WaitNode*>(e.node)->dst);
      for (u32 k = 0; k < 256; ++k) snap[k] = __ldcg(b + k);
      if (e.owner != who) log_ev(c, who, M_TABLE, A_DUTY_TRANSFER, key_dev(key), key_blk(key), e.owner);
      slot = f;
      rc = 1;
    } else {
      st_relaxed(&e.key, SE_TOMB);   // unmodified: nothing to propagate, the entry retires now
    }
  }
  st_unlock(c, h);
  return rc;
}

// after the propagation: the entry disappears unless a lookup revived it meanwhile
__device__ void st_finish_release(const DevCtx& c, u64 key, int slot) {
  const u32 h = st_home(c, key);
  if (!st_lock(c, h)) return;
  ShareEntry& e = c.st[slot];
  if (ld_relaxed(&e.key) == key + 2 && (e.state & SH_RETIRING) && e.ref == 0) st_relaxed(&e.key, SE_TOMB);
  st_unlock(c, h);
}

// ------------------------------------------------------------------ table-aware verbs (warp)

// release_shared (gpu_api.py:229-231 -> ShareTable.release), warp-collective: the last release of
// a Modified entry installs the buffer's bytes into the cache as a MODIFIED line first.
// snap: the lane's 4 KiB snapshot page; tmp: a WaitNode of the lane not tracked by the table.
__device__ void release_shared_warp(const DevCtx& c, bool active, u64 key, uint4* snap, WaitNode* tmp, u32 who,
                                    u32 sq) {
  int slot = -1;
  const bool prop = active && st_release_begin(c, key, who, snap, slot) == 1;
  if (!__any_sync(FULL, prop)) return;
  write_block_warp(c, prop, key, tmp, snap, who, sq, false);   // install_modified
  if (prop) {
    log_ev(c, who, M_TABLE, A_PROPAGATE, key_dev(key), key_blk(key));
    st_finish_release(c, key, slot);
  }
}

// async_read with the table (gpu_api.py:164-190): the caller's buffer is registered and filled
// through the cache, or an already tracked buffer is returned in `eff` (wait on eff, read eff->dst).
__device__ void async_read_t(const DevCtx& c, bool active, u64 key, WaitNode* node, uint4* dst, u32 who, u32 sq,
                             WaitNode*& eff) {
  eff = node;
  if (active && buffer_busy(c, node)) active = false;
  bool go = active;
  if (c.st_buckets && active) {
    node->dst = (u64)(uintptr_t)dst;
    node->done = 0;
    node->t_issue = 0;   // (async_read_warp stamps it; the busy check above already ran)
    bool reg;
    WaitNode* sh = st_lookup_or_register(c, key, node, who, reg);
    if (!reg) { eff = sh; go = false; }
  }
  async_read_warp(c, go, key, node, dst, who, sq);
}

// async_write with the table (gpu_api.py:192-227): a tracked buffer takes the bytes in place
// (Modified; no device write, node released at once); otherwise the cache write path, one attempt
// at a time, the table re-checked after every retry (a reader may register the block meanwhile).
__device__ void async_write_t(const DevCtx& c, bool active, u64 key, WaitNode* node, const uint4* src, u32 who,
                              u32 sq, uint4* snap, WaitNode* tmp) {
  if (!c.st_buckets) {
    async_write_warp(c, active, key, node, src, who, sq);
    return;
  }
  const u32 lane = lane_id();
  if (active && buffer_busy(c, node)) active = false;
  bool want = active;
  Spin sp;
  while (__any_sync(FULL, want)) {
    WaitNode* sh = want ? st_acquire_if_present(c, key, who) : nullptr;
    const bool shared = sh != nullptr;
    const u64 shdst = shared ? sh->dst : 0ull;
    // the tracked buffer must hold its data before it is overwritten
    if (shared) {
      Spin s2;
      while (ld_acquire(&sh->done) == 0)
        if (!s2.again(c, 1024, __LINE__ + 100000 * SPIN_FILE_ID)) break;
    }
    u32 sb = __ballot_sync(FULL, shared);
    while (sb) {
      const int l = __ffs(sb) - 1;
      sb &= sb - 1;
      const u64 kl = __shfl_sync(FULL, key, l);
      const u32 h = st_home(c, kl);
      int ok = 1;
      if (lane == (u32)l) ok = st_lock(c, h) ? 1 : 0;
      if (!__shfl_sync(FULL, ok, l)) continue;
      const uint4* s0 = reinterpret_cast<const uint4*>(__shfl_sync(FULL, (u64)(uintptr_t)src, l));
      uint4* d0 = reinterpret_cast<uint4*>(__shfl_sync(FULL, shdst, l));
      copy_page_warp(s0, d0);
      __threadfence();
      __syncwarp();
      if (lane == (u32)l) {
        log_ev(c, who, M_API, A_WRITE_COMMIT, key_dev(key), key_blk(key), *reinterpret_cast<const u64*>(src));
        u32 ins; u64 seen;
        const int f = st_find(c, key, ins, seen);   // mark_buffer_modified (share_table.py:143-149)
        if (f >= 0) {
          c.st[f].state = (c.st[f].state & SH_RETIRING) | SH_M;
          log_ev(c, who, M_TABLE, A_MODIFIED, key_dev(key), key_blk(key));
        }
        st_unlock(c, h);
      }
      __syncwarp();
    }
    release_shared_warp(c, shared, key, snap, tmp, who, sq);
    if (shared) {
      st_release(&node->done, 1u);   // no durability handle (the reference returns None)
      want = false;
    }
    const bool rest = want;
    want = write_block_warp(c, rest, key, node, src, who, sq, true, true) && rest;
    if (__any_sync(FULL, want) && !sp.again(c, 2048, __LINE__ + 100000 * SPIN_FILE_ID)) break;
  }
}

// SoftwareCache.flush (software_cache.py:283-298), one warp: every MODIFIED line is written back
// (WB_KEEP: BUSY until durable, then READY) and waited for.  nodes: 32 WaitNodes.  Returns the
// number of lines written back.
__device__ u64 flush_warp(const DevCtx& c, WaitNode* nodes, u32 who, u32 sq) {
  const u32 lane = lane_id();
  u64 total = 0;
  for (u32 l0 = 0; l0 < c.num_lines; l0 += 32) {
    const u32 line = l0 + lane;
    bool pend = line < c.num_lines && tw_state(ld_relaxed(&c.tags[line])) == ST_MODIFIED;
    Spin sp;
    while (__any_sync(FULL, pend)) {
      bool own = false;
      u64 key = 0;
      if (pend) {
        const u32 set = line / c.ways;
        if (atom_cas_acquire(&c.set_lock[set], 0u, 1u) == 0u) {
          const u64 w = ld_relaxed(&c.tags[line]);
          if (tw_state(w) != ST_MODIFIED) {
            pend = false;   // evicted (written back) or rewritten meanwhile
          } else if (tw_pins(w) == 0) {
            const u32 ver = tw_ver(w) + 1;
            if (atom_cas_acqrel(&c.tags[line], w, tw_make(ST_BUSY, tw_key(w), ver, tw_ref(w), 0)) == w) {
              st_relaxed(&c.wl[line], ((u64)(ver & 0x1FFu)) << 55);
              key = tw_key(w);
              WaitNode* nd = nodes + lane;
              nd->dst = 0;
              nd->done = 0;
              own = wl_push(c, line, ver, nd);
              log_state(c, who, line, ST_MODIFIED, ST_BUSY, key);
            }
          }
          st_release(&c.set_lock[set], 0u);
        }
      }
      if (!submit_warp(c, own, key_dev(key), key_blk(key), line, K_WB_KEEP, OP_WRITE, 0, key, who, sq)) return total;
      const u32 n = __popc(__ballot_sync(FULL, own));
      total += n;
      if (lane == 0 && n) atomicAdd(&c.stats[S_WRITEBACKS], (u64)n);
      if (!wait_nodes_warp(c, own, nodes + lane)) return total;
      if (own) pend = false;
      if (__any_sync(FULL, pend) && !sp.again(c, 1024, __LINE__ + 100000 * SPIN_FILE_ID)) return total;
    }
  }
  return total;
}

}  // namespace agile
