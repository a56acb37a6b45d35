// agile_work.cuh — user-side workloads (the consumers of the device library):
//   SeqWork        serialized async_read+wait stream (golden hit/miss/eviction parity)
//   ReadsWork      CTC sync/async epochs (bench/ctc.py:27-111)            — K8
//   LoopWork       closed-loop 4 KiB random reads (bench/bandwidth.py:20-68) — K9
//   GatherWork     prefetch + array_get gather epochs (bench/sweeps.py:39-88)
//   EmbBagWork     DLRM embedding-bag over cached rows                    — K5
#pragma once
#include <climits>
#include "agile_core.cuh"
#include "agile_share.cuh"
#undef SPIN_FILE_ID
#define SPIN_FILE_ID 2

namespace agile {

// grid barrier among user CTAs (the epoch Rendezvous, sim_core.py:139-159). All user CTAs are
// co-resident by construction (the host sizes the grid from occupancy for these workloads).
__device__ __forceinline__ bool user_grid_barrier(const DevCtx& c, u32 n_user_ctas) {
  // one user CTA: the CTA barrier is the rendezvous (the abort check rides on it, uniformly)
  if (n_user_ctas == 1) return __syncthreads_or(threadIdx.x == 0 && aborted(c)) == 0;
  __syncthreads();
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    s_ok = 1;
    const u32 gen = ld_acquire(&c.run->bar_gen);
    __threadfence();
    if (atomicAdd(&c.run->bar_count, 1u) == n_user_ctas - 1) {
      st_relaxed(&c.run->bar_count, 0u);
      st_release(&c.run->bar_gen, gen + 1);
    } else {
      Spin sp;
      while (ld_acquire(&c.run->bar_gen) == gen)
        if (!sp.again(c, 512, __LINE__ + 100000 * SPIN_FILE_ID)) { s_ok = 0; break; }
    }
  }
  __syncthreads();
  return s_ok != 0;
}

// compute phase of the benchmarks: Delay(compute_ns) of the reference (bench/ctc.py:81-83).  The
// warp sleeps in 256 ns steps and lane 0 alone reads %globaltimer, so a computing CTA does not
// steal issue slots from co-resident engine/service warps.
__device__ __forceinline__ void compute_spin(u64 ns) {
  if (!ns) return;
  int more = 1;
  u64 t0 = 0;
  if (lane_id() == 0) t0 = gtimer();
  while (more) {
    __nanosleep(256);
    if (lane_id() == 0) more = gtimer() - t0 < ns;
    more = __shfl_sync(0xffffffffu, more, 0);
  }
}

__device__ __forceinline__ u32 user_who(u32 uidx) { return WHO_USER | (uidx * kCtaThreads + threadIdx.x); }

// Read-side ordering of the cached-row readers (embedding-bag hot path).  Every tag word is read
// with a strong gpu-scope load and every row with an L2 (.cg) load, so L2 — the single point of
// coherence — serves both; the writer side publishes page bytes before the READY tag through
// release/acquire (engine fence -> CQE release -> service acquire -> tag release), and a claim
// bumps the tag's version before the line's bytes are overwritten.  The reader needs:
//   READY seen -> row read:  the confirming tag load is an acquire (ld.acquire.gpu);
//   row read -> tag re-read: the re-read's address carries a data dependency on the row values
//                            (dep_zero over a warp reduction), so it cannot be issued before
//                            every row load of the warp returned.
// No fence.acq_rel (MEMBAR + L1 invalidate) is issued on the hit path.

// ------------------------------------------------------------------ SeqWork
struct SeqWork {
  const u32* dev;
  const u64* blk;
  long long n;
  signed char* outcome;   // 0 hit, 1 miss, 2 attach
  u64* victim;            // evicted key or ~0
  uint4* pages;           // optional n * 4 KiB
  uint4* scratch;         // 4 KiB
  WaitNode* nodes;        // 1
  __device__ void run(const DevCtx& c, u32 uidx, u32 nusers) const {
    if (uidx != 0 || threadIdx.x >= 32) return;
    const u32 lane = lane_id();
    const u32 who = user_who(0) & ~31u;   // task "u0"
    for (long long i = 0; i < n; ++i) {
      if (aborted(c)) return;
      const bool act = lane == 0;
      const u64 key = make_key(dev[i], blk[i]);
      if (act) log_ev(c, who, M_API, A_ASYNC_READ, dev[i], blk[i]);
      int oc = -1;
      u64 vk = ~0ull;
      async_read_warp(c, act, key, nodes, pages ? pages + i * 256 : scratch, who, 0, &oc, &vk);
      wait_nodes_warp(c, act, nodes);
      if (act) {
        outcome[i] = (signed char)oc;
        victim[i] = vk;
      }
    }
  }
};

// ------------------------------------------------------------------ EvictWork
// SoftwareCache.evict (software_cache.py:268-281 -> _evict_locked, 335-353) per block, serially
// by one warp: a resident READY line with no pins is reset (INVALID, version + 1, evict_reset); a
// MODIFIED line with no pins starts its write-back (BUSY with the old key until durable, then
// INVALID: WB_EVICT); a BUSY or pinned line is DEFERRED.  outcome: 0 RESET, 1 DEFERRED, 2 not
// resident (the reference returns RESET for an absent or INVALID line), 3 WRITEBACK_STARTED.
struct EvictWork {
  const u32* dev;
  const u64* blk;
  long long n;
  signed char* outcome;
  __device__ void run(const DevCtx& c, u32 uidx, u32 nusers) const {
    if (uidx != 0 || threadIdx.x >= 32) return;
    const u32 lane = lane_id();
    const u32 who = user_who(0) & ~31u;
    for (long long i = 0; i < n; ++i) {
      const u64 key = make_key(dev[i], blk[i]);
      u32 line = NONE;
      u64 word = 0;
      probe_lanes(c, lane == 0, key, line, word);
      int oc = 2;
      bool wb = false;
      if (lane == 0 && line != NONE) {
        const u32 set = line / c.ways;
        oc = 1;
        if (atom_cas_acquire(&c.set_lock[set], 0u, 1u) == 0u) {
          const u64 w = ld_relaxed(&c.tags[line]);
          if (!tw_live(w) || tw_key(w) != key) {
            oc = 2;
          } else if (tw_state(w) == ST_READY && tw_pins(w) == 0) {
            const u64 nw = tw_make(ST_INVALID, 0, tw_ver(w) + 1, false, 0);
            if (atom_cas_acqrel(&c.tags[line], w, nw) == w) {
              oc = 0;
              log_ev(c, who, M_CACHE, A_EVICT_RESET, line, key_dev(key), key_blk(key));
              log_state(c, who, line, ST_READY, ST_INVALID, key);
              atomicAdd(&c.stats[S_RESETS], 1ull);
            }
          } else if (tw_state(w) == ST_MODIFIED && tw_pins(w) == 0) {
            const u32 ver = tw_ver(w) + 1;
            st_relaxed(&c.wl[line], ((u64)(ver & 0x1FFu)) << 55);
            if (atom_cas_acqrel(&c.tags[line], w, tw_make(ST_BUSY, key, ver, false, 0)) == w) {
              oc = 3;
              wb = true;
              log_ev(c, who, M_CACHE, A_EVICT_WB, line, key_dev(key), key_blk(key));
              log_state(c, who, line, ST_MODIFIED, ST_BUSY, key);
              atomicAdd(&c.stats[S_WRITEBACKS], 1ull);
            }
          }
          st_release(&c.set_lock[set], 0u);
        }
      }
      line = __shfl_sync(FULL, line, 0);
      if (__any_sync(FULL, wb) && !submit_warp(c, wb, key_dev(key), key_blk(key), line, K_WB_EVICT, OP_WRITE, 0, key, who, 0))
        return;
      if (lane == 0) outcome[i] = (signed char)oc;
      __syncwarp();
    }
  }
};

// ------------------------------------------------------------------ ReadsWork (CTC)
struct ReadsWork {
  const u64* keys;        // [epochs][tasks][reads] request keys
  uint4* bufs;            // [tasks][2][reads] 4 KiB buffers
  WaitNode* nodes;        // [tasks][2][reads]
  u64* digest;            // [tasks] xor of the first 8 bytes of every page read
  u64* epoch_t;           // [epochs + 1] barrier timestamps
  u32 tasks, reads, epochs, async_mode;
  u64 compute_ns;
  static constexpr int MAXR = 64;
  // A CTA's tasks issue their reads as one flat list of (task, i) requests spread over all of
  // the CTA's threads (request f = k * 256 + thread): with fewer than 256 tasks (the reference's
  // 16-task default fills half a warp) the otherwise idle warps issue in parallel, so an epoch's
  // issue takes ceil(tasks_in_cta * reads / 256) access passes per warp instead of `reads`.
  // Each request keeps its task's node and buffer; the epoch barrier still separates the epochs.
  __device__ __forceinline__ u32 cta_tasks(u32 uidx) const {
    return min(tasks - min(tasks, uidx * kCtaThreads), (u32)kCtaThreads);
  }
  // the key of this thread's first request of epoch e (loaded ahead of the epoch's wait, so the
  // issue after the barrier does not start with a dependent load)
  __device__ u64 first_key(u32 uidx, u32 e) const {
    const u32 total = cta_tasks(uidx) * reads;
    if (e >= epochs || threadIdx.x >= total) return 0ull;
    const u32 t = uidx * kCtaThreads + threadIdx.x / reads, i = threadIdx.x % reads;
    return keys[((u64)e * tasks + t) * reads + i];
  }
  __device__ void issue(const DevCtx& c, u32 uidx, u32 e, u32 set, u32 who, u32 sq_start, u64 key0) const {
    const u32 total = cta_tasks(uidx) * reads;
    for (u32 k = 0; k * kCtaThreads < total; ++k) {
      const u32 f = k * kCtaThreads + threadIdx.x;
      const bool a = f < total;
      const u32 t = uidx * kCtaThreads + (a ? f / reads : 0), i = a ? f % reads : 0;
      const u64 key = !a ? 0ull : k == 0 ? key0 : keys[((u64)e * tasks + t) * reads + i];
      const u64 slot = ((u64)t * 2 + set) * reads + i;
      async_read_warp(c, a, key, nodes + (a ? slot : 0), bufs + (a ? slot : 0) * 256, who,
                      sq_start + k + e * reads);
    }
  }
  // wait for the requests this thread issued; the first 8 bytes of each page go into its task's
  // digest (xor: the order of the contributions does not matter)
  __device__ void wait_set(const DevCtx& c, u32 uidx, u32 set) const {
    const u32 total = cta_tasks(uidx) * reads;
    for (u32 k = 0; k * kCtaThreads < total; ++k) {
      const u32 f = k * kCtaThreads + threadIdx.x;
      const bool a = f < total;
      const u32 t = uidx * kCtaThreads + (a ? f / reads : 0), i = a ? f % reads : 0;
      const u64 slot = ((u64)t * 2 + set) * reads + i;
      wait_nodes_warp(c, a, nodes + (a ? slot : 0));
      if (a) {
        const uint2 w = *reinterpret_cast<const uint2*>(bufs + slot * 256);
        atomicXor(reinterpret_cast<unsigned long long*>(digest + t), (u64)w.x | ((u64)w.y << 32));
      }
    }
  }
  __device__ void run(const DevCtx& c, u32 uidx, u32 nusers) const {
    const u32 who = user_who(uidx);
    const u32 sq_start = uidx * kCtaWarps + (threadIdx.x >> 5);
    if (uidx == 0 && threadIdx.x == 0) epoch_t[0] = gtimer();
    if (!async_mode) {
      u64 k0 = first_key(uidx, 0);
      for (u32 e = 0; e < epochs; ++e) {
        issue(c, uidx, e, 0, who, sq_start, k0);
        k0 = first_key(uidx, e + 1);
        wait_set(c, uidx, 0);
        // compute starts only after every task's data arrived (bench/ctc.py:80-83)
        if (!user_grid_barrier(c, nusers)) return;
        if (uidx == 0 && threadIdx.x == 0) epoch_t[e + 1] = gtimer();
        compute_spin(compute_ns);
      }
    } else {
      issue(c, uidx, 0, 0, who, sq_start, first_key(uidx, 0));
      // every task's epoch-0 reads are queued before any epoch-1 read: a task that finished its
      // issue early would otherwise interleave epoch-1 commands into the device FIFO ahead of
      // other tasks' epoch-0 commands and delay the first wait by a whole epoch (the reference's
      // cooperative scheduler issues epoch 0 in one uninterrupted pass, bench/ctc.py:47-58)
      if (!user_grid_barrier(c, nusers)) return;
      for (u32 e = 0; e < epochs; ++e) {
        const u32 cur = e & 1u;
        // the next epoch's fetches ride under this epoch's compute (bench/ctc.py:47-70)
        if (e + 1 < epochs) issue(c, uidx, e + 1, cur ^ 1u, who, sq_start, first_key(uidx, e + 1));
        wait_set(c, uidx, cur);
        if (!user_grid_barrier(c, nusers)) return;
        if (uidx == 0 && threadIdx.x == 0) epoch_t[e + 1] = gtimer();
        compute_spin(compute_ns);
      }
    }
    // final timestamp after the last compute
    if (!user_grid_barrier(c, nusers)) return;
    if (uidx == 0 && threadIdx.x == 0) epoch_t[epochs] = gtimer();
  }
};

// ------------------------------------------------------------------ LoopWork (IOPS)
// Each requester keeps exactly one 4 KiB read outstanding; requester idx issues
// dev = (idx + j) % d, blk = (j * conc + idx) % num_blocks (bench/bandwidth.py:32-33).
struct LoopWork {
  uint4* bufs;            // [conc] 4 KiB
  WaitNode* nodes;        // [conc]
  unsigned long long* counters;   // [0] completions in window, [1] window start, [2] window end
  u32 conc, ndev;
  u32 write;              // 1: async_write of the requester's buffer (bytes idx & 0xFF) + wait
  u64 num_blocks;
  u64 warmup_ns, measure_ns;
  u64 max_per_task;
  __device__ void run(const DevCtx& c, u32 uidx, u32 nusers) const {
    const u32 idx = uidx * kCtaThreads + threadIdx.x;
    const bool act = idx < conc;
    const u32 who = user_who(uidx);
    const u32 sq_start = uidx * kCtaWarps + (threadIdx.x >> 5);
    if (threadIdx.x == 0) atomicCAS(&c.run->t_first, 0ull, gtimer());
    __syncthreads();
    const u64 t0 = ld_acquire(&c.run->t_first);
    const u64 ws = t0 + warmup_ns, we = ws + measure_ns;
    u32 inwin = 0;
    uint4* dst = bufs + (u64)(act ? idx : 0) * 256;
    WaitNode* node = nodes + (act ? idx : 0);
    if (write && act) {   // buf.data[:] = bytes([idx & 0xFF]) * block_size (bench/bandwidth.py:29-30)
      const u32 b = (idx & 0xFFu) * 0x01010101u;
      for (u32 k = 0; k < 256; ++k) dst[k] = make_uint4(b, b, b, b);
    }
    // requesters progress independently: a lane issues its next read as soon as its previous
    // one completed (no warp lockstep), so the in-flight population stays at `conc`
    const u32 lane = lane_id();
    bool outst = false;
    u64 j = 0;
    Spin sp;
    while (true) {
      const bool issue = act && !outst && j < max_per_task && gtimer() < we;
      const u32 ib = __ballot_sync(FULL, issue);
      if (ib) {
        const u32 dev = (idx + (u32)j) % ndev;
        const u64 blk = (j * conc + idx) % num_blocks;
        const u32 sq = sq_start + (u32)__shfl_sync(FULL, j, __ffs(ib) - 1);
        if (write) async_write_warp(c, issue, make_key(dev, blk), node, dst, who, sq);
        else async_read_warp(c, issue, make_key(dev, blk), node, dst, who, sq);
        if (issue) { ++j; outst = true; }
      }
      const u32 done = poll_nodes_warp(outst, node);
      if ((done >> lane) & 1u) {
        outst = false;
        const u64 t = gtimer();
        if (t >= ws && t < we) ++inwin;
      }
      const bool more = outst || (act && j < max_per_task && gtimer() < we);
      if (!__any_sync(FULL, more)) break;
      if (!ib && !done) {
        if (!sp.again(c, 512, __LINE__ + 100000 * SPIN_FILE_ID)) break;
      } else {
        sp = Spin();
      }
    }
    u32 s = inwin;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    if (lane_id() == 0 && s) atomicAdd(&counters[0], (u64)s);
    if (uidx == 0 && threadIdx.x == 0) { counters[1] = ws; counters[2] = we; }
  }
};

// ------------------------------------------------------------------ CoherenceWork
// The reference's coherence replay workload (tests/test_coherence.py:27-60): `tasks` tasks, one
// warp each (lane 0 carries the task, lockstep verbs), run their plans of (read | write, block,
// think time); writes carry a unique 8-byte prefix; every read observes the first 8 bytes of the
// buffer it got (its own, or the shared one the table returned) and logs ("test", "observe") at
// that instant — under the block's share-table home lock when the table is on, the instant a
// writer into that shared buffer also commits under.  With the table, every read keeps its
// reference to the end, then releases (the last release of a Modified buffer installs it into
// the cache).  Finally warp 0 flushes every MODIFIED line to the device (the reference's flusher).
struct CoherenceWork {
  const unsigned char* op;   // [tasks][ops] 0 read, 1 write, 2 read whose think time falls between its
                             // completion and its observe (test_coherence.py:112-135 hazard reader)
  const u32* blk;            // [tasks][ops]
  const u32* think;          // [tasks][ops] ns
  u32 tasks, ops;
  uint4* wbuf;               // [tasks][256] write payload page
  uint4* rbuf;               // [tasks][ops][256] read buffers (one AgileBuf per read)
  uint4* snap;               // [tasks][256] release snapshot pages
  WaitNode* nodes;           // [tasks][ops] op nodes, [tasks] install nodes, [32] flush nodes
  u64* seen;                 // [tasks][ops] observed prefixes
  u64* flushed;              // [1]
  __device__ void run(const DevCtx& c, u32 uidx, u32 nusers) const {
    if (uidx != 0) return;
    const u32 w = threadIdx.x >> 5, lane = lane_id();
    const bool act = lane == 0 && w < tasks;
    const u32 who = WHO_USER | w;   // task "u<w>" (system.py spawn_user naming)
    const u32 sq = w;
    WaitNode* inst = nodes + (u64)tasks * ops + (w < tasks ? w : 0);
    uint4* sp = snap + (u64)(w < tasks ? w : 0) * 256;
    if (w < tasks) {
      for (u32 i = 0; i < ops; ++i) {
        if (aborted(c)) break;
        const u64 t = (u64)w * ops + i;
        if (op[t] != 2) compute_spin(think[t]);   // op 2: read, think, then observe (the hazard reader)
        const u64 key = make_key(0, blk[t]);
        WaitNode* nd = nodes + t;
        if (op[t] == 1) {
          // payload: prefix (1 << 30 | task << 16 | op) + zeros (test_coherence.py:20-24)
          uint4* pb = wbuf + (u64)w * 256;
          for (u32 k = lane; k < 256; k += 32) pb[k] = make_uint4(0u, 0u, 0u, 0u);
          __syncwarp();
          if (lane == 0) *reinterpret_cast<u64*>(pb) = (1ull << 30) | ((u64)w << 16) | i;
          __syncwarp();
          async_write_t(c, act, key, nd, pb, who, sq, sp, inst);
          wait_nodes_warp(c, act, nd);
        } else {
          WaitNode* eff = nd;
          async_read_t(c, act, key, nd, rbuf + t * 256, who, sq, eff);
          wait_nodes_warp(c, act, eff);
          if (op[t] == 2) compute_spin(think[t]);
          if (act) {
            const bool tab = c.st_buckets != 0;
            const u32 h = tab ? st_home(c, key) : 0u;
            if (!tab || st_lock(c, h)) {
              const u64 v = __ldcg(reinterpret_cast<const unsigned long long*>(eff->dst));
              log_ev(c, who, M_TEST, A_OBSERVE, 0, blk[t], v);
              seen[t] = v;
              if (tab) st_unlock(c, h);
            }
          }
          __syncwarp();
        }
      }
      if (c.st_buckets) {
        for (u32 i = 0; i < ops; ++i) {
          const u64 t = (u64)w * ops + i;
          release_shared_warp(c, act && op[t] != 1, make_key(0, blk[t]), sp, inst, who, sq);
        }
      }
    }
    __syncthreads();
    if (w == 0) {
      const u64 n = flush_warp(c, nodes + (u64)tasks * ops + tasks, who, sq);
      if (lane == 0) flushed[0] = n;
    }
  }
};

// ------------------------------------------------------------------ LockCycleWork
// Planted lock-order bugs for the debug_locks detector (tests/test_lock_chain.py:26-47, 84-95):
// mode 0 — warps 0..n-1 each take set lock w, then (after all hold theirs) set lock (w+1) mod n:
// a ring of n; mode 1 — warp 0 takes set lock 0 twice (a one-cycle).  With debug_locks the
// cycle is reported and the run aborts with E_LOCK_CYCLE; without it the spins end in the watchdog.
struct LockCycleWork {
  u32 n, mode;
  __device__ void run(const DevCtx& c, u32 uidx, u32 nusers) const {
    if (uidx != 0) return;
    const u32 w = threadIdx.x >> 5;
    const u32 who = WHO_USER | w;
    const bool part = mode == 0 ? w < n : w == 0;
    bool held = false;
    if (part) held = lock_set(c, w % c.num_sets, who);
    __syncthreads();
    if (part && held) {
      const u32 next = mode == 0 ? (w + 1) % n : w;
      if (lock_set(c, next % c.num_sets, who)) unlock_set(c, next % c.num_sets);
      unlock_set(c, w % c.num_sets);
    }
  }
};

// ------------------------------------------------------------------ BusyWork
// AgileApi's BufferBusy (gpu_api.py:132-137, 203-204): one lane starts an async_read of a block
// into its buffer and, without waiting, starts another transfer on the same buffer (read, or
// write when `write` is set) — the second call must raise BufferBusy.
struct BusyWork {
  WaitNode* nodes;   // [1]
  uint4* buf;        // [256]
  u32 write;
  __device__ void run(const DevCtx& c, u32 uidx, u32 nusers) const {
    if (uidx != 0 || threadIdx.x >= 32) return;
    const bool act = lane_id() == 0;
    async_read_warp(c, act, make_key(0, 1), nodes, buf, WHO_USER, 0);
    if (write) async_write_warp(c, act, make_key(0, 2), nodes, buf, WHO_USER, 0);
    else async_read_warp(c, act, make_key(0, 2), nodes, buf, WHO_USER, 0);
    wait_nodes_warp(c, act, nodes);
  }
};

// ------------------------------------------------------------------ FlushWork
// SoftwareCache.flush (software_cache.py:283-298) as an API call: one warp writes every MODIFIED
// line back and waits for durability.
struct FlushWork {
  WaitNode* nodes;   // [32]
  u64* flushed;
  __device__ void run(const DevCtx& c, u32 uidx, u32 nusers) const {
    if (uidx != 0 || threadIdx.x >= 32) return;
    const u64 n = flush_warp(c, nodes, user_who(0), 0);
    if (lane_id() == 0) flushed[0] = n;
  }
};

// ------------------------------------------------------------------ WriteWork
// Every thread writes one block (async_write) and waits for its write-back barrier
// (gpu_api.py:192-227 + wait, gpu_api.py:233-248): the write path of SoftwareCache.write_block.
struct WriteWork {
  const u32* dev;
  const u64* blk;
  const uint4* src;       // [n][256] 4 KiB payloads
  WaitNode* nodes;        // [n]
  u64 n;
  __device__ void run(const DevCtx& c, u32 uidx, u32 nusers) const {
    const u64 i = (u64)uidx * kCtaThreads + threadIdx.x;
    const bool act = i < n;
    const u32 who = user_who(uidx);
    const u32 sq = uidx * kCtaWarps + (threadIdx.x >> 5);
    async_write_warp(c, act, act ? make_key(dev[i], blk[i]) : 0ull, nodes + (act ? i : 0), src + (act ? i : 0) * 256,
                     who, sq);
    wait_nodes_warp(c, act, nodes + (act ? i : 0));
  }
};

// ------------------------------------------------------------------ ArrayGetWork
// AgileApi.array_get (gpu_api.py:250-278): the device viewed as a little-endian array of
// elem_size-byte elements; element idx lives in block idx * elem_size / 4096 at byte offset
// idx * elem_size % 4096 (elem_size divides 4096, so an element never straddles blocks).  One
// GPU thread per element: read_range (software_cache.py:212-219) = access (hit, attach to the
// fill in flight, or claim + submit a miss), wait READY, copy the element's bytes, release.  The
// lane pins only its own line and only once its access succeeded (no hold-and-wait).
struct ArrayGetWork {
  const u32* dev;
  const u64* idx;
  u64 n;
  u32 elem_size;
  uint8_t* out;            // [n][elem_size]
  __device__ void run(const DevCtx& c, u32 uidx, u32 nusers) const {
    const u32 lane = lane_id();
    const u32 who = user_who(uidx);
    const u32 sq = uidx * kCtaWarps + (threadIdx.x >> 5);
    for (u64 i0 = (u64)uidx * kCtaThreads; i0 < n; i0 += (u64)nusers * kCtaThreads) {
      const u64 i = i0 + threadIdx.x;
      bool pend = i < n;
      u64 key = 0;
      u32 off = 0;
      if (pend) {
        const u64 byte_off = idx[i] * elem_size;
        key = make_key(dev[i], byte_off >> kBlockShift);
        off = (u32)(byte_off & (kBlockBytes - 1));
      }
      Spin sp;
      while (__any_sync(FULL, pend)) {
        const Req r = access_warp(c, pend, key, true, who, sq, false);
        const bool pinned = pend && (r.kind == R_HIT || r.kind == R_FILLING || r.kind == R_MISS);
        u32 wp = __ballot_sync(FULL, pinned);
        Spin s2;
        while (wp) {
          bool rd = false;
          if ((wp >> lane) & 1u) {
            const u64 w = ld_acquire(&c.tags[r.line]);
            rd = tw_state(w) == ST_READY || tw_state(w) == ST_MODIFIED;
          }
          wp &= ~__ballot_sync(FULL, rd);
          if (wp && !s2.again(c, 512, __LINE__ + 100000 * SPIN_FILE_ID)) break;
        }
        if (pinned) {
          const uint8_t* src = line_ptr(c, r.line) + off;
          uint8_t* dst = out + i * elem_size;
          if ((elem_size & 15u) == 0) {
            for (u32 k = 0; k < elem_size; k += 16)
              *reinterpret_cast<uint4*>(dst + k) = __ldcg(reinterpret_cast<const uint4*>(src + k));
          } else if ((elem_size & 7u) == 0) {
            for (u32 k = 0; k < elem_size; k += 8)
              *reinterpret_cast<u64*>(dst + k) = __ldcg(reinterpret_cast<const u64*>(src + k));
          } else if ((elem_size & 3u) == 0) {
            for (u32 k = 0; k < elem_size; k += 4)
              *reinterpret_cast<u32*>(dst + k) = __ldcg(reinterpret_cast<const u32*>(src + k));
          } else {
            for (u32 k = 0; k < elem_size; ++k) dst[k] = src[k];
          }
          unpin_line(c, r.line, 1);
        }
        pend = pend && r.kind == R_RETRY;
        if (aborted(c)) return;
        if (__any_sync(FULL, pend) && !sp.again(c, 1024, __LINE__ + 100000 * SPIN_FILE_ID)) return;
      }
    }
  }
};

// ------------------------------------------------------------------ GatherWork (queue/cache sweeps)
// One warp = 32 tasks in lockstep (run_workload(..., warp_size=32)). Per epoch each task
// prefetches its gather set (warp-coalesced) and then array_gets element 0 of every block.
struct GatherWork {
  const u64* keys;        // [tasks][epochs][gathers]
  u32* values;            // [tasks][epochs][gathers] little-endian u32 read
  u64* epoch_t;
  u32 tasks, epochs, gathers, async_mode;
  u64 compute_ns;
  // A CTA's tasks sit in its first ntw warps (one task per lane, warp_size=32 as in
  // run_workload(..., warp_size=32)); its other warps would idle.  Every warp of the CTA therefore
  // takes the same 32 tasks (warp w: tasks of warp w % ntw) and a 1/nh share of each task's gather
  // list (gathers g with g % nh == w / ntw, nh = 8 / ntw).  Each task still prefetches all its
  // blocks before it reads them and the epoch barrier still separates the epochs; only the
  // per-task command stream is issued by nh warps at once instead of one (a warp pass of 32
  // misses costs ~30 µs of dependent round trips on the GPU, the reference models 350 ns).
  __device__ __forceinline__ void share(u32 uidx, u32& task, bool& act, u32& g0, u32& gstep) const {
    const u32 wid = threadIdx.x >> 5;
    const u32 cta_tasks = min(tasks - min(tasks, uidx * kCtaThreads), (u32)kCtaThreads);
    const u32 ntw = max(1u, (cta_tasks + 31) / 32);
    const u32 nh = max(1u, (u32)kCtaWarps / ntw);
    task = uidx * kCtaThreads + (wid % ntw) * 32 + lane_id();
    act = task < tasks && wid < ntw * nh;
    g0 = wid / ntw;
    gstep = nh;
  }
  __device__ void prefetch_epoch(const DevCtx& c, bool act, u32 task, u32 e, u32 who, u32 sq_start, u32 g0,
                                 u32 gstep) const {
    for (u32 g = g0; g < gathers; g += gstep) {
      const u64 key = act ? keys[((u64)task * epochs + e) * gathers + g] : 0ull;
      prefetch_warp(c, act, key, who, sq_start + g + e * gathers, false);
    }
  }
  __device__ void get_epoch(const DevCtx& c, bool act, u32 task, u32 e, u32 who, u32 sq_start, u32 g0,
                            u32 gstep) const {
    for (u32 g = g0; g < gathers; g += gstep) {
      const u64 key = act ? keys[((u64)task * epochs + e) * gathers + g] : 0ull;
      // array_get = read_range loop (software_cache.py:212-219): access, wait READY, read.  The
      // lane pins only its own line, and only after its claim succeeded (no hold-and-wait).
      bool pend = act;
      u32 val = 0;
      Spin sp;
      while (__any_sync(FULL, pend)) {
        const Req r = access_warp(c, pend, key, true, who, sq_start, false);
        const bool pinned = pend && (r.kind == R_HIT || r.kind == R_FILLING || r.kind == R_MISS);
        u32 wp = __ballot_sync(FULL, pinned);
        Spin s2;
        while (wp) {
          bool rd = false;
          if ((wp >> lane_id()) & 1u) {
            const u64 w = ld_acquire(&c.tags[r.line]);
            rd = tw_state(w) == ST_READY || tw_state(w) == ST_MODIFIED;
          }
          wp &= ~__ballot_sync(FULL, rd);
          if (wp && !s2.again(c, 512, __LINE__ + 100000 * SPIN_FILE_ID)) break;
        }
        if (pinned) {
          val = __ldcg(reinterpret_cast<const unsigned int*>(line_ptr(c, r.line)));
          unpin_line(c, r.line, 1);
        }
        pend = pend && (r.kind == R_RETRY);
        if (aborted(c)) break;
        if (__any_sync(FULL, pend) && !sp.again(c, 1024, __LINE__ + 100000 * SPIN_FILE_ID)) break;
      }
      if (act) values[((u64)task * epochs + e) * gathers + g] = val;
    }
  }
  __device__ void run(const DevCtx& c, u32 uidx, u32 nusers) const {
    u32 task, g0, gstep;
    bool act;
    share(uidx, task, act, g0, gstep);
    const u32 who = user_who(uidx);
    const u32 sq_start = task / 32 + g0;   // thread_idx % nsq start SQ per warp (nvme_queue.py:91-93)
    if (uidx == 0 && threadIdx.x == 0) epoch_t[0] = gtimer();
    if (async_mode) prefetch_epoch(c, act, task, 0, who, sq_start, g0, gstep);
    for (u32 e = 0; e < epochs; ++e) {
      if (!async_mode) prefetch_epoch(c, act, task, e, who, sq_start, g0, gstep);
      else if (e + 1 < epochs) prefetch_epoch(c, act, task, e + 1, who, sq_start, g0, gstep);
      get_epoch(c, act, task, e, who, sq_start, g0, gstep);
      if (!user_grid_barrier(c, nusers)) return;
      compute_spin(compute_ns);
    }
    if (!user_grid_barrier(c, nusers)) return;
    if (uidx == 0 && threadIdx.x == 0) epoch_t[1] = gtimer();
  }
};

// ------------------------------------------------------------------ EmbBagWork (K5)
// pooled[b, t, :] = sum_l table_t[idx(b, t, l), :] over 4 KiB pages of 4096 / (4 D) rows of D fp32.
//
// Tables are described per launch by TabDesc (= agile_table_shard of the C-ABI): the page key of
// the shard's first page, the global row range [row0, row0 + rows) the shard holds (row-wise
// sharding over ranks; a whole table has row0 = 0, rows = table_rows), the whole table's row
// count (indices outside [0, table_rows) raise OutOfRange, gpu_api.py:122-126 / ssd_model.py:24),
// the byte offset of the table's pooled vector in an output row, and whether the shard writes its
// fp64 partial sum (row shards, summed by the receiver after the exchange) or the final fp32.
//
// Accumulation is fp64, rounded once to fp32: whenever the fp64 sum is exact (always for the
// synthetic tables, whose values lie on a 2^-23 grid in [-1, 1), for any pooling factor below
// 2^29) the result is the correctly rounded exact sum, independent of summation order — so a
// table split by rows over ranks, or a bag split into 32-lookup chunks, gives bit-identical
// pooled vectors.
//
// One warp per bag; a bag's lookups are taken 32 per chunk (lane = lookup; fixed L or
// variable-length bags through offsets).  A chunk's pages are resolved with the batched
// signature probe (READY confirmed by an acquire load), misses claimed/submitted warp-aggregated
// and waited without holding anything; then every lane loads one 16 B slice of each row (512 B
// coalesced per row at D = 128) and accumulates.  Hits are validated seqlock-style once per
// chunk: the tag re-read carries a data dependency on every row value the warp loaded, so it is
// issued only after those loads returned; a changed identity redoes the chunk.
struct TabDesc {
  u64 key0;
  long long row0, rows, total;
  u32 out_off;
  u32 flags;
};
static_assert(sizeof(TabDesc) == 40, "TabDesc must match agile_table_shard");
constexpr u32 TAB_PARTIAL_F64 = 1u;

// Row loads of the hit path: L2-coherent (.cg); with AGILE_ROW_EVICT_FIRST the rows carry an
// L2 evict-first policy so a stream of cold rows does not push the signature / tag arrays out of L2
#ifndef AGILE_ROW_EVICT_FIRST
#define AGILE_ROW_EVICT_FIRST 0
#endif
__device__ __forceinline__ u64 row_policy() {
#if AGILE_ROW_EVICT_FIRST
  u64 p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
#else
  return 0;
#endif
}
__device__ __forceinline__ float4 ld_row(const float4* a, u64 pol) {
#if AGILE_ROW_EVICT_FIRST
  float4 v;
  asm volatile("ld.global.cg.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a), "l"(pol));
  return v;
#else
  (void)pol;
  return __ldcg(a);
#endif
}

// 0, computed from v: an address offset that cannot be formed before v's load returned
__device__ __forceinline__ u64 dep_zero(u32 v) {
  u32 z;
  asm volatile("and.b32 %0, %1, 0;" : "=r"(z) : "r"(v));
  return (u64)z;
}

struct EmbBagWork {
  const long long* idx;        // bag (b, t): idx[(b*T + t)*L + l], or idx[offsets[b*T + t] + l]
  const long long* offsets;    // [B*T + 1] (variable-length bags) or null
  const TabDesc* tabs;         // [T] or null: then table_key0 / table_rows, whole tables
  const u64* table_key0;       // [T] key of the table's first page (dev << 36 | page)
  const long long* table_rows; // [T]
  uint8_t* out;                // table t of sample b at out + b*out_row_bytes + out_off(t)
  u64 out_row_bytes;
  u32 out_t_bytes;             // legacy layout: out_off(t) = t * out_t_bytes
  u64* lookups_miss;           // [2] lookups, miss-path lookups
  u32 B, T, L, D;
  u32 pd;                      // > 0: prefetch the next grabbed block of bags (async mode)
  u32 rows_per_page_shift;     // log2(4096 / (D*4))
  u32 nwarps_total;
  u32 prefetch_only;           // 1: pull every page of the batch toward the cache, no pooling
  u64 t_magic;                 // floor(2^64 / T) + 1: bag / T = umul64hi(bag, t_magic) for T > 1

  // bag -> (sample b, table t) without an integer division (exact for bag < 2^32)
  __device__ __forceinline__ u32 bag_sample(u32 bag) const {
    return T == 1 ? bag : (u32)__umul64hi((u64)bag, t_magic);
  }

  __device__ __forceinline__ TabDesc tab(u32 t) const {
    TabDesc d;
    if (tabs) {
      const TabDesc* p = tabs + t;
      d.key0 = __ldg(reinterpret_cast<const unsigned long long*>(&p->key0));
      d.row0 = __ldg(&p->row0);
      d.rows = __ldg(&p->rows);
      d.total = __ldg(&p->total);
      d.out_off = __ldg(&p->out_off);
      d.flags = __ldg(&p->flags);
    } else {
      d.key0 = __ldg(reinterpret_cast<const unsigned long long*>(table_key0) + t);
      d.row0 = 0;
      d.rows = d.total = __ldg(table_rows + t);
      d.out_off = t * out_t_bytes;
      d.flags = 0;
    }
    return d;
  }
  __device__ __forceinline__ void bag_span(u32 bag, u64& start, u32& n) const {
    if (offsets) {
      const long long s0 = __ldg(offsets + bag), s1 = __ldg(offsets + bag + 1);
      start = (u64)s0;
      n = s1 > s0 ? (u32)(s1 - s0) : 0u;
    } else {
      start = (u64)bag * L;
      n = L;
    }
  }
  // the lane's lookup -> (page key, byte offset in the page); false when the lane has no lookup
  // in this shard.  Out-of-range indices raise OutOfRange (the run aborts, the host sees -103).
  __device__ __forceinline__ bool lookup_key(const DevCtx& c, const TabDesc& td, bool lact, long long r, u32 t,
                                             u64& key, u32& off) const {
    if (!lact) return false;
    if (r < 0 || r >= td.total) {
      set_error(c, E_OUT_OF_RANGE, t, (u64)r);
      return false;
    }
    if (r < td.row0 || r >= td.row0 + td.rows) return false;   // another rank's rows
    const u64 lr = (u64)(r - td.row0);
    key = td.key0 + (lr >> rows_per_page_shift);
    off = ((u32)lr & ((1u << rows_per_page_shift) - 1u)) * D * 4;
    return true;
  }

  // bags are grabbed kGrab at a time from the launch-wide counter (dynamic balance: a warp held
  // up by a slow miss does not hold back a static share of the batch)
  static constexpr u32 kGrab = 4;
  __device__ __forceinline__ u32 grab_block(const DevCtx& c) const {
    u32 b = 0;
    if (lane_id() == 0) b = (u32)atomicAdd(&c.run->work_next, (u64)kGrab);
    return __shfl_sync(FULL, b, 0);
  }
  // sync mode: kGrab bags per grab while plenty remain, single bags once the previous grab landed
  // in the last 2 bags per warp of the batch (a warp holding a block while the others ran dry was
  // the kernel's tail); the grab size comes from the previous grab's index, no extra round trip
  __device__ __forceinline__ u32 grab_adaptive(const DevCtx& c, u32 g) const {
    u32 b = 0;
    if (lane_id() == 0) b = (u32)atomicAdd(&c.run->work_next, (u64)g);
    return __shfl_sync(FULL, b, 0);
  }
  // async mode: submit the missing pages of a block's bags (first chunk of each), no waiting
  __device__ __noinline__ void prefetch_block(const DevCtx& c, u32 first, u32 nbags, u32 who, u32 sq) const {
    for (u32 k = 0; k < kGrab && first + k < nbags; ++k) {
      const u32 bag = first + k;
      const u32 t = bag - bag_sample(bag) * T;
      const TabDesc td = tab(t);
      u64 start; u32 n;
      bag_span(bag, start, n);
      const bool lact = lane_id() < n;
      const long long r = lact ? __ldg(idx + start + lane_id()) : 0ll;
      u64 key = 0; u32 off = 0;
      const bool a = lookup_key(c, td, lact, r, t, key, off);
      prefetch_warp(c, a, key, who, sq + k, true);
    }
  }

  // user-grid register budget: 4 CTAs x 8 warps per SM (64 registers per thread).  (A variant
  // that staged rows in shared memory through cp.async and pipelined three bags per warp measured
  // 20-30 % slower than this register path: its 80 KiB of stage per CTA halved the warps per SM.)
#ifndef AGILE_EMB_MIN_CTAS
#define AGILE_EMB_MIN_CTAS 4
#endif

  static constexpr int kMinCtas = AGILE_EMB_MIN_CTAS;


  __device__ void run(const DevCtx& c, u32 uidx, u32 nusers) const {
    const u32 gw = uidx * kCtaWarps + (threadIdx.x >> 5);
    const u32 who = user_who(uidx);
    if (prefetch_only) { run_prefetch(c, gw, who); return; }
    const u32 nbags = B * T;
    u32 misses = 0, lookups = 0;
    if (!pd) {
      // synchronous mode: grab just in time (no block held ahead), adaptive grab size
      u32 n = kGrab;
      while (!aborted(c)) {
        const u32 first = grab_adaptive(c, n);
        if (first >= nbags) break;
        const u32 next_n = first + n + (u64)nwarps_total * 2 < nbags ? kGrab : 1u;
        bool ok = true;
        for (u32 k = 0; k < n && first + k < nbags && ok; ++k) ok = pool_bag(c, first + k, who, gw, misses, lookups);
        if (!ok) break;
        n = next_n;
      }
      if (lane_id() == 0) {
        atomicAdd(&lookups_miss[0], (u64)lookups);
        atomicAdd(&lookups_miss[1], (u64)misses);
      }
      return;
    }
    u32 cur = grab_block(c);
    if (pd && cur < nbags) prefetch_block(c, cur, nbags, who, gw);
    u32 pass = 0;
    while (cur < nbags) {
      const u32 nxt = grab_block(c);
      if (pd && nxt < nbags) prefetch_block(c, nxt, nbags, who, gw + (++pass));
      if (!offsets && nxt < nbags) {
        // the next block's indices (kGrab * L contiguous int64) toward L2 while this block pools:
        // its first index load is then an L2 hit instead of an HBM round trip
        const u64 i0 = (u64)nxt * L, n8 = (u64)min(kGrab, nbags - nxt) * L;
        for (u64 o = (u64)lane_id() * 16; o < n8; o += 32 * 16)
          asm volatile("prefetch.global.L2::evict_last [%0];" :: "l"(idx + i0 + o));
      }
      for (u32 k = 0; k < kGrab && cur + k < nbags; ++k)
        if (!pool_bag(c, cur + k, who, gw, misses, lookups)) { cur = nbags; break; }
      if (aborted(c)) break;
      cur = nxt;
    }
    if (lane_id() == 0) {
      atomicAdd(&lookups_miss[0], (u64)lookups);
      atomicAdd(&lookups_miss[1], (u64)misses);
    }
  }

  // batch-level async (AGILE prefetch, gpu_api.py:139-162): submit every missing page of the
  // batch and return; the service keeps the launch alive until all fills completed.  Fixed-L
  // batches are taken as one flat stream of lookups, 32 per warp pass (lane = lookup, coalesced
  // index loads), so every lane probes; variable-length bags go bag by bag.
  __device__ __noinline__ void run_prefetch(const DevCtx& c, u32 gw, u32 who) const {
    const u32 lane = lane_id();
    const u32 nbags = B * T;
    u32 lookups = 0, pass = 0;
    if (offsets) {
      while (true) {
        const u32 first = grab_block(c);
        if (first >= nbags) break;
        for (u32 k = 0; k < kGrab && first + k < nbags; ++k) {
          const u32 bag = first + k, t = bag - bag_sample(bag) * T;
          const TabDesc td = tab(t);
          u64 start; u32 n;
          bag_span(bag, start, n);
          for (u32 c0 = 0; c0 < n; c0 += 32) {
            const bool lact = c0 + lane < n;
            u64 key = 0; u32 off = 0;
            const bool a = lookup_key(c, td, lact, lact ? __ldg(idx + start + c0 + lane) : 0ll, t, key, off);
            prefetch_warp(c, a, key, who, gw + (++pass), false);
          }
          lookups += n;
        }
        if (aborted(c)) break;
      }
    } else {
      const u64 nlk = (u64)nbags * L;
      u64 base = 0;
      u32 left = 0;
      while (true) {
        if (!left) {
          u64 b = 0;
          if (lane == 0) b = atomicAdd(&c.run->work_next, (u64)kGrab * 32);
          base = __shfl_sync(FULL, b, 0);
          left = kGrab;
        }
        const u64 g = base + lane;
        base += 32;
        --left;
        if (g - lane >= nlk) break;
        const bool act = g < nlk;
        u64 key = 0; u32 off = 0;
        bool a = false;
        if (act) {
          const u32 t = (u32)(g / L) % T;
          a = lookup_key(c, tab(t), true, __ldg(idx + g), t, key, off);
        }
        prefetch_warp(c, a, key, who, gw + (++pass), false);
        lookups += __popc(__ballot_sync(FULL, act));
        if ((pass & 15u) == 0 && aborted(c)) break;
      }
    }
    if (lane == 0) atomicAdd(&lookups_miss[0], (u64)lookups);
  }

  // Miss path of a chunk: lanes in `need` claim or attach to the fill of their page and wait for
  // READY; nothing is held meanwhile (a line reassigned under us goes again).  Out of line: the
  // hot (all-hit) path keeps its registers, the call saves them only when a miss happens.
  struct Resolved { u64 word; u32 line; u32 ok; };
  __device__ __noinline__ Resolved resolve_misses(const DevCtx& c, u32 need, u64 key, u32 who, u32 gw, u32 line,
                                                  u64 word) const {
    const u32 lane = lane_id();
    Resolved res;
    res.ok = 0;
    Spin sp;
    while (need) {
      const bool nm = (need >> lane) & 1u;
      const Req r = access_warp(c, nm, key, false, who, gw, false);
      const bool got = nm && (r.kind == R_HIT || r.kind == R_FILLING || r.kind == R_MISS);
      if (got) line = r.line;
      u32 wp = __ballot_sync(FULL, got);
      u32 done = 0;
      Spin s2;
      while (wp) {
        bool rd = false, gone = false;
        if ((wp >> lane) & 1u) {
          const u64 w = ld_acquire(&c.tags[line]);
          if (!tw_live(w) || tw_key(w) != key) gone = true;
          else if (tw_state(w) == ST_READY || tw_state(w) == ST_MODIFIED) { word = w; rd = true; }
        }
        done |= __ballot_sync(FULL, rd);
        wp &= ~__ballot_sync(FULL, rd || gone);
        if (wp && !s2.again(c, 1024, __LINE__ + 100000 * SPIN_FILE_ID)) break;
      }
      need &= ~done;
      if (aborted(c)) return res;
      if (need && !done && !sp.again(c, 1024, __LINE__ + 100000 * SPIN_FILE_ID)) return res;
    }
    res.line = line;
    res.word = word;
    res.ok = aborted(c) ? 0u : 1u;
    return res;
  }

  // One chunk (<= 32 lookups from position c0) of a bag, summed into a0..a3 in lookup order:
  // probe, miss path, rows, seqlock validation.  Returns 0 ok, 1 validation failed (a page changed
  // identity while the warp read it: the caller restarts the bag), -1 the run aborts.
  __device__ __forceinline__ int pool_chunk(const DevCtx& c, const TabDesc& td, u32 t, u64 start, u32 c0, u32 n,
                                            u32 who, u32 gw, bool first_visit, u32& misses, u32& lookups,
                                            double& a0, double& a1, double& a2, double& a3) const {
    const u32 lane = lane_id();
    const bool lact = c0 + lane < n;
    const long long r = lact ? __ldg(idx + start + c0 + lane) : 0ll;
    u64 key = 0; u32 off = 0;
    const bool a = lookup_key(c, td, lact, r, t, key, off);
    const u32 am = __ballot_sync(FULL, a);
    if (first_visit) lookups += __popc(am);
    u32 line = NONE; u64 word = 0;
    probe_lanes<true>(c, a, key, line, word);
    const bool ready = a && line != NONE && (tw_state(word) == ST_READY || tw_state(word) == ST_MODIFIED);
    if (ready && !tw_ref(word)) atomicOr(&c.tags[line], REF_BIT);   // on_hit
    const u32 need = __ballot_sync(FULL, a && !ready);
    if (need) {
      if (first_visit) misses += __popc(need);
      const Resolved rv = resolve_misses(c, need, key, who, gw, line, word);
      if (!rv.ok) return -1;
      line = rv.line;
      word = rv.word;
    }
      // sum the chunk's rows in lookup order, lane owns dims [4*lane, 4*lane+4) (a lane past D/4
      // reads a copy of its row's first dims and never stores): the active lookups are compacted
      // to lanes 0..n-1 once (a prefix already is), then rows are loaded 8, then 4, then 1 at a
      // time, 16 B/lane (512 B coalesced at D = 128) — no zero-padded loads, no per-row lane
      // search; only the row's 32-bit slot index in the cache's row space is shuffled
      const u32 rsh = kBlockShift - rows_per_page_shift;   // log2(row bytes)
      u32 rs = a ? ((line << rows_per_page_shift) | (off >> rsh)) : 0u;
      const u32 na = __popc(am);
      if (am & (am + 1u)) rs = __shfl_sync(FULL, rs, lane < na ? __fns(am, 0, lane + 1) : 0u);
      const u32 rb = 1u << rsh;
      const uint8_t* rowbase = c.lines + ((lane * 16u) & (rb - 1u));
      u32 dep = 0;
      const u64 pol = row_policy();
      u32 r0 = 0;
      for (; r0 + 8 <= na; r0 += 8) {
        float4 v[8];
#pragma unroll
        for (u32 j = 0; j < 8; ++j)
          v[j] = ld_row(reinterpret_cast<const float4*>(rowbase + (u64)__shfl_sync(FULL, rs, r0 + j) * rb), pol);
#pragma unroll
        for (u32 j = 0; j < 8; ++j) {
          a0 += (double)v[j].x; a1 += (double)v[j].y; a2 += (double)v[j].z; a3 += (double)v[j].w;
          dep |= __float_as_uint(v[j].x);   // the 16 B load returns at once
        }
      }
      if (r0 + 4 <= na) {
        float4 v[4];
#pragma unroll
        for (u32 j = 0; j < 4; ++j)
          v[j] = ld_row(reinterpret_cast<const float4*>(rowbase + (u64)__shfl_sync(FULL, rs, r0 + j) * rb), pol);
#pragma unroll
        for (u32 j = 0; j < 4; ++j) {
          a0 += (double)v[j].x; a1 += (double)v[j].y; a2 += (double)v[j].z; a3 += (double)v[j].w;
          dep |= __float_as_uint(v[j].x);   // the 16 B load returns at once
        }
        r0 += 4;
      }
      for (; r0 < na; ++r0) {
        const float4 v = ld_row(reinterpret_cast<const float4*>(rowbase + (u64)__shfl_sync(FULL, rs, r0) * rb), pol);
        a0 += (double)v.x; a1 += (double)v.y; a2 += (double)v.z; a3 += (double)v.w;
        dep |= __float_as_uint(v.x);
      }
      // seqlock validation, once per chunk: the tag re-read's address depends on every row value
      // of the warp (redux over the lanes), so it is issued after all of them were loaded
      const u64 z = dep_zero(__reduce_or_sync(FULL, dep));
      bool bad = false;
      if (a) bad = ((ld_relaxed(&c.tags[line] + z) ^ word) & IDENT_MASK) != 0;
      return __any_sync(FULL, bad) ? 1 : 0;
  }

  __device__ __forceinline__ void store_bag(u32 b, const TabDesc& td, double a0, double a1, double a2,
                                            double a3) const {
    const u32 lane = lane_id();
    if (lane * 4 >= D) return;
    uint8_t* o = out + (u64)b * out_row_bytes + td.out_off;
    if (td.flags & TAB_PARTIAL_F64) {
      reinterpret_cast<double2*>(o)[2 * lane] = make_double2(a0, a1);
      reinterpret_cast<double2*>(o)[2 * lane + 1] = make_double2(a2, a3);
    } else {
      reinterpret_cast<float4*>(o)[lane] = make_float4((float)a0, (float)a1, (float)a2, (float)a3);
    }
  }

  // pool one bag (fp64, 4 dims per lane) and store it; false when the run aborts.  Bags of up to
  // 32 lookups take one chunk pass with no restart state held (the hot path); a failed validation
  // or a longer bag goes to pool_bag_slow.
  __device__ __forceinline__ bool pool_bag(const DevCtx& c, u32 bag, u32 who, u32 gw, u32& misses,
                                           u32& lookups) const {
    const u32 b = bag_sample(bag), t = bag - b * T;
    const TabDesc td = tab(t);
    u64 start; u32 n;
    bag_span(bag, start, n);
    if (n > 32) return pool_bag_slow(c, bag, who, gw, misses, lookups, 0u);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const int rc = pool_chunk(c, td, t, start, 0u, n, who, gw, true, misses, lookups, a0, a1, a2, a3);
    if (rc < 0) return false;
    if (rc > 0) return pool_bag_slow(c, bag, who, gw, misses, lookups, 32u);
    store_bag(b, td, a0, a1, a2, a3);
    return true;
  }

  // The general bag: chunks of 32 lookups; a chunk whose validation fails restarts the bag (rare: a
  // page was evicted while the warp read it); after 4 failures the bag is pooled row by row, each
  // row validated on its own.  `counted`: lookups below this position were already counted.
  __device__ __noinline__ bool pool_bag_slow(const DevCtx& c, u32 bag, u32 who, u32 gw, u32& misses,
                                             u32& lookups, u32 counted) const {
    const u32 b = bag_sample(bag), t = bag - b * T;
    const TabDesc td = tab(t);
    u64 start; u32 n;
    bag_span(bag, start, n);
    double a0, a1, a2, a3;
    u32 fails = counted ? 1u : 0u;
    Spin rsp;
  restart:
    a0 = a1 = a2 = a3 = 0.0;
    for (u32 c0 = 0; c0 < n; c0 += 32) {
      const bool first_visit = c0 >= counted;
      if (fails >= 4) {
        const bool lact = c0 + lane_id() < n;
        const long long r = lact ? __ldg(idx + start + c0 + lane_id()) : 0ll;
        u64 key = 0; u32 off = 0;
        const bool a = lookup_key(c, td, lact, r, t, key, off);
        const u32 am = __ballot_sync(FULL, a);
        if (first_visit) lookups += __popc(am);
        const Acc4 r4 = pool_rows_one_by_one(c, am, key, off, who, gw, make_acc4(a0, a1, a2, a3));
        if (!r4.ok) return false;
        a0 = r4.v[0]; a1 = r4.v[1]; a2 = r4.v[2]; a3 = r4.v[3];
      } else {
        const int rc = pool_chunk(c, td, t, start, c0, n, who, gw, first_visit, misses, lookups, a0, a1, a2, a3);
        if (rc < 0) return false;
        if (rc > 0) {
          if (first_visit) counted = c0 + 32;
          ++fails;
          if (!rsp.again(c, 256, __LINE__ + 100000 * SPIN_FILE_ID)) return false;
          goto restart;
        }
      }
      if (first_visit) counted = c0 + 32;
    }
    store_bag(b, td, a0, a1, a2, a3);
    return true;
  }

  struct Acc4 { double v[4]; u32 ok; };
  static __device__ __forceinline__ Acc4 make_acc4(double x, double y, double z, double w) {
    Acc4 r; r.v[0] = x; r.v[1] = y; r.v[2] = z; r.v[3] = w; r.ok = 1; return r;
  }
  __device__ __noinline__ Acc4 pool_rows_one_by_one(const DevCtx& c, u32 am, u64 key, u32 off, u32 who, u32 gw,
                                                    Acc4 acc) const {
    const u32 lane = lane_id();
    double a0 = acc.v[0], a1 = acc.v[1], a2 = acc.v[2], a3 = acc.v[3];
    acc.ok = 0;
    for (u32 m = am; m; m &= m - 1) {
      const u32 l = __ffs(m) - 1;
      const u64 kl = __shfl_sync(FULL, key, l);
      const u32 ol = __shfl_sync(FULL, off, l);
      Spin s3;
      while (true) {
        if (aborted(c)) return acc;
        const Req r = access_warp(c, lane == l, kl, false, who, gw, false);
        const int kind = __shfl_sync(FULL, r.kind, l);
        if (kind == R_HIT || kind == R_FILLING || kind == R_MISS) {
          const u32 ln = __shfl_sync(FULL, r.line, l);
          u64 w = 0;
          Spin s4;
          while (true) {
            w = ld_acquire(&c.tags[ln]);
            if (!tw_live(w) || tw_key(w) != kl) break;
            if (tw_state(w) == ST_READY || tw_state(w) == ST_MODIFIED) break;
            if (!s4.again(c, 1024, __LINE__ + 100000 * SPIN_FILE_ID)) return acc;
          }
          if (tw_live(w) && tw_key(w) == kl && tw_state(w) >= ST_READY) {
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (lane * 4 < D) v = __ldcg(reinterpret_cast<const float4*>(line_ptr(c, ln) + ol) + lane);
            const u64 z = dep_zero(__reduce_or_sync(FULL, __float_as_uint(v.x) | __float_as_uint(v.w)));
            if (((ld_relaxed(&c.tags[ln] + z) ^ w) & IDENT_MASK) == 0) {
              a0 += (double)v.x; a1 += (double)v.y; a2 += (double)v.z; a3 += (double)v.w;
              break;
            }
          }
        }
        if (!s3.again(c, 1024, __LINE__ + 100000 * SPIN_FILE_ID)) return acc;
      }
    }
    return make_acc4(a0, a1, a2, a3);
  }
};

// ------------------------------------------------------------------ paged arrays (K6/K7)
// Graph arrays (CSR col_idx, SpMV values) live in the page store, 1024 x 4 B entries per 4 KiB
// page; key = array key0 + entry / 1024.  Warps walk them in increasing position order, so a
// warp keeps the two pages it resolved last in registers (PageRegs) and only probes the cache
// when it crosses into a new page.  Nothing is pinned: reads are validated seqlock-style against
// the tag word (identity = state | version | key) after the fact, and a pass whose page changed
// identity under it is redone (a READY line is only reassigned through a fresh claim, which bumps
// the version).  No lock or pin is held across any wait (gpu_api.py:233-248).
struct PageRegs {
  u64 key[2];
  u32 line[2];
  u64 word[2];
  __device__ __forceinline__ void clear() { key[0] = key[1] = ~0ull; }
};

// Resolve every active lane's page to a READY line.  Lanes sharing a key coalesce
// (__match_any_sync, lowest lane leads: warp_coalesce, gpu_api.py:40-54); register hits skip the
// probe; the other leaders probe, and run the miss path (claim or attach to the in-flight fill,
// submit, wait for READY) when the page is not resident.  Returns false when the run aborts.
__device__ bool resolve_pages_warp(const DevCtx& c, bool act, u64 key, PageRegs& pr, u32& line, u64& word,
                                   u32 who, u32 sq, u32& misses) {
  const u32 lane = lane_id();
  bool need = act;
  if (act) {
    if (key == pr.key[0]) { line = pr.line[0]; word = pr.word[0]; need = false; }
    else if (key == pr.key[1]) { line = pr.line[1]; word = pr.word[1]; need = false; }
  }
  if (!__any_sync(FULL, need)) return true;
  u32 grp = __match_any_sync(FULL, need ? key : ~0ull);
  if (!need) grp = 0;
  const bool leader = need && (grp & lanemask_lt()) == 0;
  u32 l = NONE;
  u64 w = 0;
  probe_lanes(c, leader, key, l, w);
  const bool ready = leader && l != NONE && tw_state(w) >= ST_READY;
  if (ready && !tw_ref(w)) atomicOr(&c.tags[l], REF_BIT);   // on_hit (software_cache.py:124-126)
  u32 pend = __ballot_sync(FULL, leader && !ready);
  misses += __popc(pend);
  Spin sp;
  while (pend) {
    const bool nm = (pend >> lane) & 1u;
    const Req r = access_warp(c, nm, key, false, who, sq, false);
    const bool got = nm && (r.kind == R_HIT || r.kind == R_FILLING || r.kind == R_MISS);
    if (got) { l = r.line; w = r.word; }
    u32 wp = __ballot_sync(FULL, got);
    u32 done = 0;
    Spin s2;
    while (wp) {
      bool rd = false, gone = false;
      if ((wp >> lane) & 1u) {
        const u64 t = ld_relaxed(&c.tags[l]);
        if (!tw_live(t) || tw_key(t) != key) gone = true;
        else if (tw_state(t) >= ST_READY) { w = t; rd = true; }
      }
      done |= __ballot_sync(FULL, rd);
      wp &= ~__ballot_sync(FULL, rd || gone);
      if (wp && !s2.again(c, 1024, __LINE__ + 100000 * SPIN_FILE_ID)) return false;
    }
    pend &= ~done;
    if (aborted(c)) return false;
    if (pend && !done && !sp.again(c, 1024, __LINE__ + 100000 * SPIN_FILE_ID)) return false;
  }
  fence_acq_rel();   // READY observed above (relaxed) -> the line's bytes are visible
  const u32 ll = need ? (u32)(__ffs(grp) - 1) : lane;
  const u32 bl = __shfl_sync(FULL, l, ll);
  const u64 bw = __shfl_sync(FULL, w, ll);
  if (need) { line = bl; word = bw; }
  // keep the pages of the two highest leaders (positions grow with the lane)
  const u32 lb = __ballot_sync(FULL, leader);
  const int h1 = 31 - __clz(lb);
  const u32 rest = lb & ~(1u << h1);
  const int h0 = rest ? 31 - __clz(rest) : -1;
  const u64 k1 = __shfl_sync(FULL, key, h1);
  const u32 l1 = __shfl_sync(FULL, line, h1);
  const u64 w1 = __shfl_sync(FULL, word, h1);
  const u64 k0 = __shfl_sync(FULL, key, h0 < 0 ? h1 : h0);
  const u32 l0 = __shfl_sync(FULL, line, h0 < 0 ? h1 : h0);
  const u64 w0 = __shfl_sync(FULL, word, h0 < 0 ? h1 : h0);
  if (h0 < 0) {   // one new page: it replaces the older register entry
    if (pr.key[1] != k1) { pr.key[0] = pr.key[1]; pr.line[0] = pr.line[1]; pr.word[0] = pr.word[1]; }
  } else {
    pr.key[0] = k0; pr.line[0] = l0; pr.word[0] = w0;
  }
  pr.key[1] = k1; pr.line[1] = l1; pr.word[1] = w1;
  return true;
}

// After reading: every distinct page the warp read must still hold the identity it was read
// under (one tag load per distinct page).  False -> redo the reads.
__device__ __forceinline__ bool validate_pages_warp(const DevCtx& c, bool act, u64 key, u32 line, u64 word) {
  fence_acq_rel();
  u32 grp = __match_any_sync(FULL, act ? key : ~0ull);
  const bool leader = act && (grp & lanemask_lt()) == 0;
  bool bad = false;
  if (leader) bad = ((ld_relaxed(&c.tags[line]) ^ word) & IDENT_MASK) != 0;
  return !__any_sync(FULL, bad);
}

// Largest i in [lo, hi] with a[i] <= x, for non-decreasing a and a[lo] <= x: 32 pivots per
// round trip, so ~log32(hi - lo) dependent loads.
__device__ __forceinline__ u64 warp_search_le(const long long* a, u64 lo, u64 hi, long long x) {
  const u32 lane = lane_id();
  while (hi - lo >= 32) {
    const u64 span = hi - lo;
    const u64 p = lo + (span * lane) / 32;
    const u32 b = __ballot_sync(FULL, __ldcg(a + p) <= x);
    const u32 k = 31 - __clz(b | 1u);
    const u64 nlo = lo + (span * k) / 32;
    const u64 nhi = k == 31 ? hi : lo + (span * (k + 1)) / 32 - 1;
    lo = nlo;
    hi = nhi;
  }
  const u64 p = lo + lane;
  const u32 b = __ballot_sync(FULL, p <= hi && __ldcg(a + p) <= x);
  return lo + (31 - __clz(b | 1u));
}

// Largest window slot j in [0, 30] with ev_j <= x (ev non-decreasing across lanes 0..31).
__device__ __forceinline__ u32 window_slot(long long ev, long long x) {
  u32 j = 0;
#pragma unroll
  for (u32 st = 16; st; st >>= 1) {
    const u32 p = j + st;
    const long long e = __shfl_sync(FULL, ev, p > 30 ? 30 : p);
    if (p <= 30 && e <= x) j = p;
  }
  return j;
}

// BFS level (K6): top-down expansion of a SORTED frontier over a CSR whose col_idx is paged.
// The frontier's out-edges form one virtual edge list [0, m) (eoff = exclusive scan of frontier
// degrees); warps take it in chunks of kChunk edges, so consecutive warps walk consecutive CSR
// positions: each col_idx page is resolved once per warp that needs it.  A window of 31 frontier
// vertices (lane j: eoff, CSR row start) maps each lane's edge to its CSR position by a 5-step
// shuffle search.  Discovery: one relaxed read of the visited bitmap (L2-resident: V/8 bytes),
// atomicOr only for unseen vertices, level[] store, and the next-frontier bitmap.  Async mode
// (pd > 0): a warp grabs pd chunks ahead and prefetches their pages before expanding the oldest
// (the AGILE prefetch pattern, gpu_api.py:139-155); pd = 0 is the synchronous baseline.
struct BfsWork {
  const long long* row_ptr;   // [rows+1] (HBM), row of vertex v at row_ptr[v - v0]
  u32 v0;                     // first vertex of the partition (1D vertex partition; 0 = whole graph)
  const int* frontier;        // [n] ascending
  const long long* eoff;      // [n+1], eoff[n] = m
  u32 n;
  u32* visited;               // [(V+31)/32]
  u32* next_bits;             // [(V+31)/32]
  int* level;
  int cur;
  u64 col_key0;
  u32 pd;
  u64* counters;              // [0] edges expanded, [1] page misses
  static constexpr u32 kChunk = 2048;
  static constexpr u32 kMaxPd = 4;

  __device__ __forceinline__ void load_window(u64 i, long long& ev, long long& rp) const {
    const u64 wi = i + lane_id();
    ev = wi <= n ? __ldcg(eoff + wi) : LLONG_MAX;
    rp = wi < n ? __ldg(row_ptr + (__ldg(frontier + wi) - (int)v0)) : 0;
  }

  __device__ void prefetch_chunk(const DevCtx& c, u64 ch, u64 m, u32 who, u32 sq) const {
    const u64 e0 = ch * kChunk, e1 = min(m, e0 + kChunk);
    const u64 i = warp_search_le(eoff, 0, n, (long long)e0);
    long long ev, rp;
    load_window(i, ev, rp);
    const long long evn = __shfl_down_sync(FULL, ev, 1);
    // lane j: the page of the first edge of window vertex j that falls in the chunk
    const bool has = lane_id() < 31 && (u64)ev < e1 && evn > ev && i + lane_id() < n;
    const long long first = ev < (long long)e0 ? (long long)e0 : ev;
    const u64 key = col_key0 + (u64)((rp + (first - ev)) >> 10);
    prefetch_warp(c, has, key, who, sq, true);
  }

  __device__ void run(const DevCtx& c, u32 uidx, u32 nusers) const {
    const u32 lane = lane_id();
    const u32 gw = uidx * kCtaWarps + (threadIdx.x >> 5);
    const u32 who = user_who(uidx);
    const u64 m = (u64)__ldcg(eoff + n);
    const u64 nch = (m + kChunk - 1) / kChunk;
    const u32 depth = pd > kMaxPd ? kMaxPd : pd;
    PageRegs pr;
    pr.clear();
    u32 misses = 0;
    u64 edges = 0;
    u64 ring[kMaxPd];
    u32 head = 0, count = 0;
    auto grab = [&]() -> u64 {
      u64 g = 0;
      if (lane == 0) g = atomicAdd(&c.run->work_next, 1ull);
      return __shfl_sync(FULL, g, 0);
    };
    for (u32 k = 0; k < depth; ++k) {
      const u64 g = grab();
      if (g >= nch) break;
      prefetch_chunk(c, g, m, who, gw + k);
      ring[(head + count) % kMaxPd] = g;
      ++count;
    }
    while (!aborted(c)) {
      u64 ch;
      if (depth) {
        if (!count) break;
        ch = ring[head];
        head = (head + 1) % kMaxPd;
        --count;
        const u64 g = grab();
        if (g < nch) {
          prefetch_chunk(c, g, m, who, gw + (u32)g);
          ring[(head + count) % kMaxPd] = g;
          ++count;
        }
      } else {
        ch = grab();
        if (ch >= nch) break;
      }
      const u64 e0 = ch * kChunk, e1 = min(m, e0 + kChunk);
      edges += e1 - e0;
      u64 i = warp_search_le(eoff, 0, n, (long long)e0);
      long long ev, rp;
      load_window(i, ev, rp);
      for (u64 e = e0; e < e1 && !aborted(c); e += 32) {
        const long long my = (long long)(e + lane);
        bool unloc = (u64)my < e1;
        Spin sp;
        while (__any_sync(FULL, unloc)) {
          const long long wend = __shfl_sync(FULL, ev, 31);
          bool inw = unloc && my < wend;
          if (!__any_sync(FULL, inw)) {
            // the earliest unlocated edge lies past the window: slide (one reload), else search
            const long long x = __shfl_sync(FULL, my, __ffs(__ballot_sync(FULL, unloc)) - 1);
            i += 31;
            load_window(i, ev, rp);
            if (x >= __shfl_sync(FULL, ev, 31)) {
              i = warp_search_le(eoff, i, n, x);
              load_window(i, ev, rp);
            }
            continue;
          }
          const u32 k = window_slot(ev, my);
          const long long pos = __shfl_sync(FULL, rp, k) + (my - __shfl_sync(FULL, ev, k));
          const u64 key = col_key0 + (u64)(pos >> 10);
          u32 line = 0;
          u64 word = 0;
          if (!resolve_pages_warp(c, inw, key, pr, line, word, who, gw, misses)) return;
          u32 u = 0;
          if (inw) u = __ldcg(reinterpret_cast<const unsigned int*>(line_ptr(c, line) + ((u32)pos & 1023u) * 4));
          if (!validate_pages_warp(c, inw, key, line, word)) {
            pr.clear();   // a page changed identity under the read: resolve again
            if (!sp.again(c, 256, __LINE__ + 100000 * SPIN_FILE_ID)) return;
            continue;
          }
          if (inw) {
            const u32 bit = 1u << (u & 31u);
            u32* vw = visited + (u >> 5);
            if (!(ld_relaxed(vw) & bit) && !(atomicOr(vw, bit) & bit)) {
              level[u] = cur + 1;
              atomicOr(next_bits + (u >> 5), bit);
            }
          }
          unloc = unloc && !inw;
        }
      }
    }
    if (lane == 0) {
      if (edges) atomicAdd(&counters[0], edges);
      if (misses) atomicAdd(&counters[1], (u64)misses);
    }
  }
};

// SpMV over a paged CSR (K7): y[r] = alpha * sum_e val[e] * x[col[e]] + beta.  col (int32) and val
// (fp32; val_key0 = ~0 -> unit weights, the PageRank A^T case) are paged; the edge list is cut
// into page-aligned chunks of 1024 edges, so one chunk = one col page (+ one val page) resolved
// once.  Lanes read 4 passes of 32 consecutive entries before touching x (ILP), map edges to rows
// through a window of 31 row starts, and sum rows with a segmented warp scan in a fixed order.
// Rows wholly inside a chunk are written directly; a row crossing a chunk boundary leaves its
// chunk partials in part_first / part_last, summed in chunk order by spmv_fixup_kernel
// (deterministic run to run).  Async mode (pd > 0) prefetches the pages of the chunks a warp
// grabbed ahead.
struct SpmvWork {
  const long long* row_ptr;   // [V+1]; row_ptr[0] > 0: edges before it belong to another partition
  u32 V;                      // rows
  u32 nx;                     // length of x (columns)
  u64 E;                      // edge positions [0, E) = row_ptr[V]
  const float* x;
  float* y;
  float alpha, beta;
  u64 col_key0, val_key0;
  double* part_first;         // [nchunks] partial of the chunk's first row if it began earlier
  double* part_last;          // [nchunks] partial of the chunk's last row if it continues
  u32* last_row;              // [nchunks]
  u32 pd;
  u64* counters;              // [0] edges, [1] page misses
  static constexpr u32 kChunk = 1024;
  static constexpr u32 kMaxPd = 4;

  __device__ void run(const DevCtx& c, u32 uidx, u32 nusers) const {
    const u32 lane = lane_id();
    const u32 gw = uidx * kCtaWarps + (threadIdx.x >> 5);
    const u32 who = user_who(uidx);
    const u64 nch = (E + kChunk - 1) / kChunk;
    const u64 e_lo = (u64)__ldg(row_ptr);
    const bool weighted = val_key0 != ~0ull;
    const u32 depth = pd > kMaxPd ? kMaxPd : pd;
    PageRegs pr;
    pr.clear();
    u32 misses = 0;
    u64 edges = 0;
    u64 ring[kMaxPd];
    u32 head = 0, count = 0;
    auto grab = [&]() -> u64 {
      u64 g = 0;
      if (lane == 0) g = atomicAdd(&c.run->work_next, 1ull);
      return __shfl_sync(FULL, g, 0);
    };
    auto prefetch = [&](u64 g, u32 sq) {
      const u64 key = (lane == 0) ? col_key0 + g : val_key0 + g;
      prefetch_warp(c, lane == 0 || (lane == 1 && weighted), key, who, sq, true);
    };
    for (u32 k = 0; k < depth; ++k) {
      const u64 g = grab();
      if (g >= nch) break;
      prefetch(g, gw + k);
      ring[(head + count) % kMaxPd] = g;
      ++count;
    }
    while (!aborted(c)) {
      u64 ch;
      if (depth) {
        if (!count) break;
        ch = ring[head];
        head = (head + 1) % kMaxPd;
        --count;
        const u64 g = grab();
        if (g < nch) {
          prefetch(g, gw + (u32)g);
          ring[(head + count) % kMaxPd] = g;
          ++count;
        }
      } else {
        ch = grab();
        if (ch >= nch) break;
      }
      const u64 e1 = min(E, ch * kChunk + kChunk);
      const u64 e0 = max(ch * kChunk, e_lo);   // a partition's first chunk may start mid-page
      const u64 ep = ch * kChunk;              // page base of the chunk
      if (e0 >= e1) continue;
      edges += e1 - e0;
      const u64 r0 = warp_search_le(row_ptr, 0, V, (long long)e0);
      Spin sp;
      while (true) {   // one attempt per chunk; redone if a page changed identity meanwhile
        // resolve the chunk's col page (lane 0) and val page (lane 1)
        const bool pa = lane == 0 || (lane == 1 && weighted);
        const u64 pkey = lane == 0 ? col_key0 + ch : val_key0 + ch;
        u32 pl = 0;
        u64 pw = 0;
        if (!resolve_pages_warp(c, pa, pkey, pr, pl, pw, who, gw, misses)) return;
        const uint8_t* colp = line_ptr(c, __shfl_sync(FULL, pl, 0));
        const uint8_t* valp = weighted ? line_ptr(c, __shfl_sync(FULL, pl, 1)) : nullptr;
        u64 r = r0;
        long long ev = (r + lane <= V) ? __ldcg(row_ptr + r + lane) : LLONG_MAX;
        u64 carry_row = ~0ull;
        double carry = 0.0;
        for (u32 p0 = 0; p0 < kChunk / 32; p0 += 4) {
          u32 col[4];
          float val[4], xv[4];
#pragma unroll
          for (u32 j = 0; j < 4; ++j) {
            const u64 e = ep + (p0 + j) * 32 + lane;
            col[j] = 0; val[j] = 1.f;
            if (e >= e0 && e < e1) {
              col[j] = __ldcg(reinterpret_cast<const unsigned int*>(colp) + ((p0 + j) * 32 + lane));
              if (weighted) val[j] = __ldcg(reinterpret_cast<const float*>(valp) + ((p0 + j) * 32 + lane));
            }
          }
#pragma unroll
          for (u32 j = 0; j < 4; ++j) {
            const u64 e = ep + (p0 + j) * 32 + lane;
            // col is speculative until the page is validated below: an index read from a line
            // that changed identity mid-read must not address outside x (the pass is redone)
            xv[j] = (e >= e0 && e < e1 && col[j] < nx) ? __ldg(x + col[j]) : 0.f;
          }
#pragma unroll
          for (u32 j = 0; j < 4; ++j) {
            const u64 pe0 = ep + (p0 + j) * 32;
            if (pe0 >= e1) break;
            if (pe0 + 32 <= e0) continue;
            const long long my = (long long)(pe0 + lane);
            bool unloc = (u64)my >= e0 && (u64)my < e1;
            // fp64: the product of two fp32 is exact, the sum is rounded once to fp32 at the end
            const double v0 = unloc ? (double)val[j] * (double)xv[j] : 0.0;
            // sub-rounds: the lanes whose edge the 31-row window covers (normally all of them)
            while (__any_sync(FULL, unloc)) {
              const long long x0 = __shfl_sync(FULL, my, __ffs(__ballot_sync(FULL, unloc)) - 1);
              long long wend = __shfl_sync(FULL, ev, 31);
              if (x0 >= wend) {
                r = warp_search_le(row_ptr, r + 31, V, x0);
                ev = (r + lane <= V) ? __ldcg(row_ptr + r + lane) : LLONG_MAX;
              } else {
                const u32 s0 = window_slot(ev, x0);
                if (s0 >= 16) {   // slide so the window starts at the current row
                  r += s0;
                  ev = (r + lane <= V) ? __ldcg(row_ptr + r + lane) : LLONG_MAX;
                }
              }
              wend = __shfl_sync(FULL, ev, 31);
              const bool inw = unloc && my < wend;
              const u32 k = window_slot(ev, my);
              const u64 row = inw ? r + k : ~0ull - lane;   // inactive lanes: distinct sentinels
              const long long rend = __shfl_sync(FULL, ev, k + 1 > 31 ? 31 : k + 1);
              double v = inw ? v0 : 0.0;
              const u32 ib = __ballot_sync(FULL, inw);
              const int fl = __ffs(ib) - 1, ll = 31 - __clz(ib);
              if ((int)lane == fl && row == carry_row) v += carry;
              double sum = v;
#pragma unroll
              for (u32 d = 1; d < 32; d <<= 1) {   // segmented inclusive scan, fixed order
                const double t = __shfl_up_sync(FULL, sum, d);
                const u64 rr = __shfl_up_sync(FULL, row, d);
                if (lane >= d && rr == row) sum += t;
              }
              const u64 rnext = __shfl_down_sync(FULL, row, 1);
              const bool seg_end = inw && ((int)lane == ll || rnext != row);
              const long long sub_end = __shfl_sync(FULL, my, ll) + 1;
              // the last segment continues past this sub-round but inside the chunk: carry it
              const bool cont = (int)lane == ll && rend > sub_end && (u64)sub_end < e1;
              carry_row = ~0ull;
              if (__any_sync(FULL, cont)) {
                carry_row = __shfl_sync(FULL, row, ll);
                carry = __shfl_sync(FULL, sum, ll);
              }
              if (seg_end && !cont) {
                const long long rstart = __ldcg(row_ptr + row);
                if (rstart < (long long)e0) {
                  part_first[ch] = sum;                     // began in an earlier chunk
                } else if (rend > (long long)e1) {
                  part_last[ch] = sum;                      // continues into later chunks
                  last_row[ch] = (u32)row;
                } else {
                  y[row] = (float)((double)alpha * sum + (double)beta);   // wholly inside this chunk
                }
              }
              unloc = unloc && !inw;
            }
          }
        }
        if (validate_pages_warp(c, pa, pkey, pl, pw)) break;
        pr.clear();
        if (!sp.again(c, 256, __LINE__ + 100000 * SPIN_FILE_ID)) return;
      }
    }
    if (lane == 0) {
      if (edges) atomicAdd(&counters[0], edges);
      if (misses) atomicAdd(&counters[1], (u64)misses);
    }
  }
};

}  // namespace agile
