// agile_work.cuh — user-side workloads (the consumers of the device library):
//   SeqWork        serialized async_read+wait stream (golden hit/miss/eviction parity)
//   ReadsWork      CTC sync/async epochs (bench/ctc.py:27-111)            — K8
//   LoopWork       closed-loop 4 KiB random reads (bench/bandwidth.py:20-68) — K9
//   GatherWork     prefetch + array_get gather epochs (bench/sweeps.py:39-88)
//   EmbBagWork     DLRM embedding-bag over cached rows                    — K5
#pragma once
#include "agile_core.cuh"
#undef SPIN_FILE_ID
#define SPIN_FILE_ID 2

namespace agile {

// grid barrier among user CTAs (the epoch Rendezvous, sim_core.py:139-159). All user CTAs are
// co-resident by construction (the host sizes the grid from occupancy for these workloads).
__device__ __forceinline__ bool user_grid_barrier(const DevCtx& c, u32 n_user_ctas) {
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
  __device__ void run(const DevCtx& c, u32 uidx, u32 nusers) {
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
  __device__ void issue(const DevCtx& c, u32 task, bool act, u32 e, u32 set, u32 who, u32 sq_start) {
    for (u32 i = 0; i < reads; ++i) {
      const u64 key = act ? keys[((u64)e * tasks + task) * reads + i] : 0ull;
      const u64 slot = ((u64)task * 2 + set) * reads + i;
      async_read_warp(c, act, key, nodes + (act ? slot : 0), bufs + (act ? slot : 0) * 256, who,
                      sq_start + i + e * reads);
    }
  }
  __device__ void wait_set(const DevCtx& c, u32 task, bool act, u32 set, u64& dg) {
    for (u32 i = 0; i < reads; ++i) {
      const u64 slot = ((u64)task * 2 + set) * reads + i;
      wait_nodes_warp(c, act, nodes + (act ? slot : 0));
      if (act) {
        const uint2 w = *reinterpret_cast<const uint2*>(bufs + slot * 256);
        dg ^= (u64)w.x | ((u64)w.y << 32);
      }
    }
  }
  __device__ void run(const DevCtx& c, u32 uidx, u32 nusers) {
    const u32 task = uidx * kCtaThreads + threadIdx.x;
    const bool act = task < tasks;
    const u32 who = user_who(uidx);
    const u32 sq_start = uidx * kCtaWarps + (threadIdx.x >> 5);
    u64 dg = 0;
    if (uidx == 0 && threadIdx.x == 0) epoch_t[0] = gtimer();
    if (!async_mode) {
      for (u32 e = 0; e < epochs; ++e) {
        issue(c, task, act, e, 0, who, sq_start);
        wait_set(c, task, act, 0, dg);
        // compute starts only after every task's data arrived (bench/ctc.py:80-83)
        if (!user_grid_barrier(c, nusers)) return;
        if (uidx == 0 && threadIdx.x == 0) epoch_t[e + 1] = gtimer();
        compute_spin(compute_ns);
      }
    } else {
      issue(c, task, act, 0, 0, who, sq_start);
      for (u32 e = 0; e < epochs; ++e) {
        const u32 cur = e & 1u;
        // the next epoch's fetches ride under this epoch's compute (bench/ctc.py:47-70)
        if (e + 1 < epochs) issue(c, task, act, e + 1, cur ^ 1u, who, sq_start);
        wait_set(c, task, act, cur, dg);
        if (!user_grid_barrier(c, nusers)) return;
        if (uidx == 0 && threadIdx.x == 0) epoch_t[e + 1] = gtimer();
        compute_spin(compute_ns);
      }
    }
    if (act) digest[task] = dg;
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
  u64 num_blocks;
  u64 warmup_ns, measure_ns;
  u64 max_per_task;
  __device__ void run(const DevCtx& c, u32 uidx, u32 nusers) {
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
        async_read_warp(c, issue, make_key(dev, blk), node, dst, who,
                        sq_start + (u32)__shfl_sync(FULL, j, __ffs(ib) - 1));
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

// ------------------------------------------------------------------ GatherWork (queue/cache sweeps)
// One warp = 32 tasks in lockstep (run_workload(..., warp_size=32)). Per epoch each task
// prefetches its gather set (warp-coalesced) and then array_gets element 0 of every block.
struct GatherWork {
  const u64* keys;        // [tasks][epochs][gathers]
  u32* values;            // [tasks][epochs][gathers] little-endian u32 read
  u64* epoch_t;
  u32 tasks, epochs, gathers, async_mode;
  u64 compute_ns;
  __device__ void prefetch_epoch(const DevCtx& c, bool act, u32 task, u32 e, u32 who, u32 sq_start) {
    for (u32 g = 0; g < gathers; ++g) {
      const u64 key = act ? keys[((u64)task * epochs + e) * gathers + g] : 0ull;
      prefetch_warp(c, act, key, who, sq_start + g + e * gathers, false);
    }
  }
  __device__ void get_epoch(const DevCtx& c, bool act, u32 task, u32 e, u32 who, u32 sq_start) {
    for (u32 g = 0; g < gathers; ++g) {
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
  __device__ void run(const DevCtx& c, u32 uidx, u32 nusers) {
    const u32 task = uidx * kCtaThreads + threadIdx.x;
    const bool act = task < tasks;
    const u32 who = user_who(uidx);
    const u32 sq_start = task / 32;   // thread_idx % nsq start SQ per warp (nvme_queue.py:91-93)
    if (uidx == 0 && threadIdx.x == 0) epoch_t[0] = gtimer();
    if (async_mode) prefetch_epoch(c, act, task, 0, who, sq_start);
    for (u32 e = 0; e < epochs; ++e) {
      if (!async_mode) prefetch_epoch(c, act, task, e, who, sq_start);
      else if (e + 1 < epochs) prefetch_epoch(c, act, task, e + 1, who, sq_start);
      get_epoch(c, act, task, e, who, sq_start);
      if (!user_grid_barrier(c, nusers)) return;
      compute_spin(compute_ns);
    }
    if (!user_grid_barrier(c, nusers)) return;
    if (uidx == 0 && threadIdx.x == 0) epoch_t[1] = gtimer();
  }
};

// ------------------------------------------------------------------ EmbBagWork (K5)
// pooled[b, t, :] = sum_l table_t[idx[b, t, l], :] over 4 KiB pages of 8 rows x 128 fp32.
// One warp per bag: lanes 0..L-1 map their index to (page, row slot), the warp probes all L
// pages with the batched ballot probe, misses are claimed/submitted warp-aggregated, then every
// lane loads one float4 of each row (16 B/lane, 512 B coalesced per row) and sums in registers.
// Hits are validated seqlock-style against the tag word after a fence (no pin atomics on the
// hot path).  Async mode prefetches the warp's bag `pd` positions ahead before processing.
struct EmbBagWork {
  const long long* idx;        // [B][T][L]
  const u64* table_key0;       // [T] key of the table's first page (dev << 36 | page)
  const long long* table_rows; // [T]
  float* out;                  // [B][T][D]
  u64* lookups_miss;           // [2] lookups, miss-path lookups
  u32 B, T, L, D;
  u32 pd;                      // prefetch distance in bags (0 = sync)
  u32 rows_per_page_shift;     // log2(4096 / (D*4))
  u32 out_b_stride, out_t_stride;   // in floats
  u32 nwarps_total;
  u32 prefetch_only;           // 1: pull every page of the batch toward the cache, no pooling

  __device__ __forceinline__ bool bag_keys(u32 bag, bool lane_act, u64& key, u32& off) const {
    const u32 b = bag / T, t = bag % T;
    if (!lane_act) return false;
    long long r = idx[((u64)b * T + t) * L + lane_id()];
    const long long rows = table_rows[t];
    if (r < 0 || r >= rows) r = 0;   // invalid index -> row 0 (callers validate on host)
    const u64 page = (u64)r >> rows_per_page_shift;
    const u32 slot = (u32)r & ((1u << rows_per_page_shift) - 1u);
    key = table_key0[t] + page;
    off = slot * D * 4;
    return true;
  }

  static constexpr u32 kMaxPd = 8;
  // next bag for this warp from the launch-wide counter (dynamic balance: a warp held up by a
  // slow miss does not hold back a static share of the batch)
  static constexpr u32 kGrab = 4;   // bags taken per counter atomic
  __device__ __forceinline__ u32 grab(const DevCtx& c, u32& pool, u32& left) const {
    if (!left) {
      u32 b = 0;
      if (lane_id() == 0) b = (u32)atomicAdd(&c.run->work_next, (u64)kGrab);
      pool = __shfl_sync(FULL, b, 0);
      left = kGrab;
    }
    --left;
    return pool++;
  }

  __device__ void run(const DevCtx& c, u32 uidx, u32 nusers) {
    const u32 lane = lane_id();
    const u32 gw = uidx * kCtaWarps + (threadIdx.x >> 5);
    const u32 nbags = B * T;
    const u32 who = user_who(uidx);
    const bool lact = lane < L;
    const u32 depth = pd > kMaxPd ? kMaxPd : pd;
    u32 misses_local = 0, lookups_local = 0;
    u32 gpool = 0, gleft = 0;
    if (prefetch_only) {
      // batch-level async (AGILE prefetch, gpu_api.py:345-361): submit every missing page of the
      // batch and return; the service keeps the launch alive until all fills completed
      while (true) {
        const u32 nb = grab(c, gpool, gleft);
        if (nb >= nbags) break;
        u64 key = 0; u32 off = 0;
        const bool a = bag_keys(nb, lact, key, off);
        prefetch_warp(c, a, key, who, gw + nb, false);
        lookups_local += L;
        if (aborted(c)) break;
      }
      if (lane == 0) atomicAdd(&lookups_miss[0], (u64)lookups_local);
      return;
    }
    // ring of grabbed-and-prefetched bags (async mode): the warp always has `depth` future bags'
    // misses in flight while it sums the oldest one
    u32 ring[kMaxPd];
    u32 head = 0, count = 0;
    for (u32 k = 0; k < depth; ++k) {
      const u32 nb = grab(c, gpool, gleft);
      if (nb >= nbags) break;
      u64 key = 0; u32 off = 0;
      const bool a = bag_keys(nb, lact, key, off);
      prefetch_warp(c, a, key, who, gw + k, true);
      ring[(head + count) % kMaxPd] = nb;
      ++count;
    }
    u32 pass = 0;
    while (true) {
      u32 bag;
      if (depth) {
        if (!count) break;
        bag = ring[head];
        head = (head + 1) % kMaxPd;
        --count;
        const u32 nb = grab(c, gpool, gleft);
        if (nb < nbags) {
          u64 key = 0; u32 off = 0;
          const bool a = bag_keys(nb, lact, key, off);
          prefetch_warp(c, a, key, who, gw + (++pass), true);
          ring[(head + count) % kMaxPd] = nb;
          ++count;
        }
      } else {
        bag = grab(c, gpool, gleft);
        if (bag >= nbags) break;
      }
      if (aborted(c)) break;
      u64 key = 0; u32 off = 0;
      const bool a = bag_keys(bag, lact, key, off);
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      bool first = true;
      u32 fails = 0;
      Spin rsp;
      while (true) {
        // 1. resolve every lookup to a READY line: batched ballot probe, then the miss path
        //    (claim or find the in-flight fill, wait for it) for the rest
        u32 line; u64 word;
        probe_lanes(c, a, key, line, word);
        bool ready = a && line != NONE && (tw_state(word) == ST_READY || tw_state(word) == ST_MODIFIED);
        if (ready && !tw_ref(word)) atomicOr(&c.tags[line], REF_BIT);   // on_hit
        u32 need = __ballot_sync(FULL, a && !ready);
        if (need && first) misses_local += __popc(need);
        Spin sp;
        while (need) {
          const bool nm = (need >> lane) & 1u;
          const Req r = access_warp(c, nm, key, false, who, gw, false);
          bool got = nm && (r.kind == R_HIT || r.kind == R_FILLING || r.kind == R_MISS);
          if (got) { line = r.line; word = r.word; }
          // wait for the fill; nothing is held meanwhile (a line reassigned under us goes again)
          u32 wp = __ballot_sync(FULL, got);
          u32 done = 0;
          Spin s2;
          while (wp) {
            bool rd = false, gone = false;
            if ((wp >> lane) & 1u) {
              const u64 w = ld_relaxed(&c.tags[line]);
              if (!tw_live(w) || tw_key(w) != key) gone = true;
              else if (tw_state(w) == ST_READY || tw_state(w) == ST_MODIFIED) { word = w; rd = true; }
            }
            done |= __ballot_sync(FULL, rd);
            wp &= ~__ballot_sync(FULL, rd || gone);
            if (wp && !s2.again(c, 1024, __LINE__ + 100000 * SPIN_FILE_ID)) break;
          }
          need &= ~done;
          if (aborted(c)) break;
          if (need && !done && !sp.again(c, 1024, __LINE__ + 100000 * SPIN_FILE_ID)) break;
        }
        if (aborted(c)) break;
        first = false;
        fence_acq_rel();
        // 2. sum the L rows, lane owns dims [4*lane, 4*lane+4): 8 row loads (16 B/lane, 512 B
        //    coalesced each) in flight per chunk, rows added in l order (bit-exact with the oracle)
        acc = make_float4(0.f, 0.f, 0.f, 0.f);
        const u64 rowaddr = a ? (u64)(uintptr_t)(line_ptr(c, line) + off) : 0ull;
        for (u32 l0 = 0; l0 < L; l0 += 8) {
          float4 v[8];
#pragma unroll
          for (u32 j = 0; j < 8; ++j) {
            const u64 ra = __shfl_sync(FULL, rowaddr, (l0 + j) & 31);
            v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (l0 + j < L && lane * 4 < D) v[j] = __ldcg(reinterpret_cast<const float4*>(ra) + lane);
          }
#pragma unroll
          for (u32 j = 0; j < 8; ++j) { acc.x += v[j].x; acc.y += v[j].y; acc.z += v[j].z; acc.w += v[j].w; }
        }
        // 3. seqlock validation, once per bag: no page changed identity while we read it;
        //    otherwise (rare) the whole bag is recomputed
        fence_acq_rel();
        bool bad = false;
        if (a) bad = ((ld_relaxed(&c.tags[line]) ^ word) & IDENT_MASK) != 0;
        if (!__any_sync(FULL, bad)) break;
        if (++fails >= 4) {
          // heavy eviction pressure: rows one at a time, each validated on its own (a single page
          // only has to survive one row read), still summed in l order
          acc = make_float4(0.f, 0.f, 0.f, 0.f);
          for (u32 l = 0; l < L && !aborted(c); ++l) {
            const u64 kl = __shfl_sync(FULL, key, l);
            const u32 ol = __shfl_sync(FULL, off, l);
            Spin s3;
            while (true) {
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
                  if (!s4.again(c, 1024, __LINE__ + 100000 * SPIN_FILE_ID)) break;
                }
                if (tw_live(w) && tw_key(w) == kl && tw_state(w) >= ST_READY) {
                  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                  if (lane * 4 < D) v = __ldcg(reinterpret_cast<const float4*>(line_ptr(c, ln) + ol) + lane);
                  fence_acq_rel();
                  if (((ld_relaxed(&c.tags[ln]) ^ w) & IDENT_MASK) == 0) {
                    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
                    break;
                  }
                }
              }
              if (!s3.again(c, 1024, __LINE__ + 100000 * SPIN_FILE_ID)) break;
            }
          }
          break;
        }
        if (!rsp.again(c, 256, __LINE__ + 100000 * SPIN_FILE_ID)) break;
      }
      lookups_local += L;
      const u32 b = bag / T, t = bag % T;
      if (lane * 4 < D) reinterpret_cast<float4*>(out + (u64)b * out_b_stride + (u64)t * out_t_stride)[lane] = acc;
    }
    if (lane == 0) {
      atomicAdd(&lookups_miss[0], (u64)lookups_local);
      atomicAdd(&lookups_miss[1], (u64)misses_local);
    }
  }
};

// ------------------------------------------------------------------ paged CSR reads (K6/K7)
// Read one u32 per active lane from page `key` at byte offset `off` through the cache: batched
// probe, miss path (claim or find the fill, wait), read, seqlock validation, retry.  Nothing is
// held across a wait.  Returns the value; lanes that gave up (abort) get 0.
__device__ u32 read_u32_warp(const DevCtx& c, bool active, u64 key, u32 off, u32 who, u32 sq_start) {
  const u32 lane = lane_id();
  u32 val = 0;
  bool pend = active;
  Spin sp;
  while (__any_sync(FULL, pend)) {
    u32 line; u64 word;
    probe_lanes(c, pend, key, line, word);
    bool ready = pend && line != NONE && (tw_state(word) == ST_READY || tw_state(word) == ST_MODIFIED);
    if (ready && !tw_ref(word)) atomicOr(&c.tags[line], REF_BIT);
    const bool nm = pend && !ready;
    if (__any_sync(FULL, nm)) {
      const Req r = access_warp(c, nm, key, false, who, sq_start, false);
      bool got = nm && (r.kind == R_HIT || r.kind == R_FILLING || r.kind == R_MISS);
      if (got) { line = r.line; word = r.word; }
      u32 wp = __ballot_sync(FULL, got);
      Spin s2;
      while (wp) {
        bool rd = false, gone = false;
        if ((wp >> lane) & 1u) {
          const u64 w = ld_relaxed(&c.tags[line]);
          if (!tw_live(w) || tw_key(w) != key) gone = true;
          else if (tw_state(w) == ST_READY || tw_state(w) == ST_MODIFIED) { word = w; rd = true; }
        }
        if (gone) got = false;
        wp &= ~__ballot_sync(FULL, rd || gone);
        if (wp && !s2.again(c, 1024, __LINE__ + 100000 * SPIN_FILE_ID)) break;
      }
      ready = ready || got;
      fence_acq_rel();
    }
    u32 v = 0;
    if (ready) v = __ldcg(reinterpret_cast<const unsigned int*>(line_ptr(c, line) + off));
    fence_acq_rel();
    bool ok = false;
    if (ready) ok = ((ld_relaxed(&c.tags[line]) ^ word) & IDENT_MASK) == 0;
    if (ok) { val = v; pend = false; }
    if (aborted(c)) break;
    if (__any_sync(FULL, pend) && !__any_sync(FULL, ok) && !sp.again(c, 1024, __LINE__ + 100000 * SPIN_FILE_ID)) break;
  }
  return val;
}

// BFS level (K6): top-down expansion of `frontier` over a CSR whose col_idx array is paged
// (1024 int32 per 4 KiB page, page p of the array = key col_key0 + p).  Warps take frontier
// vertices dynamically; lanes walk the vertex's edges 32 at a time, claim unvisited neighbours
// with a CAS on level[] and append them (warp-aggregated) to the next frontier.  With prefetch,
// each newly discovered vertex's first col_idx page is pulled toward the cache right away, so the
// next level's reads overlap this level's expansion (the AGILE async pattern).
struct BfsWork {
  const long long* row_ptr;   // [V+1] (HBM)
  int* level;                 // [V], -1 = unvisited
  const int* frontier;        // [n_in]
  int* next;                  // [V]
  unsigned int* next_count;
  u64 col_key0;
  u32 n_in;
  int cur;
  u32 prefetch;
  u64* counters;              // [0] edges traversed
  __device__ void run(const DevCtx& c, u32 uidx, u32 nusers) {
    const u32 lane = lane_id();
    const u32 gw = uidx * kCtaWarps + (threadIdx.x >> 5);
    const u32 who = user_who(uidx);
    u64 edges = 0;
    while (true) {
      u32 i = 0;
      if (lane == 0) i = (u32)atomicAdd(&c.run->work_next, 1ull);
      i = __shfl_sync(FULL, i, 0);
      if (i >= n_in || aborted(c)) break;
      const int v = frontier[i];
      const long long s = row_ptr[v], e = row_ptr[v + 1];
      edges += (u64)(e - s);
      for (long long b = s; b < e; b += 32) {
        const long long ed = b + lane;
        const bool act = ed < e;
        const u64 key = col_key0 + (u64)(act ? (ed >> 10) : 0);
        const u32 u = read_u32_warp(c, act, key, (u32)(act ? (ed & 1023) * 4 : 0), who, gw);
        bool disc = false;
        if (act && ld_relaxed(reinterpret_cast<const u32*>(level) + u) == 0xffffffffu)
          disc = atomicCAS(level + u, -1, cur + 1) == -1;
        const u32 db = __ballot_sync(FULL, disc);
        if (db) {
          u32 base = 0;
          if (lane == __ffs(db) - 1) base = atomicAdd(next_count, (u32)__popc(db));
          base = __shfl_sync(FULL, base, __ffs(db) - 1);
          if (disc) next[base + __popc(db & lanemask_lt())] = (int)u;
          if (prefetch) {
            u64 pk = 0;
            if (disc) pk = col_key0 + (u64)(row_ptr[u] >> 10);
            const bool has = disc && row_ptr[u + 1] > row_ptr[u];
            prefetch_warp(c, has, pk, who, gw, true);
          }
        }
      }
    }
    if (lane == 0 && edges) atomicAdd(&counters[0], edges);
  }
};

// SpMV over a paged CSR (K7): y[r] = alpha * sum_e val[e] * x[col[e]] + beta, col (int32) and val
// (fp32) paged (1024 per page; val_key0 = ~0 -> unit weights, the PageRank A^T case).  Warps take
// blocks of 32 rows dynamically; the next block's first pages are prefetched before the current
// block is processed (next-chunk prefetch).  One warp per row: lanes over the edges, warp sum.
struct SpmvWork {
  const long long* row_ptr;
  const float* x;
  float* y;
  u64 col_key0, val_key0;
  u32 V;
  float alpha, beta;
  u32 prefetch;
  u64* counters;   // [0] edges
  __device__ void run(const DevCtx& c, u32 uidx, u32 nusers) {
    const u32 lane = lane_id();
    const u32 gw = uidx * kCtaWarps + (threadIdx.x >> 5);
    const u32 who = user_who(uidx);
    const u32 nblocks = (V + 31) / 32;
    u64 edges = 0;
    u32 blk = 0;
    if (lane == 0) blk = (u32)atomicAdd(&c.run->work_next, 1ull);
    blk = __shfl_sync(FULL, blk, 0);
    while (blk < nblocks && !aborted(c)) {
      u32 nxt = 0;
      if (lane == 0) nxt = (u32)atomicAdd(&c.run->work_next, 1ull);
      nxt = __shfl_sync(FULL, nxt, 0);
      if (prefetch && nxt < nblocks) {
        // pull the next block's edge pages (col, and val when weighted) toward the cache
        const u32 r0 = nxt * 32, r1 = min(V, r0 + 32);
        const long long s0 = row_ptr[r0], s1 = row_ptr[r1];
        const long long p0 = s0 >> 10, p1 = (s1 + 1023) >> 10;
        const long long np = p1 - p0;
        const bool h = (long long)lane < np;
        prefetch_warp(c, h, col_key0 + (u64)(p0 + lane), who, gw + 1, true);
        if (val_key0 != ~0ull) prefetch_warp(c, h, val_key0 + (u64)(p0 + lane), who, gw + 2, true);
      }
      const u32 r0 = blk * 32, r1 = min(V, r0 + 32);
      for (u32 r = r0; r < r1; ++r) {
        const long long s = row_ptr[r], e = row_ptr[r + 1];
        float acc = 0.f;
        for (long long b = s; b < e; b += 32) {
          const long long ed = b + lane;
          const bool act = ed < e;
          const u64 pg = (u64)(act ? (ed >> 10) : 0);
          const u32 off = (u32)(act ? (ed & 1023) * 4 : 0);
          const u32 col = read_u32_warp(c, act, col_key0 + pg, off, who, gw);
          float w = 1.f;
          if (val_key0 != ~0ull) w = __uint_as_float(read_u32_warp(c, act, val_key0 + pg, off, who, gw));
          if (act) acc += w * __ldg(x + col);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
        if (lane == 0) y[r] = alpha * acc + beta;
        edges += (u64)(e - s);
      }
      blk = nxt;
    }
    if (lane == 0 && edges) atomicAdd(&counters[0], edges);
  }
};

}  // namespace agile
