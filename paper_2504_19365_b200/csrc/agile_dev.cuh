// agile_dev.cuh — B200 (sm_100a) device library for the AGILE async page-I/O hot path.
//
// Re-designs, for real GPU concurrency, the four hot-path layers of the reference
// simulator (/root/reference/pkg/src/agile_sim):
//   * software cache   software_cache.py:154-570  -> set-associative HBM page cache with packed
//                       64-bit tag words (state|ref|pins|version|key), warp-cooperative probe
//                       (__ballot_sync over ways), per-set clock hand, per-set claim lock held
//                       only across the O(1) claim (never across a wait), in-flight dedup.
//   * queue pairs      nvme_queue.py:96-354     -> SQ/CQ rings in HBM; warp-aggregated capacity-
//                       checked CAS reservation of the SQ tail (__match_any_sync), 64 B SQEs with
//                       EMPTY->UPDATED->ISSUED entry words, one doorbell publisher per SQ doing a
//                       lane-parallel batch scan, 16 B CQEs with phase bits.
//   * device engine    ssd_model.py:104-206     -> persistent warps that observe SQ doorbells,
//                       fetch ISSUED SQEs, run the channel/latency model on %globaltimer (model
//                       mode) or none (link mode), copy 4 KiB from the host-pinned mapped page
//                       store into the cache line and post CQEs, stalling on a full CQ.
//   * completion svc   agile_service.py:90-236  -> service warps rotating over CQs, 32-entry
//                       phase-checked windows, CQ doorbell only on full windows, SQE released
//                       before the cache completion, drain of partial windows at stop.
// Completion fan-out: async_read waiters sit on a per-line versioned waiter stack the service
// drains (copy + barrier), array/row readers poll the per-line tag word; nobody holds a lock or a
// pin while waiting, exactly the "no lock across a wait" rule of gpu_api.py:233-248.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace agile {

typedef unsigned long long u64;
typedef unsigned int u32;

constexpr int kBlockShift = 12;            // 4 KiB blocks == cache lines
constexpr u32 kBlockBytes = 1u << kBlockShift;
constexpr int kMaxDevices = 16;
constexpr int kWarp = 32;
constexpr int kCtaThreads = 256;
constexpr int kCtaWarps = kCtaThreads / kWarp;

// ---------------------------------------------------------------- tag word layout
// [63:62] state  [61] ref  [60:51] pins (async_read waiters)  [50:42] version  [41:0] key
// key = dev << 36 | blk   (64 devices x 2^36 blocks)
constexpr int KEY_BITS = 42;
constexpr u64 KEY_MASK = (1ull << KEY_BITS) - 1;
constexpr int DEV_SHIFT = 36;
constexpr u64 BLK_MASK = (1ull << DEV_SHIFT) - 1;
constexpr int VER_SHIFT = 42;
constexpr u64 VER_MASK = 0x1FFull << VER_SHIFT;
constexpr int PIN_SHIFT = 51;
constexpr u64 PIN_MASK = 0x3FFull << PIN_SHIFT;
constexpr u64 PIN_ONE = 1ull << PIN_SHIFT;
constexpr int REF_SHIFT = 61;
constexpr u64 REF_BIT = 1ull << REF_SHIFT;
constexpr int ST_SHIFT = 62;
constexpr u64 ST_MASK = 3ull << ST_SHIFT;
constexpr u64 IDENT_MASK = ST_MASK | VER_MASK | KEY_MASK;   // everything a reader validates

// victim-selection plug-ins (CachePolicy, software_cache.py:67-143)
enum : u32 { POL_CLOCK = 0, POL_MODULO = 1 };

// CacheState (software_cache.py:30-34)
enum : u32 { ST_INVALID = 0, ST_BUSY = 1, ST_READY = 2, ST_MODIFIED = 3 };

__host__ __device__ __forceinline__ u64 make_key(u32 dev, u64 blk) { return ((u64)dev << DEV_SHIFT) | (blk & BLK_MASK); }
__host__ __device__ __forceinline__ u32 key_dev(u64 key) { return (u32)(key >> DEV_SHIFT); }
__host__ __device__ __forceinline__ u64 key_blk(u64 key) { return key & BLK_MASK; }
__device__ __forceinline__ u32 tw_state(u64 w) { return (u32)(w >> ST_SHIFT); }
__device__ __forceinline__ u64 tw_key(u64 w) { return w & KEY_MASK; }
__device__ __forceinline__ u32 tw_pins(u64 w) { return (u32)((w & PIN_MASK) >> PIN_SHIFT); }
__device__ __forceinline__ bool tw_ref(u64 w) { return (w & REF_BIT) != 0; }
__device__ __forceinline__ u64 tw_make(u32 st, u64 key, u32 ver, bool ref, u32 pins) {
  return ((u64)st << ST_SHIFT) | (ref ? REF_BIT : 0ull) | ((u64)pins << PIN_SHIFT) |
         (((u64)ver << VER_SHIFT) & VER_MASK) | (key & KEY_MASK);
}
__device__ __forceinline__ u32 tw_ver(u64 w) { return (u32)((w & VER_MASK) >> VER_SHIFT); }
__device__ __forceinline__ bool tw_live(u64 w) { return tw_state(w) != ST_INVALID; }
// ident of the READY image of a BUSY word with the same key/version
__device__ __forceinline__ u64 ident_ready(u64 w) { return ((w & ~ST_MASK) & IDENT_MASK) | ((u64)ST_READY << ST_SHIFT); }

// SQ entry states (nvme_queue.py:27-30)
enum : u32 { SQ_EMPTY = 0, SQ_UPDATED = 1, SQ_ISSUED = 2 };
enum : u32 { OP_READ = 0, OP_WRITE = 1 };
// command context kinds (nvme_queue.py:41-44)
enum : u32 { K_FILL = 0, K_WB_KEEP = 1, K_WB_EVICT = 2, K_RAW = 3 };

// error codes, mapped back to the reference exception names by the host library
enum : u32 {
  E_OK = 0, E_PROTOCOL = 1,     // ProtocolViolation  nvme_queue.py:23
  E_UNKNOWN_CID = 2,            // UnknownCid         agile_service.py:27
  E_OUT_OF_RANGE = 3,           // OutOfRange         ssd_model.py:24
  E_ILLEGAL_STATE = 4,          // IllegalState       software_cache.py:26
  E_LIVELOCK = 5,               // LivelockSuspected  sim_core.py:23
  E_BUFFER_BUSY = 6,            // BufferBusy         gpu_api.py:21
  E_LOCK_CYCLE = 7,             // DeadlockDetector report (lock_chain.py:70-121), debug_locks
};

// stats slots (software_cache.py:166-170, agile_service.py:75-87, ssd_model.py:125-128)
enum : int {
  S_HITS = 0, S_MISSES, S_FILLS, S_WRITEBACKS, S_RESETS, S_ATTACHES, S_COMPLETIONS, S_WINDOWS,
  S_DRAIN_ENTRIES, S_BYTES_READ, S_BYTES_WRITTEN, S_FETCHED, S_DOORBELLS, S_SQ_FULL, S_CQE_STALLS,
  S_BARRIER_COUNT, S_BARRIER_NS, S_RETRIES, S_ENQUEUES, S_LOOKUPS, S_WAITS, S_NUM
};

// event-log codes (K10); rendered host-side into the reference trace tuples (sim_core.py:162-191)
enum : u32 { M_NVME = 0, M_SSD = 1, M_SVC = 2, M_CACHE = 3, M_API = 4, M_TABLE = 5, M_TEST = 6, M_LOCK = 7 };
enum : u32 {
  A_ENQUEUE = 0, A_SQE_UPDATED, A_SQE_ISSUED, A_DOORBELL, A_SQE_RELEASE, A_HEAD,
  A_FETCH, A_COMPLETE, A_CQE_POST, A_CQE_STALL,
  A_WINDOW_RING, A_DRAIN_RING, A_STOP, A_START, A_CQE_PROCESS,
  A_STATE, A_MISS, A_HIT, A_ATTACH, A_EVICT_RESET, A_DRAIN, A_ASYNC_READ, A_PREFETCH, A_INSTALL,
  A_WRITE_COMMIT, A_OBSERVE, A_REGISTER, A_SHARE, A_RELEASE, A_MODIFIED, A_PROPAGATE, A_DUTY_TRANSFER,
  A_EVICT_WB, A_WRITE_INTENT, A_DEADLOCK
};
enum : u32 { WHO_USER = 0u << 30, WHO_SVC = 1u << 30, WHO_DEV = 2u << 30, WHO_HOST = 3u << 30 };

struct alignas(64) SqWords {
  u64 tail;      // virtual reservation counter (CAS, capacity depth-1)
  u64 head;      // virtual head (advanced over completed prefix)
  u64 dbl;       // doorbell word: published doorbell (virtual, strictly increasing) << 1 | lock bit
                 // (one publisher at a time, nvme_queue.py:114): taking the lock returns the
                 // doorbell, one release store publishes the new doorbell and unlocks
  u64 pad0;
  u64 db_time;   // %globaltimer of the last publish (device model arrival)
  u64 fetched;   // engine-owned: next virtual index to fetch
  u64 pad1[2];
};

struct alignas(64) CqWords {
  u64 poll_offset;   // service-owned (under claim)
  u32 poll_mask;
  u32 claim;         // one poller warp at a time (nvme_queue.py:258)
  u64 host_db;       // CQ head doorbell rung by the service
  u64 dev_tail;      // engine-owned virtual post index
  u64 pad[4];
};

struct CmdCtx {      // side table indexed by (sq, slot) == CommandContext (nvme_queue.py:57-74)
  u64 key;
  u64 vidx;          // virtual SQ index of the command
  u64 t_submit;
  u32 line;          // 0xffffffff: raw command (no cache line)
  u32 kind;
  u64 buf;           // raw destination / source device address
};

struct alignas(64) RunWords {   // reset before every launch
  u32 ticket;        // fused launch: role by arrival order
  u32 users_started;
  u32 users_done;
  u32 infra_exited;
  u32 svc_exited;
  u32 engine_stop;
  u32 abort;
  u32 stop_logged;
  u32 bar_count;   // user-CTA grid barrier (epoch Rendezvous, sim_core.py:139-159)
  u32 bar_gen;
  u64 t_first;     // first user start (globaltimer)
  u64 work_next;   // dynamic work counter
  u64 t_marks[4];  // workload timestamps
};

struct alignas(64) PersistWords {   // survives launches
  unsigned long long outstanding;   // reserved - released commands (system.py:41)
  u32 error_code;
  u32 error_info;
  u64 error_a;
  u64 error_b;
  u64 pad[4];
};

struct Model {
  u32 link_mode;        // 1 = no latency model (raw host link), 0 = LatencyModel replay
  u32 parallelism;
  u64 read_ns, write_ns, fetch_ns;
  u32 jitter;           // 0 none, 1 uniform, 2 exponential
  u32 pad;
  u64 jitter_ns;
  u64 occupancy_ns;     // 0: occupancy == service (per_channel_rate unset)
  u64 seed;
};

struct DevCtx {
  // geometry
  u32 num_devices, pairs_per_device, num_qp, sq_depth, cq_depth, cq_window;
  u32 num_lines, ways, num_sets, sets_pow2;
  u32 service_warps, engine_warps, n_engine_ctas, n_service_ctas;
  u32 poll_ns, idle_max_ns;
  u32 trace;
  u32 solo_ok;              // 1: a user grid that never started is not an error (profiling mode)
  u32 policy;               // victim policy inside a set: POL_CLOCK | POL_MODULO (CachePolicy seam)
  u32 find_another;         // busy_eviction_choice: 0 wait, 1 find_another (software_cache.py:366-371)
  u32 st_buckets;           // share table (share_table.py:52-200): buckets (power of two), 0 = disabled
  u32 dbg_locks;            // debug_locks: wait-for cycle detection on every lock (lock_chain.py)
  u32 dbg_threads;          // size of lk_wait (user threads tracked)
  u64 watchdog_ns;
  u64 user_start_ns;        // the infra grid gives up on a user grid that has not started by then
  // cache
  u64* tags;
  unsigned short* sig;      // per-line 16-bit key signature: probe hint, the tag word decides
  u64* wl;                 // per-line async_read waiter stack (agile_core.cuh WaitNode)
  u32* set_lock;
  u32* hand;
  uint8_t* lines;
  u64 nodes_lo, nodes_hi;   // this run's WaitNode array (range checks on waiter-list walks)
  struct ShareEntry* st;    // share table entries [st_buckets]
  u32* st_lock;             // per-bucket locks [st_buckets]
  u32* lk_holder;           // debug_locks: holder thread + 1 per lock id (sets, SQ doorbells, buckets)
  u32* lk_wait;             // debug_locks: lock id + 1 each user thread spins on, 0 = none
  // queues
  uint4* sqe;              // num_qp * sq_depth * 4 (64 B each)
  u32* sq_state;
  u64* sq_done_v;
  SqWords* sqw;
  CmdCtx* cmd;
  uint4* cqe;              // num_qp * cq_depth (16 B each)
  CqWords* cqw;
  // engine
  u64* chan_free;          // num_devices * parallelism
  u64* chan_turn;          // num_devices * parallelism (round-robin dispatch turn)
  u32* dev_lock;           // num_devices
  u64* dev_seq;            // num_devices (jitter draw counter)
  const uint8_t* store[kMaxDevices];   // mapped host pointers (device view)
  uint8_t* store_w[kMaxDevices];
  u64 store_blocks[kMaxDevices];
  Model model;
  // control / metrics
  RunWords* run;
  PersistWords* pw;
  u64* stats;
  uint4* log;              // event records, 64 B each
  u64* log_count;
  u64 log_cap;
};

// ---------------------------------------------------------------- PTX memory-order helpers
__device__ __forceinline__ u64 ld_acquire(const u64* p) {
  u64 v; asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ u32 ld_acquire(const u32* p) {
  u32 v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ u64 ld_relaxed(const u64* p) {
  u64 v; asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ u32 ld_relaxed(const u32* p) {
  u32 v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void st_release(u64* p, u64 v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release(u32* p, u32 v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(u64* p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(u32* p, u32 v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ u64 atom_add_release(u64* p, u64 v) {
  u64 o; asm volatile("atom.release.gpu.global.add.u64 %0, [%1], %2;" : "=l"(o) : "l"(p), "l"(v) : "memory"); return o;
}
__device__ __forceinline__ u64 atom_cas_acqrel(u64* p, u64 cmp, u64 val) {
  u64 o; asm volatile("atom.acq_rel.gpu.global.cas.b64 %0, [%1], %2, %3;" : "=l"(o) : "l"(p), "l"(cmp), "l"(val) : "memory"); return o;
}
__device__ __forceinline__ u32 atom_cas_acqrel(u32* p, u32 cmp, u32 val) {
  u32 o; asm volatile("atom.acq_rel.gpu.global.cas.b32 %0, [%1], %2, %3;" : "=r"(o) : "l"(p), "r"(cmp), "r"(val) : "memory"); return o;
}
__device__ __forceinline__ u32 atom_cas_acquire(u32* p, u32 cmp, u32 val) {
  u32 o; asm volatile("atom.acquire.gpu.global.cas.b32 %0, [%1], %2, %3;" : "=r"(o) : "l"(p), "r"(cmp), "r"(val) : "memory"); return o;
}
__device__ __forceinline__ u64 atom_exch_acqrel(u64* p, u64 val) {
  u64 o; asm volatile("atom.acq_rel.gpu.global.exch.b64 %0, [%1], %2;" : "=l"(o) : "l"(p), "l"(val) : "memory"); return o;
}
__device__ __forceinline__ u64 atom_or_acquire(u64* p, u64 val) {
  u64 o; asm volatile("atom.acquire.gpu.global.or.b64 %0, [%1], %2;" : "=l"(o) : "l"(p), "l"(val) : "memory"); return o;
}
__device__ __forceinline__ u64 atom_or_acqrel(u64* p, u64 val) {
  u64 o; asm volatile("atom.acq_rel.gpu.global.or.b64 %0, [%1], %2;" : "=l"(o) : "l"(p), "l"(val) : "memory"); return o;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void fence_sc() { asm volatile("fence.sc.gpu;" ::: "memory"); }
__device__ __forceinline__ u64 gtimer() { u64 t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ u32 lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ u32 lanemask_lt() { u32 m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m; }
#ifndef AGILE_NAP_MAX_NS
#define AGILE_NAP_MAX_NS 0xffffffffu   // probe builds cap every backoff nap (tools: nap A/B)
#endif
__device__ __forceinline__ void nap(u32 ns) { __nanosleep(ns < AGILE_NAP_MAX_NS ? ns : AGILE_NAP_MAX_NS); }

__device__ __forceinline__ void set_error(const DevCtx& c, u32 code, u64 a, u64 b) {
  if (atomicCAS(&c.pw->error_code, 0u, code) == 0u) {
    c.pw->error_a = a; c.pw->error_b = b;
  }
  atomicExch(&c.run->abort, 1u);
}
__device__ __forceinline__ bool aborted(const DevCtx& c) { return ld_relaxed(&c.run->abort) != 0; }

// watchdog for every spin (LivelockSuspected-equivalent, sim_core.py:290-293)
struct Spin {
  u64 t0; u32 backoff;
  __device__ __forceinline__ Spin() : t0(0), backoff(32) {}
  // returns false when the run must unwind
  // site = __LINE__ + 100000 * file id of the spinning loop (reported as error_b)
  __device__ __forceinline__ bool again(const DevCtx& c, u32 max_ns = 2048, u32 site = 0) {
    if (aborted(c)) return false;
    u64 now = gtimer();
    if (t0 == 0) t0 = now;
    else if (now - t0 > c.watchdog_ns) { set_error(c, E_LIVELOCK, now - t0, site); return false; }
    nap(backoff);
    backoff = backoff * 2 > max_ns ? max_ns : backoff * 2;
    return true;
  }
};

// ---------------------------------------------------------------- event log (K10)
__device__ __forceinline__ void log_ev(const DevCtx& c, u32 who, u32 mod, u32 act, u64 a0 = 0, u64 a1 = 0,
                                       u64 a2 = 0, u64 a3 = 0, u64 a4 = 0, u64 a5 = 0) {
  if (!c.trace) return;
  u64 i = atomicAdd(c.log_count, 1ull);
  if (i >= c.log_cap) return;
  u64 t = gtimer();
  uint4* r = c.log + i * 4;
  r[0] = make_uint4((u32)t, (u32)(t >> 32), who, mod | (act << 8));
  r[1] = make_uint4((u32)a0, (u32)(a0 >> 32), (u32)a1, (u32)(a1 >> 32));
  r[2] = make_uint4((u32)a2, (u32)(a2 >> 32), (u32)a3, (u32)(a3 >> 32));
  r[3] = make_uint4((u32)a4, (u32)(a4 >> 32), (u32)a5, (u32)(a5 >> 32));
}

// warp-aggregated stats (one atomic per warp-flush)
struct LocalStats {
  u32 v[S_NUM];
  __device__ __forceinline__ LocalStats() { for (int i = 0; i < S_NUM; ++i) v[i] = 0; }
};
__device__ __forceinline__ void stat_add(const DevCtx& c, int slot, u64 n) {
  if (n) atomicAdd(&c.stats[slot], n);
}
// lane 0 adds a warp-uniform count
__device__ __forceinline__ void stat_warp(const DevCtx& c, int slot, u32 n) {
  if (lane_id() == 0 && n) atomicAdd(&c.stats[slot], (u64)n);
}

// ---------------------------------------------------------------- cache geometry
// set index: the plug-in hash of SURVEY A.2 (constants of share_table.py:66-68)
__host__ __device__ __forceinline__ u32 set_of_key(u64 key, u32 num_sets, u32 pow2) {
  // Fibonacci hashing (oracle/cache.py:set_of): x = blk * 2^32/phi (+ the high block bits and the
  // device, other odd constants) mod 2^32, scaled to [0, S) by a multiply-high: arithmetic
  // progressions of block ids spread with near-minimal discrepancy (the LOW bits of a
  // multiplicative hash fold strided ids onto a few sets)
  const u64 blk = key_blk(key);
  const u32 x = (u32)blk * 0x9E3779B9u + (u32)(blk >> 32) * 0x85EBCA77u + key_dev(key) * 0xC2B2AE35u;
  (void)pow2;
  return (u32)(((u64)x * num_sets) >> 32);
}
__device__ __forceinline__ u32 set_of(const DevCtx& c, u64 key) { return set_of_key(key, c.num_sets, c.sets_pow2); }
// 16-bit signature of a key (independent of the set-index bits): a set's W signatures are 2W
// bytes, so one lane scans a 32-way set with four 16 B loads instead of 32 tag words
__host__ __device__ __forceinline__ u32 sig16(u64 key) { return (u32)((key * 0x9E3779B97F4A7C15ull) >> 48); }
__device__ __forceinline__ uint8_t* line_ptr(const DevCtx& c, u32 line) { return c.lines + ((u64)line << kBlockShift); }

}  // namespace agile
