/* agile_b200.h — C-ABI of the B200-native AGILE async page-I/O hot path.
 *
 * One context per GPU (one process per rank under torch.distributed).  The context owns the HBM
 * page cache (tag words + 4 KiB lines), the SQ/CQ rings and side tables, the completion service
 * and device-engine state, and one host-pinned GPU-mapped page store per emulated device.
 * Every workload entry point is one AGILE run on the caller's stream: an infra grid (device
 * engine K4 + completion service K3) and a PDL-launched user grid running the workload against
 * the device library (K1 cache, K2 queue engine), which starts only once every infra CTA is
 * resident.  When a co-residency probe at agile_create sees a PDL dependent NOT run beside its
 * primary (kernel-serialising tools), the context launches one fused grid instead, whose CTAs
 * take their roles by arrival order (AGILE_LAUNCH=split|fused forces either).
 *
 * Every function returns 0 on success or a negative code; agile_last_error() has the message.
 * Codes -101.. map to the reference exception types:
 *   AGILE_E_PROTOCOL     ProtocolViolation   (nvme_queue.py:23)
 *   AGILE_E_UNKNOWN_CID  UnknownCid          (agile_service.py:27)
 *   AGILE_E_OUT_OF_RANGE OutOfRange          (ssd_model.py:24)
 *   AGILE_E_ILLEGAL      IllegalState        (software_cache.py:26)
 *   AGILE_E_LIVELOCK     LivelockSuspected   (sim_core.py:23)
 *   AGILE_E_BUFFER_BUSY  BufferBusy          (gpu_api.py:21)
 *   AGILE_E_LOCK_CYCLE   DeadlockDetector report (lock_chain.py:70-121; debug_locks = on)
 * Config errors (unknown key / bad value) return AGILE_E_CONFIG (ValueError/KeyError in Python).
 */
#ifndef AGILE_B200_H
#define AGILE_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct agile_ctx agile_ctx;

#define AGILE_OK 0
#define AGILE_E_CUDA (-1)
#define AGILE_E_ARG (-2)
#define AGILE_E_CONFIG (-3)
#define AGILE_E_PROTOCOL (-101)
#define AGILE_E_UNKNOWN_CID (-102)
#define AGILE_E_OUT_OF_RANGE (-103)
#define AGILE_E_ILLEGAL (-104)
#define AGILE_E_LIVELOCK (-105)
#define AGILE_E_BUFFER_BUSY (-106)
#define AGILE_E_LOCK_CYCLE (-107)

/* stats slots (agile_stats) — software_cache.py:166-170, agile_service.py:75-87, ssd_model.py:125-128 */
enum {
  AGILE_S_HITS = 0, AGILE_S_MISSES, AGILE_S_FILLS, AGILE_S_WRITEBACKS, AGILE_S_RESETS, AGILE_S_ATTACHES,
  AGILE_S_COMPLETIONS, AGILE_S_WINDOWS, AGILE_S_DRAIN_ENTRIES, AGILE_S_BYTES_READ, AGILE_S_BYTES_WRITTEN,
  AGILE_S_FETCHED, AGILE_S_DOORBELLS, AGILE_S_SQ_FULL, AGILE_S_CQE_STALLS, AGILE_S_BARRIER_COUNT,
  AGILE_S_BARRIER_NS, AGILE_S_RETRIES, AGILE_S_ENQUEUES, AGILE_S_LOOKUPS, AGILE_S_WAITS, AGILE_S_NUM
};

/* Replaces AgileSystem.__init__ (system.py:35-90): geometry comes from the resolved config text
 * (config.py:220-230 `config_text`, key = value lines).  Keys read here: num_devices, seed,
 * device.{num_blocks,block_size,read_latency_ns,write_latency_ns,parallelism,jitter,jitter_ns,
 * per_channel_rate,emulation}, queues.{pairs_per_device,sq_depth,cq_depth},
 * cache.{lines,bytes,ways,policy,busy_choice}, share_table.enabled, service.{warps,poll_ns,
 * idle_max_ns}, engine.warps, timing.fetch_ns, debug_locks, livelock_budget. */
int agile_create(const char* config_text, int cuda_device, agile_ctx** out);
int agile_destroy(agile_ctx* ctx);
const char* agile_last_error(agile_ctx* ctx);
/* geometry[0..10] = num_devices, pairs_per_device, sq_depth, cq_depth, lines, ways, sets,
 * engine_warps, service_warps, infra_ctas, launch mode (0 split, 1 fused) */
int agile_geometry(agile_ctx* ctx, uint64_t* out, int n);

/* Launch mode of later runs: 0 split (infra grid + PDL user grid), 1 fused (one grid, roles by
 * arrival ticket), 2 split with solo users (when a kernel-serialising tool keeps the user grid
 * from starting beside the infra grid, the infra grid leaves after 100 ms and the user grid runs
 * alone), 3 users only (profiling: no infra grid; an all-hit replay needs neither engine nor
 * service, a miss ends in the watchdog). */
int agile_set_launch_mode(agile_ctx* ctx, int mode);
/* engine.copy of later runs: 0 registers (register-staged page moves, whole infra SMs), 1 bulk
 * (TMA bulk copies through shared-memory slots; user CTAs fit beside the infra CTAs) */
int agile_set_engine_copy(agile_ctx* ctx, int bulk);

/* Third-party user kernels (include/agile_device.cuh, the paper's Listing 1 API): begin one split
 * run on `stream` — run words reset, infra grid launched — and receive the DevCtx / Launch values
 * (sizes checked against the caller's build) the user grid must be launched with
 * (agile::launch_user), plus a device array of n_bufs WaitNodes for AgileBufPtr barriers.  The
 * user kernel must run n_user_ctas CTAs of 256 threads, each constructing agile::UserRun.
 * agile_user_run_end waits for the run and surfaces device-side errors. */
int agile_user_run_begin(agile_ctx* ctx, void* stream, uint32_t n_user_ctas, uint64_t n_bufs, void* devctx_out,
                         uint64_t devctx_size, void* launch_out, uint64_t launch_size, void** nodes_out);
int agile_user_run_end(agile_ctx* ctx, void* stream);

/* Backing store (BlockStore, ssd_model.py:61-101): pinned + GPU-mapped host memory, caller-owned
 * when host_ptr != NULL (registered), else context-owned and zeroed.  image_path (optional) is a
 * raw little-endian block image, offset = blk * 4096, short tail zero-padded (load_image). */
int agile_store_attach(agile_ctx* ctx, int dev, void* host_ptr, uint64_t num_blocks, const char* image_path);
int agile_store_ptr(agile_ctx* ctx, int dev, void** host_ptr, uint64_t* num_blocks);
/* BlockStore.load_image (ssd_model.py:84-95) into the attached store: blocks present in the raw
 * image are overwritten (short last block zero-padded), the others keep their bytes, views from
 * agile_store_ptr stay valid, and the device's cache lines are invalidated (IllegalState if a run
 * of the context is still in flight). */
int agile_store_load_image(agile_ctx* ctx, int dev, const char* path);
/* synthetic page contents (oracle/pages.py): kind 0 = u64 word k of block b is
 * page_word(seed, dev, b, k); kind 1 = fp32 table values, each 32-bit half h of that word stored
 * as (h >> 8) * 2^-23 - 1 (page_floats) */
int agile_store_fill(agile_ctx* ctx, int dev, uint64_t seed, uint64_t first_blk, uint64_t nblk, int kind);
int agile_store_save_image(agile_ctx* ctx, int dev, const char* path);
/* embedding rows keyed by (table, global row) (oracle/pages.py row_floats): pages
 * [first_blk, first_blk + ceil(rows / (1024 / D))) receive rows [row0, row0 + rows) of table
 * `table` (< 256), 1024 / D rows of D fp32 per page; u64 word k of row r is
 * splitmix64(seed ^ table<<56 ^ r<<8 ^ k), each 32-bit half h stored as (h >> 8) * 2^-23 - 1.
 * Any row-wise sharding of a table therefore holds the same values as the whole table. */
int agile_store_fill_rows(agile_ctx* ctx, int dev, uint64_t seed, uint64_t first_blk, uint32_t table, uint64_t row0,
                          uint64_t rows, uint32_t D);

/* reset flags: 1 cache (tags/hands/locks), 2 queues + service/engine state, 4 stats */
int agile_reset(agile_ctx* ctx, int flags);
int agile_stats(agile_ctx* ctx, uint64_t* out, int n);
/* K10 event log: enable with capacity (records of 64 B); read back rendered by the host */
int agile_trace_enable(agile_ctx* ctx, uint64_t capacity);
int agile_event_log(agile_ctx* ctx, void* out, uint64_t cap, uint64_t* n);
/* wait for the stream and surface device-side protocol errors */
int agile_sync(agile_ctx* ctx, void* stream);

/* Serialized async_read + wait stream (one task): golden hit/miss/eviction sequence and page
 * bytes under a fixed issue order.  Host arrays.  outcome: 0 hit, 1 miss, 2 attach; victim: key
 * (dev << 36 | blk) of the READY line evicted by the access, or UINT64_MAX. */
int agile_run_seq(agile_ctx* ctx, const uint32_t* dev, const uint64_t* blk, int64_t n, int8_t* outcome,
                  uint64_t* victim, void* pages_out);

/* CTC epochs (bench/ctc.py:27-111): device pointers.  keys[epochs][tasks][reads] (dev<<36|blk),
 * bufs = tasks*2*reads*4096 bytes, digest[tasks], epoch_t[epochs+1] (globaltimer ns). */
int agile_run_reads(agile_ctx* ctx, const uint64_t* keys, uint32_t tasks, uint32_t reads, uint32_t epochs,
                    int async_mode, uint64_t compute_ns, void* bufs, uint64_t* digest, uint64_t* epoch_t,
                    void* stream);

/* Closed-loop 4 KiB reads (bench/bandwidth.py:20-68): conc requesters, one outstanding each.
 * counters[0] = completions inside [warmup, warmup+measure), counters[1..2] = window (ns). */
int agile_run_loop(agile_ctx* ctx, uint32_t conc, uint64_t warmup_ns, uint64_t measure_ns,
                   uint64_t max_per_task, void* bufs, uint64_t* counters, void* stream);

/* Same, write_mode != 0: each requester keeps one async_write (bench/bandwidth.py:20-42 write
 * mode): its buffer (bytes idx & 0xFF) lands in the cache line and is written through to the
 * device; counters[0] counts completed writes. */
int agile_run_loop_rw(agile_ctx* ctx, uint32_t conc, uint64_t warmup_ns, uint64_t measure_ns,
                      uint64_t max_per_task, void* bufs, uint64_t* counters, int write_mode, void* stream);

/* async_write + wait of n whole blocks (SoftwareCache.write_block / AgileApi.async_write,
 * software_cache.py:221-235, gpu_api.py:192-227), one GPU thread per block, host buffers:
 * pages[n][4096].  Each block lands in its cache line (resident: overwritten in place; else a
 * victim is claimed) and is written through to the device store before the call returns. */
int agile_write_blocks(agile_ctx* ctx, const uint32_t* dev, const uint64_t* blk, int64_t n, const void* pages);

/* SoftwareCache.evict per block (software_cache.py:268-281, _evict_locked 335-353): outcome[i]
 * 0 = RESET (the READY line was dropped), 1 = DEFERRED (busy or pinned), 2 = not resident (the
 * reference reports RESET for an absent / INVALID line), 3 = WRITEBACK_STARTED (a MODIFIED line:
 * written back, then INVALID). */
int agile_evict_blocks(agile_ctx* ctx, const uint32_t* dev, const uint64_t* blk, int64_t n, int8_t* outcome);

/* AgileApi.array_get (gpu_api.py:250-278), n elements at once, host arrays: element idx[i] of
 * device dev[i] viewed as a little-endian array of elem_size-byte elements (elem_size must divide
 * 4096, else AGILE_E_ARG = ValueError; a block past the store raises AGILE_E_OUT_OF_RANGE).  Each
 * element is read through the cache (hit, attach to a fill in flight, or miss + fill) and its raw
 * bytes land at out + i * elem_size. */
int agile_array_get(agile_ctx* ctx, const uint32_t* dev, const uint64_t* idx, int64_t n, uint32_t elem_size,
                    void* out);

/* debug_locks demonstration (tests/test_lock_chain.py:26-95): mode 0 plants a ring of n warps, each
 * holding set lock w and taking set lock (w+1) mod n; mode 1 has one warp take set lock 0 twice.
 * With debug_locks the wait-for cycle is reported in the event log ("lock", "deadlock") and the
 * call returns AGILE_E_LOCK_CYCLE; without it the spins end in LivelockSuspected. */
int agile_lock_cycle_demo(agile_ctx* ctx, uint32_t n, int mode);
/* BufferBusy (gpu_api.py:132-137): a transfer started on a buffer whose previous transfer is still
 * pending (async_read, then async_read / async_write without wait) returns AGILE_E_BUFFER_BUSY. */
int agile_buffer_busy_demo(agile_ctx* ctx, int write);
/* SoftwareCache.flush (software_cache.py:283-298): write back every MODIFIED line (lines the share
 * table drained into the cache) and wait for durability; *flushed = lines written back. */
int agile_flush(agile_ctx* ctx, uint64_t* flushed);
/* ShareTable.live_entries (share_table.py:198-199) */
int agile_share_live(agile_ctx* ctx, uint64_t* live);
/* The reference's coherence replay workload (tests/test_coherence.py:27-60) with share_table.enabled
 * on or off: tasks (<= 8, one warp each) run plans of op[t][i] (0 read, 1 write) on block
 * blk[t][i] of device 0 after think[t][i] ns; writes carry the prefix 1<<30 | t<<16 | i; reads
 * observe the first 8 bytes of the buffer they got (seen[t][i]); with the table every read holds
 * its reference to the end, then releases; finally every MODIFIED line is flushed (*flushed).  The
 * event log (agile_trace_enable) carries the reference's install / write_commit / observe records
 * in a commit-consistent order for the sequential replay. */
int agile_run_coherence(agile_ctx* ctx, const uint8_t* op, const uint32_t* blk, const uint32_t* think, uint32_t tasks,
                        uint32_t ops, uint64_t* seen, uint64_t* flushed);

/* Gather epochs (bench/sweeps.py:39-88): keys[tasks][epochs][gathers]; values = u32 element 0
 * of every gathered block; epoch_t[2] = start/end. */
int agile_run_gather(agile_ctx* ctx, const uint64_t* keys, uint32_t tasks, uint32_t epochs, uint32_t gathers,
                     int async_mode, uint64_t compute_ns, uint32_t* values, uint64_t* epoch_t, void* stream);

/* DLRM embedding-bag (K5), device pointers: idx[B][T][L] int64 rows, table_key0[T] first page
 * key of each table, table_rows[T], out[b*out_b_stride + t*out_t_stride + d] fp32 (sum pooling,
 * fp64 accumulation rounded once), counters[2] += {lookups, miss-path lookups}.  Indices outside
 * [0, table_rows[t]) raise AGILE_E_OUT_OF_RANGE.  prefetch_distance 0 = sync mode, > 0 = each
 * warp prefetches the next block of bags it grabbed while it pools the current one. */
int agile_embbag(agile_ctx* ctx, const int64_t* idx, const uint64_t* table_key0, const int64_t* table_rows,
                 float* out, uint64_t* counters, uint32_t B, uint32_t T, uint32_t L, uint32_t D,
                 uint32_t out_b_stride, uint32_t out_t_stride, uint32_t prefetch_distance, void* stream);
/* Sharded / variable-length embedding-bag (K5), device pointers.  One agile_table_shard per
 * table of the launch: a whole table (row0 = 0, rows = table_rows) or one rank's row range of a
 * table split row-wise over ranks (BASELINE configs[4]).  Lookup l of bag (b, t) is
 * idx[(b*T + t)*L + l] (offsets == NULL) or idx[offsets[b*T + t] + l] for l < offsets[b*T+t+1] -
 * offsets[b*T+t] (offsets[B*T + 1], variable-length bags, torch embedding_bag's include_last_offset
 * convention).  Indices outside [0, table_rows) raise AGILE_E_OUT_OF_RANGE; indices outside the
 * shard's [row0, row0 + rows) are another rank's and skipped.  Sums accumulate in fp64: a shard
 * with AGILE_TAB_PARTIAL_F64 writes its D fp64 partial sums (for the receiver to add after the
 * exchange), otherwise the sum is rounded once to D fp32.  Table t of sample b lands at
 * (char*)out + b*out_row_bytes + tables[t].out_offset — e.g. straight into a peer-major
 * all-to-all send buffer.  mode 0 = pool, 1 = prefetch only (AgileApi.prefetch over the batch:
 * every missing page submitted, the call completes when all fills landed; out may be NULL). */
typedef struct agile_table_shard {
  uint64_t key0;        /* page key of the shard's first page: dev << 36 | page */
  int64_t row0;         /* first global row held by this shard */
  int64_t rows;         /* rows held: global rows [row0, row0 + rows) */
  int64_t table_rows;   /* rows of the whole table */
  uint32_t out_offset;  /* byte offset of the table's pooled vector in an output row (16 B aligned) */
  uint32_t flags;       /* AGILE_TAB_PARTIAL_F64 */
} agile_table_shard;
#define AGILE_TAB_PARTIAL_F64 1u
int agile_embbag_sharded(agile_ctx* ctx, const int64_t* idx, const int64_t* offsets, const agile_table_shard* tables,
                         void* out, uint64_t out_row_bytes, uint64_t* counters, uint32_t B, uint32_t T, uint32_t L,
                         uint32_t D, uint32_t prefetch_distance, uint32_t user_ctas, int mode, void* stream);
/* Same, with the launch bounded to user_ctas user CTAs (0 = every resident slot): a gather issued
 * on a side stream beside compute (the DLRM MLPs) leaves the remaining SMs to that compute. */
int agile_embbag_ctas(agile_ctx* ctx, const int64_t* idx, const uint64_t* table_key0, const int64_t* table_rows,
                      float* out, uint64_t* counters, uint32_t B, uint32_t T, uint32_t L, uint32_t D,
                      uint32_t out_b_stride, uint32_t out_t_stride, uint32_t prefetch_distance, uint32_t user_ctas,
                      void* stream);
/* Same, host buffers (end-to-end through the C-ABI: H2D of indices, kernel, D2H of pooled out). */
int agile_embbag_host(agile_ctx* ctx, const int64_t* idx, const uint64_t* table_key0, const int64_t* table_rows,
                      float* out, uint64_t* counters, uint32_t B, uint32_t T, uint32_t L, uint32_t D,
                      uint32_t prefetch_distance);
/* Asynchronous host-buffer entry, double-buffered (slot 0 / 1): enqueue H2D of the indices, the
 * run and D2H of the pooled output on the slot's own stream and return.  Runs of the two slots
 * execute in submission order (one context), while one slot's copies overlap the other's run.
 * Host buffers should be pinned for the copies to be asynchronous; `out` and `counters` are
 * valid after agile_embbag_host_wait(slot), which must precede the slot's next submit.  When `out`
 * is pinned, device-mapped host memory (cudaHostAlloc / cudaHostRegister), the kernel stores the
 * pooled rows into it directly instead of staging them for a copy-engine download. */
int agile_embbag_host_submit(agile_ctx* ctx, const int64_t* idx, const uint64_t* table_key0,
                             const int64_t* table_rows, float* out, uint64_t* counters, uint32_t B, uint32_t T,
                             uint32_t L, uint32_t D, uint32_t prefetch_distance, int slot);
int agile_embbag_host_wait(agile_ctx* ctx, int slot);
/* Batch-level prefetch (AGILE prefetch): submit every missing page of the batch into the cache
 * and complete once all fills landed; no pooling.  user_ctas (0 = all) bounds the SMs it takes
 * so the DLRM MLPs of the previous batch can run beside it. */
int agile_embbag_prefetch(agile_ctx* ctx, const int64_t* idx, const uint64_t* table_key0, const int64_t* table_rows,
                          uint64_t* counters, uint32_t B, uint32_t T, uint32_t L, uint32_t D, uint32_t user_ctas,
                          void* stream);
/* Breadth-first search over a paged CSR (K6; BASELINE configs[2]; new workload, the reference
 * has no graph driver).  row_ptr[V+1] int64 in HBM; col_idx int32 lives in the page
 * store from page key col_key0 (1024 entries per 4 KiB page) and is read through the HBM cache.
 * level[V] int32 (device) receives the BFS level of every vertex, -1 if unreached.  Level-
 * synchronous top-down over a sorted frontier; prefetch_distance = edge chunks a warp grabs and
 * prefetches ahead (0 = synchronous).  stats (host, may be NULL): [0] levels, [1] edges expanded,
 * [2] page misses, [3] device ns. */
int agile_bfs(agile_ctx* ctx, const int64_t* row_ptr, uint32_t V, uint32_t source, uint64_t col_key0,
              int32_t* level, uint32_t prefetch_distance, uint64_t* stats, void* stream);
/* SpMV over a paged CSR (K7; configs[3]): y = alpha * A x + beta for E edges; col int32 and val
 * fp32 paged one page per 1024 edges (val_key0 = UINT64_MAX: unit weights, the PageRank A^T
 * case).  Deterministic summation order; exact fp64 products summed in fp64, y rounded once to
 * fp32.  counters (device u64[2]) += {edges, page misses}. */
int agile_spmv(agile_ctx* ctx, const int64_t* row_ptr, uint32_t V, uint64_t E, uint64_t col_key0, uint64_t val_key0,
               const float* x, float* y, float alpha, float beta, uint32_t prefetch_distance, uint64_t* counters,
               void* stream);
/* SpMV over the rows of a 1D vertex partition (configs[3] over N GPUs): rows [0, n_rows) of the
 * rank's CSR; row_ptr[0] may be > 0 — edge positions [0, row_ptr[0]) belong to the previous
 * partition and are skipped, so a rank whose col/val pages start at the unpartitioned CSR's page
 * holding its first edge (positions = global - a page-aligned base) cuts its edges into the same
 * 1024-edge chunks as one GPU would, and every row sum is formed in the same order.  x has x_len
 * entries (the global vertex vector, col ids index it).  Products are exact in fp64 and summed in
 * fp64, y rounded once to fp32; y[r] = alpha * sum + beta, rows without edges get beta. */
int agile_spmv_rows(agile_ctx* ctx, const int64_t* row_ptr, uint32_t n_rows, uint64_t e_end, uint32_t x_len,
                    uint64_t col_key0, uint64_t val_key0, const float* x, float* y, float alpha, float beta,
                    uint32_t prefetch_distance, uint64_t* counters, void* stream);
/* One top-down BFS level over the frontier vertices a rank owns (1D vertex partition, configs[2]
 * over N GPUs): row_ptr[v - v0] for owned v (positions into the rank's paged col_idx from
 * col_key0), frontier[n] ascending global vertex ids, visited / next_bits (global bitmaps,
 * (V+31)/32 words; next_bits zeroed by the caller) and level[V] (global) updated for every
 * vertex discovered here; the caller ORs next_bits over ranks (all-gather) to form the next
 * frontier.  counters (device u64[2]) += {edges expanded, page misses}.  Async launch. */
int agile_bfs_level(agile_ctx* ctx, const int64_t* row_ptr, uint32_t v0, const int32_t* frontier, uint32_t n,
                    uint32_t* visited, uint32_t* next_bits, int32_t* level, int32_t cur, uint64_t col_key0,
                    uint32_t prefetch_distance, uint64_t* counters, void* stream);
/* number of user CTAs the embbag launch uses (for roofline accounting) */
int agile_embbag_grid(agile_ctx* ctx, uint32_t* user_ctas, uint32_t* infra_ctas);

#ifdef __cplusplus
}
#endif
#endif
