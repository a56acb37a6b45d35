/* agile_oracle.c — CPU port of the paged embedding-bag through the AGILE software cache.
 *
 * TEST INFRASTRUCTURE / CPU BASELINE ONLY (see oracle/__init__.py).  Restates, on host cores:
 *   - the block-granular software cache with clock replacement (software_cache.py:91-126,
 *     355-456), generalised to S sets x W ways exactly as SURVEY A.2's plug-in (per-set hand,
 *     same skip/ref rules, hit and insert set ref);
 *   - the device read of a missing block into its cache line (ssd_model.py:188-192); the block's
 *     bytes are the synthetic store contents of oracle/pages.py (page_floats: every 32-bit half h
 *     of splitmix64(seed ^ dev<<56 ^ blk<<9 ^ k) stored as (h >> 8) * 2^-23 - 1);
 *   - the embedding-bag built on read_range (software_cache.py:212-219, the gather stand-in of
 *     bench/sweeps.py): pooled[b,t,:] = sum_l row(idx[b,t,l]), accumulated in fp64 (l ascending)
 *     and rounded once to fp32 — the GPU kernel's definition (exact sum, correctly rounded,
 *     whenever the fp64 sum is exact).
 * Threads split the bags; a per-set spinlock serialises each set (the reference's policy lock,
 * software_cache.py:163, narrowed to one set).
 */
#include <pthread.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define BLOCK 4096

typedef struct {
  uint64_t lines, ways, sets;
  uint64_t* tag;      /* key + 1, 0 = invalid */
  uint8_t* ref;
  uint32_t* hand;
  atomic_flag* lock;
  float* data;        /* lines * 1024 floats */
  uint64_t seed;
  uint32_t row_dim;   /* 0: page-keyed contents (page_floats); D: row-keyed tables (row_floats) */
  atomic_ullong hits, misses, evictions;
} ocache;

static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

static inline uint32_t set_of(uint64_t dev, uint64_t blk, uint64_t sets) {
  const uint32_t x = (uint32_t)blk * 0x9E3779B9u + (uint32_t)(blk >> 32) * 0x85EBCA77u +
                     (uint32_t)dev * 0xC2B2AE35u;   /* Fibonacci hashing */
  return (uint32_t)(((uint64_t)x * sets) >> 32);
}

void* oracle_cache_create(uint64_t lines, uint64_t ways, uint64_t seed) {
  if (!ways || ways > lines) ways = lines;
  if (lines % ways) return NULL;
  ocache* c = calloc(1, sizeof(ocache));
  c->lines = lines; c->ways = ways; c->sets = lines / ways; c->seed = seed;
  c->tag = calloc(lines, sizeof(uint64_t));
  c->ref = calloc(lines, 1);
  c->hand = calloc(c->sets, sizeof(uint32_t));
  c->lock = calloc(c->sets, sizeof(atomic_flag));
  for (uint64_t s = 0; s < c->sets; ++s) atomic_flag_clear(&c->lock[s]);
  c->data = malloc(lines * (uint64_t)BLOCK);   /* touched lazily as lines fill */
  return c;
}

void oracle_cache_destroy(void* h) {
  ocache* c = h;
  if (!c) return;
  free(c->tag); free(c->ref); free(c->hand); free(c->lock); free(c->data); free(c);
}

void oracle_cache_stats(void* h, uint64_t* out) {
  ocache* c = h;
  out[0] = atomic_load(&c->hits); out[1] = atomic_load(&c->misses); out[2] = atomic_load(&c->evictions);
}

/* device read of block (dev, blk) into a line: the page_floats contents */
static void fetch_block(const ocache* c, uint64_t dev, uint64_t blk, float* dst) {
  for (uint32_t k = 0; k < 512; ++k) {
    uint64_t x = splitmix64(c->seed ^ (dev << 56) ^ (blk << 9) ^ k);
    dst[2 * k] = (float)((uint32_t)x >> 8) * (1.0f / 8388608.0f) - 1.0f;
    dst[2 * k + 1] = (float)((uint32_t)(x >> 32) >> 8) * (1.0f / 8388608.0f) - 1.0f;
  }
}

/* row-keyed table page (oracle/pages.py row_floats): rows first_row.. of `table`, D fp32 each */
static void fetch_rows(const ocache* c, uint32_t table, uint64_t first_row, uint64_t table_rows, float* dst) {
  const uint32_t D = c->row_dim, rpp = BLOCK / (4 * D);
  for (uint32_t s = 0; s < rpp; ++s) {
    const uint64_t r = first_row + s;
    for (uint32_t k = 0; k < D / 2; ++k) {
      uint64_t x = 0;
      if (r < table_rows) x = splitmix64(c->seed ^ ((uint64_t)table << 56) ^ (r << 8) ^ k);
      float lo = (float)((uint32_t)x >> 8) * (1.0f / 8388608.0f) - 1.0f;
      float hi = (float)((uint32_t)(x >> 32) >> 8) * (1.0f / 8388608.0f) - 1.0f;
      if (r >= table_rows) lo = hi = 0.0f;
      dst[s * D + 2 * k] = lo;
      dst[s * D + 2 * k + 1] = hi;
    }
  }
}

void oracle_cache_rowkeyed(void* h, uint32_t D) { ((ocache*)h)->row_dim = D; }

/* access (dev, blk) under its set lock; returns the line index (lock held on return).  A miss
 * fills the line with the block's contents: page-keyed, or rows of (table, page_in_table). */
static uint64_t access_locked(ocache* c, uint64_t dev, uint64_t blk, uint32_t table, uint64_t page_in_table,
                              uint64_t table_rows, uint32_t* set_out) {
  const uint32_t s = set_of(dev, blk, c->sets);
  *set_out = s;
  while (atomic_flag_test_and_set_explicit(&c->lock[s], memory_order_acquire)) { }
  const uint64_t base = (uint64_t)s * c->ways;
  const uint64_t key = ((dev << 36) | blk) + 1;
  for (uint64_t w = 0; w < c->ways; ++w) {
    if (c->tag[base + w] == key) {
      c->ref[base + w] = 1;
      atomic_fetch_add_explicit(&c->hits, 1, memory_order_relaxed);
      return base + w;
    }
  }
  atomic_fetch_add_explicit(&c->misses, 1, memory_order_relaxed);
  uint64_t victim = base;
  for (uint64_t scanned = 0; scanned < 2 * c->ways; ++scanned) {
    const uint32_t w = c->hand[s];
    c->hand[s] = (uint32_t)((w + 1) % c->ways);
    if (c->ref[base + w]) { c->ref[base + w] = 0; continue; }
    victim = base + w;
    break;
  }
  if (c->tag[victim]) atomic_fetch_add_explicit(&c->evictions, 1, memory_order_relaxed);
  c->tag[victim] = key;
  c->ref[victim] = 1;
  if (c->row_dim)
    fetch_rows(c, table, page_in_table * (BLOCK / (4 * c->row_dim)), table_rows, c->data + victim * 1024);
  else
    fetch_block(c, dev, blk, c->data + victim * 1024);
  return victim;
}

typedef struct {
  ocache* c;
  const int64_t* idx;
  const uint64_t* key0;
  const int64_t* rows;
  const int64_t* table_id;   /* global table id of every table of the launch (row-keyed mode) */
  float* out;
  uint32_t B, T, L, D;
  uint64_t bag0, bag1;
  int bad;   /* an index outside [0, rows) was seen (OutOfRange) */
} job;

static void* run_bags(void* arg) {
  job* j = arg;
  ocache* c = j->c;
  const uint32_t rpp = BLOCK / (4 * j->D);
  for (uint64_t bag = j->bag0; bag < j->bag1; ++bag) {
    const uint64_t t = bag % j->T;
    float* o = j->out + bag * j->D;
    double acc[BLOCK / 4];
    memset(acc, 0, sizeof(double) * j->D);
    const uint64_t dev = j->key0[t] >> 36;
    const uint64_t page0 = j->key0[t] & ((1ull << 36) - 1);
    for (uint32_t l = 0; l < j->L; ++l) {
      int64_t r = j->idx[bag * j->L + l];
      if (r < 0 || r >= j->rows[t]) { j->bad = 1; continue; }
      uint32_t s;
      const uint64_t line = access_locked(c, dev, page0 + (uint64_t)r / rpp, (uint32_t)j->table_id[t],
                                          (uint64_t)r / rpp, (uint64_t)j->rows[t], &s);
      const float* row = c->data + line * 1024 + (uint64_t)(r % rpp) * j->D;
      for (uint32_t d = 0; d < j->D; ++d) acc[d] += (double)row[d];
      atomic_flag_clear_explicit(&c->lock[s], memory_order_release);
    }
    for (uint32_t d = 0; d < j->D; ++d) o[d] = (float)acc[d];
  }
  return NULL;
}

/* pooled[B][T][D]; idx[B][T][L]; returns 0, or -2 when an index is out of range */
int oracle_embbag(void* h, const int64_t* idx, const uint64_t* key0, const int64_t* rows, const int64_t* table_id,
                  float* out, uint32_t B, uint32_t T, uint32_t L, uint32_t D, int nthreads) {
  ocache* c = h;
  if (!c || D == 0 || (BLOCK / 4) % D || (c->row_dim && (c->row_dim != D || !table_id))) return -1;
  if (nthreads < 1) nthreads = 1;
  const uint64_t nb = (uint64_t)B * T;
  pthread_t th[256];
  job jobs[256];
  if (nthreads > 256) nthreads = 256;
  for (int i = 0; i < nthreads; ++i) {
    jobs[i] = (job){c, idx, key0, rows, table_id, out, B, T, L, D, nb * i / nthreads, nb * (i + 1) / nthreads, 0};
    if (nthreads == 1) run_bags(&jobs[i]);
    else pthread_create(&th[i], NULL, run_bags, &jobs[i]);
  }
  if (nthreads > 1)
    for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
  for (int i = 0; i < nthreads; ++i)
    if (jobs[i].bad) return -2;
  return 0;
}
