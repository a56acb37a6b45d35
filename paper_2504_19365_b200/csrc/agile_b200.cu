// agile_b200.cu — host side of the C-ABI (include/agile_b200.h): context construction from the
// reference's config text, HBM layout, pinned/mapped page stores, fused launches, error surfacing.
#include <cuda_runtime.h>
#include <cub/cub.cuh>
#include <algorithm>
#include <type_traits>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/agile_b200.h"
#include "agile_work.cuh"

using namespace agile;

struct agile_ctx {
  int device = 0;
  DevCtx d{};
  std::vector<void*> dev_allocs;
  void* host_store[kMaxDevices] = {};
  bool store_owned[kMaxDevices] = {};
  uint64_t store_blocks[kMaxDevices] = {};
  std::string err;
  int sms = 148;
  uint64_t seed = 0;
  // pinned staging for agile_embbag_host
  void* h_stage = nullptr;
  size_t h_stage_bytes = 0;
  void* d_stage = nullptr;
  size_t d_stage_bytes = 0;
  cudaStream_t stream = nullptr;
  // double-buffered host-buffer pipeline (agile_embbag_host_submit / _wait): per slot a stream,
  // device staging, pinned counters and the event of its run (runs are ordered across slots)
  struct HostSlot {
    cudaStream_t st = nullptr;
    void* d = nullptr;
    size_t bytes = 0;
    uint64_t* h_cnt = nullptr;   // pinned [2]
    uint64_t* user_cnt = nullptr;
    cudaEvent_t ran = nullptr;
    bool busy = false;
  } hs[2];
  int last_slot = -1;
  // launch mode: false = split (infra grid + PDL user grid, the default), true = one fused grid
  // with roles by arrival ticket (AGILE_LAUNCH=fused: what a kernel-serialising profiler captures)
  bool fused = false;
  // engine.copy: false = register-staged page moves, true = TMA bulk copies through shared memory
  bool bulk_engine = false;
  // launch mode 3 (profiling): the user grid runs without an infra grid
  bool users_only = false;
  // infra grid of bounded side-stream runs (engine.side_warps / service.side_warps; 0 = full)
  uint32_t side_engine_warps = 0, side_service_warps = 0;
  // async_read WaitNodes (AgileBuf barriers) for the reads / loop / seq workloads
  void* nodes = nullptr;
  size_t nodes_cap = 0;
  // named device scratch for the graph drivers (frontiers, bitmaps, scans, chunk partials)
  std::map<std::string, std::pair<void*, size_t>> scratch;
};

namespace {

int fail(agile_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(ctx, AGILE_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

std::map<std::string, std::string> parse_kv(const char* text) {
  std::map<std::string, std::string> kv;
  std::istringstream in(text ? text : "");
  std::string line;
  while (std::getline(in, line)) {
    const size_t hash = line.find('#');
    if (hash != std::string::npos) line = line.substr(0, hash);
    const size_t eq = line.find('=');
    if (eq == std::string::npos) continue;
    auto trim = [](std::string s) {
      const size_t a = s.find_first_not_of(" \t\r\n");
      const size_t b = s.find_last_not_of(" \t\r\n");
      return a == std::string::npos ? std::string() : s.substr(a, b - a + 1);
    };
    kv[trim(line.substr(0, eq))] = trim(line.substr(eq + 1));
  }
  return kv;
}

struct Cfg {
  std::map<std::string, std::string> kv;
  std::string bad;
  // integer keys: exact 64-bit parse (config_text renders Python ints in decimal), the whole value
  // must be consumed; negative values are rejected except where `allow_neg` (the seed, stored as
  // its two's complement so distinct seeds stay distinct)
  uint64_t u(const char* k, uint64_t def, bool allow_neg = false) {
    auto it = kv.find(k);
    if (it == kv.end() || it->second.empty()) return def;
    const char* txt = it->second.c_str();
    char* end = nullptr;
    errno = 0;
    uint64_t v;
    if (txt[0] == '-') {
      const long long sv = strtoll(txt, &end, 10);
      if (!allow_neg) { bad = k; return def; }
      v = (uint64_t)sv;
    } else {
      v = strtoull(txt, &end, 10);
    }
    while (end && (*end == ' ' || *end == '\t')) ++end;
    if (end == txt || (end && *end) || errno == ERANGE) { bad = k; return def; }
    return v;
  }
  double f(const char* k, double def) {
    auto it = kv.find(k);
    if (it == kv.end() || it->second.empty()) return def;
    return atof(it->second.c_str());
  }
  std::string s(const char* k, const char* def) {
    auto it = kv.find(k);
    return it == kv.end() ? std::string(def) : it->second;
  }
  bool b(const char* k, bool def) {
    auto it = kv.find(k);
    if (it == kv.end()) return def;
    std::string v = it->second;
    for (auto& ch : v) ch = (char)tolower(ch);
    return v == "true" || v == "1" || v == "yes" || v == "on";
  }
};

bool pow2(uint64_t x) { return x && !(x & (x - 1)); }

// per-call device scratch, freed on every return path (the early returns of CK included)
struct DevTmp {
  std::vector<void*> p;
  DevTmp() = default;
  DevTmp(const DevTmp&) = delete;
  DevTmp& operator=(const DevTmp&) = delete;
  ~DevTmp() {
    for (void* q : p) cudaFree(q);
  }
  template <class T>
  cudaError_t alloc(T** out, size_t bytes) {
    void* q = nullptr;
    const cudaError_t e = cudaMalloc(&q, std::max<size_t>(bytes, 16));
    if (e == cudaSuccess) p.push_back(q);
    *out = reinterpret_cast<T*>(q);
    return e;
  }
};

template <class T>
int dalloc(agile_ctx* ctx, T** p, size_t count) {
  void* q = nullptr;
  const size_t bytes = std::max<size_t>(count * sizeof(T), 64);
  CK(cudaMalloc(&q, bytes));
  CK(cudaMemset(q, 0, bytes));
  ctx->dev_allocs.push_back(q);
  *p = reinterpret_cast<T*>(q);
  return 0;
}

int device_error(agile_ctx* ctx) {
  PersistWords pw;
  CK(cudaMemcpy(&pw, ctx->d.pw, sizeof(pw), cudaMemcpyDeviceToHost));
  if (!pw.error_code) return 0;
  static const char* names[] = {"ok", "ProtocolViolation", "UnknownCid", "OutOfRange", "IllegalState",
                                "LivelockSuspected", "BufferBusy", "LockCycle"};
  char buf[256];
  snprintf(buf, sizeof buf, "%s (device) a=%llu b=%llu", pw.error_code < 8 ? names[pw.error_code] : "?",
           (unsigned long long)pw.error_a, (unsigned long long)pw.error_b);
  ctx->err = buf;
  const int code = -(100 + (int)pw.error_code);
  // clear so the context can be reset and reused
  PersistWords z{};
  z.outstanding = pw.outstanding;
  cudaMemcpy(ctx->d.pw, &z, sizeof(z), cudaMemcpyHostToDevice);
  return code;
}

WaitNode* get_nodes_raw(agile_ctx* ctx, size_t n) {
  if (n > ctx->nodes_cap) {
    if (ctx->nodes) { cudaDeviceSynchronize(); cudaFree(ctx->nodes); }
    ctx->nodes = nullptr;
    ctx->nodes_cap = 0;
    if (cudaMalloc(&ctx->nodes, n * sizeof(WaitNode)) != cudaSuccess) return nullptr;
    cudaMemset(ctx->nodes, 0, n * sizeof(WaitNode));
    ctx->nodes_cap = n;
  }
  return reinterpret_cast<WaitNode*>(ctx->nodes);
}

// the run's AgileBuf barriers, zeroed on the run's stream (t_issue 0 = never used: the BufferBusy
// check of a fresh run never sees a previous run's state)
WaitNode* get_nodes(agile_ctx* ctx, size_t n, cudaStream_t st = nullptr) {
  WaitNode* w = get_nodes_raw(ctx, n);
  if (w && cudaMemsetAsync(w, 0, n * sizeof(WaitNode), st ? st : ctx->stream) != cudaSuccess) return nullptr;
  return w;
}

// dynamic shared memory of a workload's launch (W::kDynSmem when it declares one: the embedding-
// bag row stages); set once per instantiation above the 48 KiB default
template <class W, class = void>
struct DynSmem { static constexpr size_t bytes = 0; };
template <class W>
struct DynSmem<W, std::void_t<decltype(W::kDynSmem)>> { static constexpr size_t bytes = W::kDynSmem; };

template <class W>
size_t dyn_smem() {
  constexpr size_t b = DynSmem<W>::bytes;
  if (b > 48 * 1024) {
    static bool set = false;
    if (!set) {
      cudaFuncSetAttribute(agile_user_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b);
      cudaFuncSetAttribute(agile_fused_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b);
      set = true;
    }
  }
  return b;
}

// the context's infra kernel (engine.copy) and its dynamic shared memory (the bulk engine's slots)
using InfraFn = void (*)(const DevCtx, const Launch);
InfraFn infra_fn(const agile_ctx* ctx) { return ctx->bulk_engine ? agile_infra_kernel<true> : agile_infra_kernel<false>; }
size_t infra_smem(const agile_ctx* ctx) {
  if (!ctx->bulk_engine) return 0;
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(agile_infra_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kInfraSmem);
    set = true;
  }
  return kInfraSmem;
}

// Lazy module loading would load the user kernel at its first launch, i.e. while the infra grid
// it must run beside is already spinning — loading can wait for the device to drain, and the two
// grids would deadlock.  Touching both functions first loads them before any run starts.
template <class W>
void load_kernels() {
  static bool loaded = false;
  if (loaded) return;
  cudaFuncAttributes a{};
  cudaFuncGetAttributes(&a, agile_infra_kernel<false>);
  cudaFuncGetAttributes(&a, agile_infra_kernel<true>);
  cudaFuncGetAttributes(&a, agile_user_kernel<W>);
  cudaFuncGetAttributes(&a, agile_fused_kernel<W>);
  loaded = true;
}

// side: a bounded run beside other work (user_ctas given): its infra grid may be smaller
// (engine.side_warps / service.side_warps).  Engine and service ownership is by stride over the
// queue pairs and all their state persists in the context, so the infra size can change from run
// to run.
// reset the run words and launch the infra grid of one split run; dc / L receive what the user grid
// of the run is launched with
int launch_infra(agile_ctx* ctx, uint32_t n_user_ctas, cudaStream_t st, bool side, DevCtx& dc, Launch& L) {
  dc = ctx->d;
  dc.nodes_lo = (u64)(uintptr_t)ctx->nodes;
  dc.nodes_hi = dc.nodes_lo + (u64)ctx->nodes_cap * sizeof(WaitNode);
  if (side && !ctx->fused) {
    if (ctx->side_engine_warps) {
      dc.engine_warps = ctx->side_engine_warps;
      dc.n_engine_ctas = (dc.engine_warps + kCtaWarps - 1) / kCtaWarps;
    }
    if (ctx->side_service_warps) {
      dc.service_warps = ctx->side_service_warps;
      dc.n_service_ctas = (dc.service_warps + kCtaWarps - 1) / kCtaWarps;
    }
  }
  CK(cudaMemsetAsync(ctx->d.run, 0, sizeof(RunWords), st));
  L.n_user_ctas = n_user_ctas;
  L.pad = 0;
  if (ctx->fused) return 0;
  if (ctx->users_only) {
    // profiling replays of all-hit batches: no infra grid at all; the user grid finds the
    // "infra gave up" mark and runs alone (a miss would end in the watchdog)
    static const u32 gave_up = kInfraGaveUp;
    CK(cudaMemcpyAsync(&ctx->d.run->users_started, &gave_up, 4, cudaMemcpyHostToDevice, st));
    dc.n_engine_ctas = dc.n_service_ctas = 0;
    return 0;
  }
  infra_fn(ctx)<<<dc.n_engine_ctas + dc.n_service_ctas, kCtaThreads, infra_smem(ctx), st>>>(dc, L);
  CK(cudaGetLastError());
  return 0;
}

// side: a bounded run beside other work (user_ctas given): its infra grid may be smaller
// (engine.side_warps / service.side_warps).  Engine and service ownership is by stride over the
// queue pairs and all their state persists in the context, so the infra size can change from run
// to run.
template <class W>
int launch(agile_ctx* ctx, const W& work, uint32_t n_user_ctas, cudaStream_t st, bool side = false) {
  if (n_user_ctas == 0) n_user_ctas = 1;
  load_kernels<W>();
  dyn_smem<W>();
  DevCtx dc;
  Launch L;
  int rc = launch_infra(ctx, n_user_ctas, st, side, dc, L);
  if (rc) return rc;
  if (ctx->fused) {
    const uint32_t ninfra = dc.n_engine_ctas + dc.n_service_ctas;
    agile_fused_kernel<W><<<ninfra + n_user_ctas, kCtaThreads, dyn_smem<W>(), st>>>(dc, L, work);
    CK(cudaGetLastError());
    return 0;
  }
  // the user grid may start once every infra CTA executed griddepcontrol.launch_dependents
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_user_ctas);
  cfg.blockDim = dim3(kCtaThreads);
  cfg.dynamicSmemBytes = dyn_smem<W>();
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, agile_user_kernel<W>, dc, L, work));
  return 0;
}

// user CTAs of workload W that are co-resident with the infra grid: the user grid's occupancy
// over all SMs minus the user CTAs each infra CTA displaces on its SM (registers bound both)
template <class W>
uint32_t resident_ctas(agile_ctx* ctx) {
  if (ctx->fused) {
    int f = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&f, agile_fused_kernel<W>, kCtaThreads, dyn_smem<W>());
    const uint32_t tot = (uint32_t)std::max(1, f) * (uint32_t)ctx->sms;
    const uint32_t ninfra = ctx->d.n_engine_ctas + ctx->d.n_service_ctas;
    return tot > ninfra + 1 ? tot - ninfra : 1;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, agile_user_kernel<W>, kCtaThreads, dyn_smem<W>());
  if (per_sm < 1) per_sm = 1;
  cudaFuncAttributes ua{}, ia{};
  cudaFuncGetAttributes(&ua, agile_user_kernel<W>);
  cudaFuncGetAttributes(&ia, infra_fn(ctx));
  // user CTAs left on an SM that also hosts one infra CTA: registers (allocated per warp in units
  // of 8 per thread), shared memory (the engine's page slots) and warp slots all bound it
  int regs_sm = 65536, smem_sm = 233472, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  auto warp_regs = [](int r) { return (uint32_t)((std::max(1, r) + 7) / 8 * 8 * 32); };
  const uint32_t u_regs = warp_regs(ua.numRegs) * kCtaWarps, i_regs = warp_regs(ia.numRegs) * kCtaWarps;
  const uint64_t u_smem = (uint64_t)ua.sharedSizeBytes + dyn_smem<W>() + 1024, i_smem = ia.sharedSizeBytes + infra_smem(ctx) + 1024;
  uint32_t beside = (uint32_t)per_sm;
  beside = std::min<uint32_t>(beside, regs_sm > (int)i_regs ? ((uint32_t)regs_sm - i_regs) / u_regs : 0u);
  beside = std::min<uint64_t>(beside, (uint64_t)smem_sm > i_smem ? ((uint64_t)smem_sm - i_smem) / u_smem : 0u);
  beside = std::min<uint32_t>(beside, (64u - kCtaWarps) / kCtaWarps);
  const uint32_t displaced = (uint32_t)per_sm - beside;
  const uint32_t total = (uint32_t)per_sm * (uint32_t)ctx->sms;
  const uint32_t taken = (ctx->d.n_engine_ctas + ctx->d.n_service_ctas) * displaced;
  return total > taken + 1 ? total - taken : 1;
}

__global__ void fill_store_kernel(uint8_t* base, uint64_t seed, uint32_t dev, uint64_t first, uint64_t nblk, int kind) {
  // page_word(seed, dev, blk, k) = splitmix64(seed ^ dev<<56 ^ blk<<9 ^ k)  (oracle/pages.py)
  const uint64_t nwords = nblk * 512;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nwords; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t blk = first + i / 512, k = i % 512;
    uint64_t x = seed ^ ((uint64_t)dev << 56) ^ (blk << 9) ^ k;
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    x ^= x >> 31;
    if (kind == 1) {
      const float lo = (float)((uint32_t)x >> 8) * (1.0f / 8388608.0f) - 1.0f;
      const float hi = (float)((uint32_t)(x >> 32) >> 8) * (1.0f / 8388608.0f) - 1.0f;
      x = (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32);
    }
    reinterpret_cast<uint64_t*>(base)[first * 512 + i] = x;
  }
}

// Embedding rows keyed by (table, global row) rather than by page (oracle/pages.py row_floats):
// u64 word k of row r of table t is splitmix64(seed ^ t<<56 ^ r<<8 ^ k); each 32-bit half h is
// stored as the fp32 (h >> 8) * 2^-23 - 1.  A shard holding rows [row0, row0 + rows) of the table
// gets the same values wherever its pages sit, so any sharding of the tables over ranks pools the
// same numbers.  Page p (from first) holds rows row0 + p*rpp .. ; slots past the shard are zero.
__global__ void fill_rows_kernel(uint8_t* base, uint64_t seed, uint32_t table, uint64_t first, uint64_t row0,
                                 uint64_t rows, uint32_t D) {
  const uint32_t rpp = 4096u / (4u * D), wpr = D / 2;   // rows per page, u64 words per row
  const uint64_t npages = (rows + rpp - 1) / rpp;
  const uint64_t nwords = npages * 512;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nwords; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t pg = i / 512, w = i % 512;
    const uint64_t slot = w / wpr, k = w % wpr;
    const uint64_t rr = pg * rpp + slot;
    uint64_t x = 0;
    if (rr < rows) {
      x = seed ^ ((uint64_t)table << 56) ^ ((row0 + rr) << 8) ^ k;
      x += 0x9E3779B97F4A7C15ull;
      x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
      x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
      x ^= x >> 31;
      const float lo = (float)((uint32_t)x >> 8) * (1.0f / 8388608.0f) - 1.0f;
      const float hi = (float)((uint32_t)(x >> 32) >> 8) * (1.0f / 8388608.0f) - 1.0f;
      x = (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32);
    }
    AGILE_FILL_STORE(reinterpret_cast<unsigned long long*>(base + (first + pg) * 4096) + w, (unsigned long long)x);
  }
}

// Drop every line of device `dev` (between runs: nothing is in flight).  READY lines go INVALID
// with a version bump (readers validating the old identity see the change); a BUSY or pinned line
// would mean a run is still active and is counted instead.
__global__ void invalidate_dev_kernel(u64* tags, u32 nlines, u32 dev, unsigned long long* busy) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < nlines; i += (u64)gridDim.x * blockDim.x) {
    const u64 w = tags[i];
    if (tw_state(w) == ST_INVALID || key_dev(tw_key(w)) != dev) continue;
    if (tw_state(w) == ST_BUSY || tw_pins(w)) { atomicAdd(busy, 1ull); continue; }
    tags[i] = tw_make(ST_INVALID, 0, tw_ver(w) + 1, false, 0);
  }
}

// Co-residency probe for the split launch.  A one-CTA primary executes launch_dependents and
// then waits (bounded) for a PDL-launched dependent to set a flag: if the dependent never starts
// while the primary runs — a kernel-serialising tool (ncu, compute-sanitizer) or a driver that
// does not overlap programmatic dependents — the context uses the fused single-grid launch, whose
// roles are taken by arrival order and so never wait on a CTA that is not resident.
__global__ void coresidency_primary(u32* w, u64 timeout_ns) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x != 0) return;
  const u64 t0 = gtimer();
  while (ld_acquire(&w[0]) == 0u) {
    if (gtimer() - t0 > timeout_ns) { st_relaxed(&w[1], 2u); return; }
    __nanosleep(1000);
  }
  st_relaxed(&w[1], 1u);
}
__global__ void coresidency_dependent(u32* w) {
  if (threadIdx.x == 0) st_release(&w[0], 1u);
}

// 1: the dependent ran beside the primary (split launch is safe), 0: it did not, <0: CUDA error
int probe_coresidency(agile_ctx* ctx) {
  u32* w = nullptr;
  // load both kernels first: lazily loading the dependent's module while the primary spins waits
  // for the device to drain, i.e. for the primary's timeout (the probe would always say "fused")
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, coresidency_primary));
  CK(cudaFuncGetAttributes(&fa, coresidency_dependent));
  CK(cudaMalloc(&w, 8));
  CK(cudaMemset(w, 0, 8));
  CK(cudaStreamSynchronize(ctx->stream));
  coresidency_primary<<<1, 32, 0, ctx->stream>>>(w, 200ull * 1000 * 1000);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(32);
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, coresidency_dependent, w);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  u32 h[2] = {0, 0};
  if (e == cudaSuccess) e = cudaMemcpy(h, w, 8, cudaMemcpyDeviceToHost);
  cudaFree(w);
  if (e != cudaSuccess) return fail(ctx, AGILE_E_CUDA, std::string("co-residency probe: ") + cudaGetErrorString(e));
  return h[1] == 1u ? 1 : 0;
}

}  // namespace

extern "C" {

const char* agile_last_error(agile_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int agile_create(const char* config_text, int cuda_device, agile_ctx** out) {
  if (!out) return AGILE_E_ARG;
  *out = nullptr;
  agile_ctx* ctx = new agile_ctx();
  ctx->device = cuda_device;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    ctx->err = "no CUDA device visible: the B200 path has no CPU fallback";
    *out = ctx;
    return AGILE_E_CUDA;
  }
  CK(cudaSetDevice(cuda_device));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cuda_device));
  ctx->sms = sms;
  Cfg cfg;
  cfg.kv = parse_kv(config_text);
  DevCtx& d = ctx->d;
  d.num_devices = (uint32_t)cfg.u("num_devices", 1);
  const uint64_t block = cfg.u("device.block_size", 4096);
  const uint64_t nblocks = cfg.u("device.num_blocks", 1 << 16);
  d.pairs_per_device = (uint32_t)cfg.u("queues.pairs_per_device", 128);
  d.sq_depth = (uint32_t)cfg.u("queues.sq_depth", 256);
  d.cq_depth = (uint32_t)cfg.u("queues.cq_depth", 256);
  uint64_t lines = cfg.u("cache.lines", 512);
  const uint64_t cbytes = cfg.u("cache.bytes", 0);
  if (cbytes) lines = std::max<uint64_t>(1, cbytes / block);   // config.py:64-67
  uint64_t ways = cfg.u("cache.ways", 32);
  if (ways == 0 || ways > lines) ways = lines;   // 0 = fully associative (reference-exact clock)
  const std::string policy = cfg.s("cache.policy", "clock");
  const std::string busy = cfg.s("cache.busy_choice", "wait");
  const std::string engine_copy = cfg.s("engine.copy", "registers");
  d.service_warps = (uint32_t)std::max<uint64_t>(1, cfg.u("service.warps", 4));
  d.poll_ns = (uint32_t)cfg.u("service.poll_ns", 400);
  d.idle_max_ns = (uint32_t)std::max<uint64_t>(d.poll_ns, cfg.u("service.idle_max_ns", 3200));
  d.engine_warps = (uint32_t)std::max<uint64_t>(1, cfg.u("engine.warps", 16));
  const std::string emu = cfg.s("device.emulation", "model");
  const std::string jitter = cfg.s("device.jitter", "none");
  ctx->seed = cfg.u("seed", 0, true);
  if (!cfg.bad.empty()) return fail(ctx, AGILE_E_CONFIG, "bad numeric value for " + cfg.bad), *out = ctx, AGILE_E_CONFIG;
  *out = ctx;
  if (block != kBlockBytes) return fail(ctx, AGILE_E_CONFIG, "device.block_size must be 4096 on the B200 path");
  if (d.num_devices < 1 || d.num_devices > (uint32_t)kMaxDevices) return fail(ctx, AGILE_E_CONFIG, "num_devices out of range [1,16]");
  if (!pow2(d.sq_depth) || d.sq_depth < 2 || d.sq_depth > 65536 || !pow2(d.cq_depth) || d.cq_depth < 2 || d.cq_depth > 65536)
    return fail(ctx, AGILE_E_CONFIG, "depth must be a power of two in [2, 65536]");   // nvme_queue.py:100-103
  if (d.pairs_per_device < 1) return fail(ctx, AGILE_E_CONFIG, "queues.pairs_per_device must be >= 1");
  if ((uint64_t)d.num_devices * d.pairs_per_device > 65535) return fail(ctx, AGILE_E_CONFIG, "too many queue pairs");
  if (lines % ways) return fail(ctx, AGILE_E_CONFIG, "cache.lines must be a multiple of cache.ways");
  if (lines >= (1ull << 32) - 1) return fail(ctx, AGILE_E_CONFIG, "cache too large");
  if (policy != "clock" && policy != "modulo") return fail(ctx, AGILE_E_CONFIG, "unknown cache policy '" + policy + "'");
  if (busy != "wait" && busy != "find_another") return fail(ctx, AGILE_E_CONFIG, "cache.busy_choice must be wait|find_another");
  if (engine_copy != "registers" && engine_copy != "bulk") return fail(ctx, AGILE_E_CONFIG, "engine.copy must be registers|bulk");
  const bool st_on = cfg.b("share_table.enabled", false);
  const uint64_t st_buckets = cfg.u("share_table.buckets", 256);
  if (st_on && (st_buckets < 2 || !pow2(st_buckets) || st_buckets > (1ull << 24)))
    return fail(ctx, AGILE_E_CONFIG, "share_table.buckets must be a power of two >= 2");   // share_table.py:57-58
  if (cfg.u("device.parallelism", 16) > 32 * kMaxChanPerLane) return fail(ctx, AGILE_E_CONFIG, "device.parallelism must be <= 256");
  if (emu != "model" && emu != "link") return fail(ctx, AGILE_E_CONFIG, "device.emulation must be model|link");
  if (jitter != "none" && jitter != "uniform" && jitter != "exponential") return fail(ctx, AGILE_E_CONFIG, "unknown jitter kind");
  d.num_qp = d.num_devices * d.pairs_per_device;
  // each service warp serves at most 128 CQs (kMaxCqPerLane x 32 lanes)
  d.service_warps = std::max<uint32_t>(d.service_warps, (d.num_qp + 32 * kMaxCqPerLane - 1) / (32 * kMaxCqPerLane));
  d.cq_window = std::min<uint32_t>(32, d.cq_depth);
  d.num_lines = (uint32_t)lines;
  d.ways = (uint32_t)ways;
  d.num_sets = (uint32_t)(lines / ways);
  d.sets_pow2 = pow2(d.num_sets) ? 1u : 0u;
  d.n_engine_ctas = (d.engine_warps + kCtaWarps - 1) / kCtaWarps;
  d.n_service_ctas = (d.service_warps + kCtaWarps - 1) / kCtaWarps;
  ctx->side_engine_warps = (uint32_t)cfg.u("engine.side_warps", 0);
  ctx->side_service_warps = (uint32_t)cfg.u("service.side_warps", 0);
  if (ctx->side_service_warps)
    ctx->side_service_warps = std::max<uint32_t>(ctx->side_service_warps, (d.num_qp + 32 * kMaxCqPerLane - 1) / (32 * kMaxCqPerLane));
  d.trace = 0;
  const uint64_t budget = cfg.u("livelock_budget", 5000000);
  d.watchdog_ns = std::max<uint64_t>(budget, 1000000) * 4000ull;   // events -> ~ns budget (>= 4 s)
  if (d.watchdog_ns > 60ull * 1000000000ull) d.watchdog_ns = 60ull * 1000000000ull;
  d.user_start_ns = d.watchdog_ns;
  d.policy = policy == "modulo" ? POL_MODULO : POL_CLOCK;   // system.py:23-31 _make_policy
  ctx->bulk_engine = engine_copy == "bulk";
  d.find_another = busy == "find_another" ? 1u : 0u;
  d.solo_ok = 0;
  if (const char* so = getenv("AGILE_SOLO_USERS")) {
    // profiling mode: a split launch whose user grid cannot start beside the infra grid (ncu
    // kernel replay) lets the infra grid leave after 100 ms and runs the user grid alone — an
    // all-hit replay then profiles the production user kernel with its own register budget
    if (so[0] == '1') { d.solo_ok = 1; d.user_start_ns = 100ull * 1000 * 1000; }
  }
  Model& m = d.model;
  m.link_mode = emu == "link" ? 1u : 0u;
  m.parallelism = (uint32_t)std::max<uint64_t>(1, cfg.u("device.parallelism", 16));
  m.read_ns = cfg.u("device.read_latency_ns", 17712);
  m.write_ns = cfg.u("device.write_latency_ns", 29789);
  m.fetch_ns = cfg.u("timing.fetch_ns", 300);
  m.jitter = jitter == "none" ? 0u : (jitter == "uniform" ? 1u : 2u);
  m.jitter_ns = cfg.u("device.jitter_ns", 0);
  const double rate = cfg.f("device.per_channel_rate", 0.0);
  m.occupancy_ns = rate > 0 ? (uint64_t)std::max(1.0, std::floor(1e9 / rate)) : 0;   // ssd_model.py:55-58
  m.seed = ctx->seed;
  int rc;
  if ((rc = dalloc(ctx, &d.tags, lines))) return rc;
  if ((rc = dalloc(ctx, &d.sig, lines))) return rc;
  if ((rc = dalloc(ctx, &d.wl, lines))) return rc;
  if ((rc = dalloc(ctx, &d.set_lock, d.num_sets))) return rc;
  if ((rc = dalloc(ctx, &d.hand, d.num_sets))) return rc;
  d.st_buckets = st_on ? (uint32_t)st_buckets : 0u;
  // debug_locks (lock_chain.py DeadlockDetector): holder word per lock, wait word per user thread
  d.dbg_locks = cfg.b("debug_locks", true) ? 1u : 0u;
  if (d.dbg_locks) {
    d.dbg_threads = (uint32_t)ctx->sms * 2048u + 65536u;
    if ((rc = dalloc(ctx, &d.lk_holder, (size_t)d.num_sets + (size_t)d.num_devices * d.pairs_per_device + d.st_buckets)))
      return rc;
    if ((rc = dalloc(ctx, &d.lk_wait, d.dbg_threads))) return rc;
  }
  if (st_on) {
    if ((rc = dalloc(ctx, &d.st, st_buckets))) return rc;
    if ((rc = dalloc(ctx, &d.st_lock, st_buckets))) return rc;
  }
  if ((rc = dalloc(ctx, &d.lines, lines * kBlockBytes))) return rc;
  const size_t nsq = (size_t)d.num_qp * d.sq_depth;
  if ((rc = dalloc(ctx, &d.sqe, nsq * 4))) return rc;
  if ((rc = dalloc(ctx, &d.sq_state, nsq))) return rc;
  if ((rc = dalloc(ctx, &d.sq_done_v, nsq))) return rc;
  if ((rc = dalloc(ctx, &d.sqw, d.num_qp))) return rc;
  if ((rc = dalloc(ctx, &d.cmd, nsq))) return rc;
  if ((rc = dalloc(ctx, &d.cqe, (size_t)d.num_qp * d.cq_depth))) return rc;
  if ((rc = dalloc(ctx, &d.cqw, d.num_qp))) return rc;
  if ((rc = dalloc(ctx, &d.chan_free, (size_t)d.num_devices * m.parallelism))) return rc;
  if ((rc = dalloc(ctx, &d.chan_turn, (size_t)d.num_devices * m.parallelism))) return rc;
  if ((rc = dalloc(ctx, &d.dev_lock, d.num_devices))) return rc;
  if ((rc = dalloc(ctx, &d.dev_seq, d.num_devices))) return rc;
  if ((rc = dalloc(ctx, &d.run, 1))) return rc;
  if ((rc = dalloc(ctx, &d.pw, 1))) return rc;
  if ((rc = dalloc(ctx, &d.stats, S_NUM))) return rc;
  if ((rc = dalloc(ctx, &d.log_count, 1))) return rc;
  d.log = nullptr;
  d.log_cap = 0;
  // attach zeroed stores of the configured size for every device (callers may re-attach)
  for (uint32_t dv = 0; dv < d.num_devices; ++dv) {
    if ((rc = agile_store_attach(ctx, (int)dv, nullptr, nblocks, nullptr))) return rc;
  }
  CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  // launch mode: AGILE_LAUNCH=split|fused forces it; otherwise split when a PDL dependent is seen
  // running beside its primary, fused when not (kernel-serialising tools)
  const char* lm = getenv("AGILE_LAUNCH");
  if (lm && std::string(lm) == "fused") {
    ctx->fused = true;
  } else if (lm && std::string(lm) == "split") {
    ctx->fused = false;
  } else {
    const int co = probe_coresidency(ctx);
    if (co < 0) return co;
    ctx->fused = co == 0;
  }
  return 0;
}

int agile_destroy(agile_ctx* ctx) {
  if (!ctx) return 0;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  for (void* p : ctx->dev_allocs) cudaFree(p);
  for (int i = 0; i < kMaxDevices; ++i) {
    if (!ctx->host_store[i]) continue;
    if (ctx->store_owned[i]) cudaFreeHost(ctx->host_store[i]);
    else cudaHostUnregister(ctx->host_store[i]);
  }
  if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
  if (ctx->d_stage) cudaFree(ctx->d_stage);
  for (auto& h : ctx->hs) {
    if (h.st) cudaStreamSynchronize(h.st);
    if (h.d) cudaFree(h.d);
    if (h.h_cnt) cudaFreeHost(h.h_cnt);
    if (h.ran) cudaEventDestroy(h.ran);
    if (h.st) cudaStreamDestroy(h.st);
  }
  if (ctx->d.log) cudaFree(ctx->d.log);
  if (ctx->nodes) cudaFree(ctx->nodes);
  for (auto& kv : ctx->scratch) cudaFree(kv.second.first);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return 0;
}

int agile_geometry(agile_ctx* ctx, uint64_t* out, int n) {
  if (!ctx || !out) return AGILE_E_ARG;
  const DevCtx& d = ctx->d;
  const uint64_t g[11] = {d.num_devices, d.pairs_per_device, d.sq_depth, d.cq_depth, d.num_lines,
                          d.ways, d.num_sets, d.engine_warps, d.service_warps, d.n_engine_ctas + d.n_service_ctas,
                          ctx->fused ? 1ull : 0ull};
  for (int i = 0; i < n && i < 11; ++i) out[i] = g[i];
  return 0;
}

int agile_store_attach(agile_ctx* ctx, int dev, void* host_ptr, uint64_t num_blocks, const char* image_path) {
  if (!ctx || dev < 0 || dev >= (int)ctx->d.num_devices || num_blocks == 0) return fail(ctx, AGILE_E_ARG, "bad store args");
  CK(cudaSetDevice(ctx->device));
  if (num_blocks > BLK_MASK) return fail(ctx, AGILE_E_ARG, "num_blocks exceeds the 36-bit block space");
  // drop the previous store
  if (ctx->host_store[dev]) {
    CK(cudaDeviceSynchronize());
    if (ctx->store_owned[dev]) cudaFreeHost(ctx->host_store[dev]);
    else cudaHostUnregister(ctx->host_store[dev]);
    ctx->host_store[dev] = nullptr;
  }
  const size_t bytes = (size_t)num_blocks * kBlockBytes;
  void* h = host_ptr;
  if (h) {
    CK(cudaHostRegister(h, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
    ctx->store_owned[dev] = false;
  } else {
    CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    ctx->store_owned[dev] = true;
  }
  void* dptr = nullptr;
  CK(cudaHostGetDevicePointer(&dptr, h, 0));
  ctx->host_store[dev] = h;
  ctx->store_blocks[dev] = num_blocks;
  ctx->d.store[dev] = reinterpret_cast<const uint8_t*>(dptr);
  ctx->d.store_w[dev] = reinterpret_cast<uint8_t*>(dptr);
  ctx->d.store_blocks[dev] = num_blocks;
  if (!host_ptr) {
    // zero-default store (BlockStore: unwritten blocks read back as zeros); written by the GPU
    // through the mapping at link speed
    CK(cudaMemset(dptr, 0, bytes));
    CK(cudaDeviceSynchronize());
  }
  if (image_path && image_path[0]) {
    FILE* f = fopen(image_path, "rb");
    if (!f) return fail(ctx, AGILE_E_ARG, std::string("cannot open image ") + image_path);
    const size_t got = fread(h, 1, bytes, f);
    fclose(f);
    if (got < bytes) memset(reinterpret_cast<uint8_t*>(h) + got, 0, bytes - got);   // short tail zero-padded
  }
  return 0;
}

int agile_store_load_image(agile_ctx* ctx, int dev, const char* path) {
  if (!ctx || dev < 0 || dev >= (int)ctx->d.num_devices || !path) return fail(ctx, AGILE_E_ARG, "bad load_image args");
  CK(cudaSetDevice(ctx->device));
  CK(cudaDeviceSynchronize());
  FILE* f = fopen(path, "rb");
  if (!f) return fail(ctx, AGILE_E_ARG, std::string("cannot open image ") + path);
  // BlockStore.load_image (ssd_model.py:84-95): blocks present in the file are overwritten (a
  // short last block zero-padded), the rest of the store keeps its contents
  uint8_t* h = reinterpret_cast<uint8_t*>(ctx->host_store[dev]);
  const uint64_t nb = ctx->store_blocks[dev];
  uint64_t blk = 0;
  while (blk < nb) {
    const size_t got = fread(h + blk * kBlockBytes, 1, kBlockBytes, f);
    if (got == 0) break;
    if (got < kBlockBytes) memset(h + blk * kBlockBytes + got, 0, kBlockBytes - got);
    ++blk;
  }
  fclose(f);
  // the HBM cache must not keep serving the device's previous bytes
  unsigned long long* busy = nullptr;
  CK(cudaMalloc(&busy, 8));
  CK(cudaMemset(busy, 0, 8));
  invalidate_dev_kernel<<<ctx->sms * 4, 256>>>(ctx->d.tags, ctx->d.num_lines, (u32)dev, busy);
  unsigned long long nbusy = 0;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(&nbusy, busy, 8, cudaMemcpyDeviceToHost);
  cudaFree(busy);
  if (e != cudaSuccess) return fail(ctx, AGILE_E_CUDA, std::string("load_image invalidate: ") + cudaGetErrorString(e));
  if (nbusy) return fail(ctx, AGILE_E_ILLEGAL, "load_image while I/O of the device is in flight");
  return 0;
}

int agile_store_ptr(agile_ctx* ctx, int dev, void** host_ptr, uint64_t* num_blocks) {
  if (!ctx || dev < 0 || dev >= (int)ctx->d.num_devices) return AGILE_E_ARG;
  if (host_ptr) *host_ptr = ctx->host_store[dev];
  if (num_blocks) *num_blocks = ctx->store_blocks[dev];
  return 0;
}

int agile_store_fill(agile_ctx* ctx, int dev, uint64_t seed, uint64_t first_blk, uint64_t nblk, int kind) {
  if (!ctx || dev < 0 || dev >= (int)ctx->d.num_devices) return AGILE_E_ARG;
  if (first_blk + nblk > ctx->store_blocks[dev]) return fail(ctx, AGILE_E_OUT_OF_RANGE, "fill beyond store");
  CK(cudaSetDevice(ctx->device));
  fill_store_kernel<<<ctx->sms * 8, 256>>>(ctx->d.store_w[dev], seed, (uint32_t)dev, first_blk, nblk, kind);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return 0;
}

int agile_store_fill_rows(agile_ctx* ctx, int dev, uint64_t seed, uint64_t first_blk, uint32_t table, uint64_t row0,
                          uint64_t rows, uint32_t D) {
  if (!ctx || dev < 0 || dev >= (int)ctx->d.num_devices) return AGILE_E_ARG;
  if (D == 0 || D > 128 || D % 4 || (1024u % D) != 0 || table > 255 || row0 + rows >= (1ull << 48))
    return fail(ctx, AGILE_E_ARG, "bad fill_rows geometry");
  const uint64_t rpp = 1024 / D, npages = (rows + rpp - 1) / rpp;
  if (first_blk + npages > ctx->store_blocks[dev]) return fail(ctx, AGILE_E_OUT_OF_RANGE, "fill beyond store");
  if (!npages) return 0;
  CK(cudaSetDevice(ctx->device));
  fill_rows_kernel<<<ctx->sms * 8, 256>>>(ctx->d.store_w[dev], seed, table, first_blk, row0, rows, D);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return 0;
}

int agile_store_save_image(agile_ctx* ctx, int dev, const char* path) {
  if (!ctx || dev < 0 || dev >= (int)ctx->d.num_devices || !path) return AGILE_E_ARG;
  CK(cudaDeviceSynchronize());
  const uint8_t* h = reinterpret_cast<const uint8_t*>(ctx->host_store[dev]);
  // top = last block holding a non-zero byte (+1): the dense analogue of save_image's
  // max(written)+1 (ssd_model.py:97-101)
  uint64_t top = ctx->store_blocks[dev];
  while (top > 0) {
    const uint64_t* w = reinterpret_cast<const uint64_t*>(h + (top - 1) * kBlockBytes);
    bool nz = false;
    for (int k = 0; k < 512 && !nz; ++k) nz = w[k] != 0;
    if (nz) break;
    --top;
  }
  FILE* f = fopen(path, "wb");
  if (!f) return fail(ctx, AGILE_E_ARG, std::string("cannot open ") + path);
  fwrite(h, 1, top * kBlockBytes, f);
  fclose(f);
  return 0;
}

int agile_reset(agile_ctx* ctx, int flags) {
  if (!ctx) return AGILE_E_ARG;
  CK(cudaSetDevice(ctx->device));
  CK(cudaDeviceSynchronize());
  DevCtx& d = ctx->d;
  if (flags & 1) {
    CK(cudaMemset(d.tags, 0, (size_t)d.num_lines * 8));
    CK(cudaMemset(d.sig, 0, (size_t)d.num_lines * 2));
    CK(cudaMemset(d.wl, 0, (size_t)d.num_lines * 8));
    CK(cudaMemset(d.hand, 0, (size_t)d.num_sets * 4));
    CK(cudaMemset(d.set_lock, 0, (size_t)d.num_sets * 4));
    if (d.st_buckets) {
      CK(cudaMemset(d.st, 0, (size_t)d.st_buckets * sizeof(ShareEntry)));
      CK(cudaMemset(d.st_lock, 0, (size_t)d.st_buckets * 4));
    }
  }
  if (flags & 2) {
    const size_t nsq = (size_t)d.num_qp * d.sq_depth;
    CK(cudaMemset(d.sqe, 0, nsq * 64));
    CK(cudaMemset(d.sq_state, 0, nsq * 4));
    CK(cudaMemset(d.sq_done_v, 0, nsq * 8));
    CK(cudaMemset(d.sqw, 0, (size_t)d.num_qp * sizeof(SqWords)));
    CK(cudaMemset(d.cmd, 0, nsq * sizeof(CmdCtx)));
    CK(cudaMemset(d.cqe, 0, (size_t)d.num_qp * d.cq_depth * 16));
    CK(cudaMemset(d.cqw, 0, (size_t)d.num_qp * sizeof(CqWords)));
    CK(cudaMemset(d.chan_free, 0, (size_t)d.num_devices * d.model.parallelism * 8));
    CK(cudaMemset(d.chan_turn, 0, (size_t)d.num_devices * d.model.parallelism * 8));
    CK(cudaMemset(d.dev_seq, 0, (size_t)d.num_devices * 8));
    CK(cudaMemset(d.pw, 0, sizeof(PersistWords)));
  }
  if (flags & 4) {
    CK(cudaMemset(d.stats, 0, S_NUM * 8));
    CK(cudaMemset(d.log_count, 0, 8));
  }
  CK(cudaDeviceSynchronize());
  return 0;
}

int agile_stats(agile_ctx* ctx, uint64_t* out, int n) {
  if (!ctx || !out) return AGILE_E_ARG;
  CK(cudaSetDevice(ctx->device));
  CK(cudaDeviceSynchronize());
  uint64_t s[S_NUM];
  CK(cudaMemcpy(s, ctx->d.stats, sizeof s, cudaMemcpyDeviceToHost));
  for (int i = 0; i < n && i < S_NUM; ++i) out[i] = s[i];
  return 0;
}

int agile_trace_enable(agile_ctx* ctx, uint64_t capacity) {
  if (!ctx) return AGILE_E_ARG;
  CK(cudaSetDevice(ctx->device));
  if (ctx->d.log) { cudaFree(ctx->d.log); ctx->d.log = nullptr; }
  ctx->d.log_cap = 0;
  ctx->d.trace = 0;
  if (capacity) {
    void* p = nullptr;
    CK(cudaMalloc(&p, capacity * 64));
    ctx->d.log = reinterpret_cast<uint4*>(p);
    ctx->d.log_cap = capacity;
    ctx->d.trace = 1;
  }
  CK(cudaMemset(ctx->d.log_count, 0, 8));
  return 0;
}

int agile_event_log(agile_ctx* ctx, void* out, uint64_t cap, uint64_t* n) {
  if (!ctx || !n) return AGILE_E_ARG;
  CK(cudaSetDevice(ctx->device));
  CK(cudaDeviceSynchronize());
  uint64_t cnt = 0;
  CK(cudaMemcpy(&cnt, ctx->d.log_count, 8, cudaMemcpyDeviceToHost));
  *n = cnt;
  if (cnt > ctx->d.log_cap) return fail(ctx, AGILE_E_ARG, "event log overflow: raise the trace capacity");
  if (out && cap) CK(cudaMemcpy(out, ctx->d.log, std::min(cnt, cap) * 64, cudaMemcpyDeviceToHost));
  return 0;
}

int agile_sync(agile_ctx* ctx, void* stream) {
  if (!ctx) return AGILE_E_ARG;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream)));
  return device_error(ctx);
}

int agile_run_seq(agile_ctx* ctx, const uint32_t* dev, const uint64_t* blk, int64_t n, int8_t* outcome,
                  uint64_t* victim, void* pages_out) {
  if (!ctx || n < 0 || (n && (!dev || !blk || !outcome || !victim))) return fail(ctx, AGILE_E_ARG, "bad seq args");
  CK(cudaSetDevice(ctx->device));
  for (int64_t i = 0; i < n; ++i) {
    if (dev[i] >= ctx->d.num_devices) return fail(ctx, AGILE_E_OUT_OF_RANGE, "no such device");
    if (blk[i] >= ctx->store_blocks[dev[i]]) return fail(ctx, AGILE_E_OUT_OF_RANGE, "block out of range");
  }
  if (n == 0) return 0;
  DevTmp tmp;
  uint32_t* d_dev; uint64_t* d_blk; int8_t* d_out; uint64_t* d_vic; uint4* d_pages = nullptr; uint4* d_scr;
  CK(tmp.alloc(&d_dev, n * 4));
  CK(tmp.alloc(&d_blk, n * 8));
  CK(tmp.alloc(&d_out, n));
  CK(tmp.alloc(&d_vic, n * 8));
  CK(tmp.alloc(&d_scr, kBlockBytes));
  if (pages_out) CK(tmp.alloc(&d_pages, (size_t)n * kBlockBytes));
  CK(cudaMemcpy(d_dev, dev, n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_blk, blk, n * 8, cudaMemcpyHostToDevice));
  SeqWork w;
  w.dev = d_dev; w.blk = reinterpret_cast<const u64*>(d_blk); w.n = n;
  w.outcome = reinterpret_cast<signed char*>(d_out); w.victim = reinterpret_cast<u64*>(d_vic);
  w.pages = d_pages; w.scratch = d_scr;
  w.nodes = get_nodes(ctx, 1);
  if (!w.nodes) return fail(ctx, AGILE_E_CUDA, "node allocation failed");
  int rc = launch(ctx, w, 1, ctx->stream);
  if (!rc) rc = agile_sync(ctx, ctx->stream);
  if (!rc) {
    CK(cudaMemcpy(outcome, d_out, n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(victim, d_vic, n * 8, cudaMemcpyDeviceToHost));
    if (pages_out) CK(cudaMemcpy(pages_out, d_pages, (size_t)n * kBlockBytes, cudaMemcpyDeviceToHost));
  }
  return rc;
}

int agile_evict_blocks(agile_ctx* ctx, const uint32_t* dev, const uint64_t* blk, int64_t n, int8_t* outcome) {
  if (!ctx || n < 0 || (n && (!dev || !blk || !outcome))) return fail(ctx, AGILE_E_ARG, "bad evict args");
  CK(cudaSetDevice(ctx->device));
  for (int64_t i = 0; i < n; ++i)
    if (dev[i] >= ctx->d.num_devices || blk[i] >= ctx->store_blocks[dev[i]])
      return fail(ctx, AGILE_E_OUT_OF_RANGE, "block out of range");
  if (n == 0) return 0;
  DevTmp tmp;
  uint32_t* d_dev; uint64_t* d_blk; int8_t* d_out;
  CK(tmp.alloc(&d_dev, n * 4));
  CK(tmp.alloc(&d_blk, n * 8));
  CK(tmp.alloc(&d_out, n));
  CK(cudaMemcpy(d_dev, dev, n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_blk, blk, n * 8, cudaMemcpyHostToDevice));
  EvictWork w;
  w.dev = d_dev; w.blk = reinterpret_cast<const u64*>(d_blk); w.n = n;
  w.outcome = reinterpret_cast<signed char*>(d_out);
  int rc = launch(ctx, w, 1, ctx->stream);
  if (!rc) rc = agile_sync(ctx, ctx->stream);
  if (!rc) CK(cudaMemcpy(outcome, d_out, n, cudaMemcpyDeviceToHost));
  return rc;
}

int agile_user_run_begin(agile_ctx* ctx, void* stream, uint32_t n_user_ctas, uint64_t n_bufs, void* devctx_out,
                         uint64_t devctx_size, void* launch_out, uint64_t launch_size, void** nodes_out) {
  if (!ctx || !devctx_out || !launch_out || !n_user_ctas) return fail(ctx, AGILE_E_ARG, "bad user_run_begin args");
  if (devctx_size != sizeof(DevCtx) || launch_size != sizeof(Launch))
    return fail(ctx, AGILE_E_ARG, "DevCtx / Launch size mismatch: rebuild against include/agile_device.cuh");
  if (ctx->fused)
    return fail(ctx, AGILE_E_ARG, "third-party user kernels need the split launch (a kernel-serialising tool is attached)");
  CK(cudaSetDevice(ctx->device));
  WaitNode* nodes = get_nodes(ctx, std::max<uint64_t>(1, n_bufs), reinterpret_cast<cudaStream_t>(stream));
  if (!nodes) return fail(ctx, AGILE_E_CUDA, "node allocation failed");
  if (nodes_out) *nodes_out = nodes;
  cudaFuncAttributes a{};
  cudaFuncGetAttributes(&a, agile_infra_kernel<false>);   // loaded before the infra grid spins
  cudaFuncGetAttributes(&a, agile_infra_kernel<true>);
  DevCtx dc;
  Launch L;
  int rc = launch_infra(ctx, n_user_ctas, reinterpret_cast<cudaStream_t>(stream), false, dc, L);
  if (rc) return rc;
  std::memcpy(devctx_out, &dc, sizeof(DevCtx));
  std::memcpy(launch_out, &L, sizeof(Launch));
  return 0;
}

int agile_user_run_end(agile_ctx* ctx, void* stream) { return agile_sync(ctx, stream); }

int agile_set_engine_copy(agile_ctx* ctx, int bulk) {
  if (!ctx) return AGILE_E_ARG;
  ctx->bulk_engine = bulk != 0;
  return 0;
}

int agile_set_launch_mode(agile_ctx* ctx, int mode) {
  if (!ctx || mode < 0 || mode > 3)
    return fail(ctx, AGILE_E_ARG, "launch mode must be 0 (split), 1 (fused), 2 (split, solo users) or 3 (users only)");
  ctx->fused = mode == 1;
  ctx->users_only = mode == 3;
  ctx->d.solo_ok = mode >= 2 ? 1u : 0u;
  ctx->d.user_start_ns = mode == 2 ? 100ull * 1000 * 1000 : ctx->d.watchdog_ns;
  return 0;
}

int agile_run_coherence(agile_ctx* ctx, const uint8_t* op, const uint32_t* blk, const uint32_t* think, uint32_t tasks,
                        uint32_t ops, uint64_t* seen, uint64_t* flushed) {
  if (!ctx || !tasks || tasks > kCtaWarps || !ops || !op || !blk || !think || !seen)
    return fail(ctx, AGILE_E_ARG, "bad coherence args (1..8 tasks)");
  CK(cudaSetDevice(ctx->device));
  const size_t n = (size_t)tasks * ops;
  for (size_t i = 0; i < n; ++i)
    if (blk[i] >= ctx->store_blocks[0]) return fail(ctx, AGILE_E_OUT_OF_RANGE, "block out of range");
  DevTmp tmp;
  uint8_t* d_op; uint32_t* d_blk; uint32_t* d_think; uint64_t* d_seen; uint64_t* d_fl; uint4* d_w; uint4* d_r; uint4* d_s;
  CK(tmp.alloc(&d_op, n));
  CK(tmp.alloc(&d_blk, n * 4));
  CK(tmp.alloc(&d_think, n * 4));
  CK(tmp.alloc(&d_seen, n * 8));
  CK(tmp.alloc(&d_fl, 8));
  CK(tmp.alloc(&d_w, (size_t)tasks * kBlockBytes));
  CK(tmp.alloc(&d_r, n * kBlockBytes));
  CK(tmp.alloc(&d_s, (size_t)tasks * kBlockBytes));
  CK(cudaMemcpy(d_op, op, n, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_blk, blk, n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_think, think, n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(d_seen, 0, n * 8));
  CoherenceWork w;
  w.op = d_op; w.blk = d_blk; w.think = d_think; w.tasks = tasks; w.ops = ops;
  w.wbuf = d_w; w.rbuf = d_r; w.snap = d_s; w.seen = reinterpret_cast<u64*>(d_seen);
  w.flushed = reinterpret_cast<u64*>(d_fl);
  w.nodes = get_nodes(ctx, n + tasks + 32);
  if (!w.nodes) return fail(ctx, AGILE_E_CUDA, "node allocation failed");
  int rc = launch(ctx, w, 1, ctx->stream);
  if (!rc) rc = agile_sync(ctx, ctx->stream);
  if (!rc) CK(cudaMemcpy(seen, d_seen, n * 8, cudaMemcpyDeviceToHost));
  if (!rc && flushed) CK(cudaMemcpy(flushed, d_fl, 8, cudaMemcpyDeviceToHost));
  return rc;
}

int agile_flush(agile_ctx* ctx, uint64_t* flushed) {
  if (!ctx) return AGILE_E_ARG;
  CK(cudaSetDevice(ctx->device));
  DevTmp tmp;
  uint64_t* d_fl;
  CK(tmp.alloc(&d_fl, 8));
  FlushWork w;
  w.nodes = get_nodes(ctx, 32);
  w.flushed = reinterpret_cast<u64*>(d_fl);
  if (!w.nodes) return fail(ctx, AGILE_E_CUDA, "node allocation failed");
  int rc = launch(ctx, w, 1, ctx->stream);
  if (!rc) rc = agile_sync(ctx, ctx->stream);
  if (!rc && flushed) CK(cudaMemcpy(flushed, d_fl, 8, cudaMemcpyDeviceToHost));
  return rc;
}

int agile_share_live(agile_ctx* ctx, uint64_t* live) {
  if (!ctx || !live) return AGILE_E_ARG;
  *live = 0;
  if (!ctx->d.st_buckets) return 0;
  CK(cudaSetDevice(ctx->device));
  std::vector<ShareEntry> e(ctx->d.st_buckets);
  CK(cudaMemcpy(e.data(), ctx->d.st, e.size() * sizeof(ShareEntry), cudaMemcpyDeviceToHost));
  for (const auto& x : e) *live += x.key >= 2 ? 1 : 0;   // share_table.py:198-199 live_entries
  return 0;
}

int agile_lock_cycle_demo(agile_ctx* ctx, uint32_t n, int mode) {
  if (!ctx || n < 1 || n > kCtaWarps || mode < 0 || mode > 1) return fail(ctx, AGILE_E_ARG, "bad lock demo args");
  CK(cudaSetDevice(ctx->device));
  LockCycleWork w;
  w.n = n;
  w.mode = (uint32_t)mode;
  int rc = launch(ctx, w, 1, ctx->stream);
  if (!rc) rc = agile_sync(ctx, ctx->stream);
  return rc;
}

int agile_buffer_busy_demo(agile_ctx* ctx, int write) {
  if (!ctx) return AGILE_E_ARG;
  CK(cudaSetDevice(ctx->device));
  DevTmp tmp;
  uint4* d_buf;
  CK(tmp.alloc(&d_buf, kBlockBytes));
  BusyWork w;
  w.nodes = get_nodes(ctx, 1);
  w.buf = d_buf;
  w.write = write ? 1u : 0u;
  if (!w.nodes) return fail(ctx, AGILE_E_CUDA, "node allocation failed");
  int rc = launch(ctx, w, 1, ctx->stream);
  if (!rc) rc = agile_sync(ctx, ctx->stream);
  return rc;
}

int agile_array_get(agile_ctx* ctx, const uint32_t* dev, const uint64_t* idx, int64_t n, uint32_t elem_size,
                    void* out) {
  if (!ctx || n < 0 || (n && (!dev || !idx || !out))) return fail(ctx, AGILE_E_ARG, "bad array_get args");
  if (elem_size == 0 || kBlockBytes % elem_size) return fail(ctx, AGILE_E_ARG, "element size must divide the block size");
  CK(cudaSetDevice(ctx->device));
  for (int64_t i = 0; i < n; ++i) {   // AgileApi._check_block (gpu_api.py:122-126)
    if (dev[i] >= ctx->d.num_devices) return fail(ctx, AGILE_E_OUT_OF_RANGE, "no such device");
    if (idx[i] > (UINT64_MAX >> 13) || idx[i] * elem_size / kBlockBytes >= ctx->store_blocks[dev[i]])
      return fail(ctx, AGILE_E_OUT_OF_RANGE, "element out of range");
  }
  if (n == 0) return 0;
  DevTmp tmp;
  uint32_t* d_dev; uint64_t* d_idx; uint8_t* d_out;
  CK(tmp.alloc(&d_dev, n * 4));
  CK(tmp.alloc(&d_idx, n * 8));
  CK(tmp.alloc(&d_out, (size_t)n * elem_size));
  CK(cudaMemcpy(d_dev, dev, n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_idx, idx, n * 8, cudaMemcpyHostToDevice));
  ArrayGetWork w;
  w.dev = d_dev; w.idx = reinterpret_cast<const u64*>(d_idx); w.n = (u64)n; w.elem_size = elem_size; w.out = d_out;
  const uint32_t users = (uint32_t)std::min<uint64_t>((n + kCtaThreads - 1) / kCtaThreads, resident_ctas<ArrayGetWork>(ctx));
  int rc = launch(ctx, w, std::max<uint32_t>(1, users), ctx->stream);
  if (!rc) rc = agile_sync(ctx, ctx->stream);
  if (!rc) CK(cudaMemcpy(out, d_out, (size_t)n * elem_size, cudaMemcpyDeviceToHost));
  return rc;
}

int agile_write_blocks(agile_ctx* ctx, const uint32_t* dev, const uint64_t* blk, int64_t n, const void* pages) {
  if (!ctx || n < 0 || (n && (!dev || !blk || !pages))) return fail(ctx, AGILE_E_ARG, "bad write args");
  CK(cudaSetDevice(ctx->device));
  for (int64_t i = 0; i < n; ++i) {
    if (dev[i] >= ctx->d.num_devices) return fail(ctx, AGILE_E_OUT_OF_RANGE, "no such device");
    if (blk[i] >= ctx->store_blocks[dev[i]]) return fail(ctx, AGILE_E_OUT_OF_RANGE, "block out of range");
  }
  if (n == 0) return 0;
  DevTmp tmp;
  uint32_t* d_dev; uint64_t* d_blk; uint4* d_src;
  CK(tmp.alloc(&d_dev, n * 4));
  CK(tmp.alloc(&d_blk, n * 8));
  CK(tmp.alloc(&d_src, (size_t)n * kBlockBytes));
  CK(cudaMemcpy(d_dev, dev, n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_blk, blk, n * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_src, pages, (size_t)n * kBlockBytes, cudaMemcpyHostToDevice));
  WriteWork w;
  w.dev = d_dev; w.blk = reinterpret_cast<const u64*>(d_blk); w.src = d_src; w.n = (u64)n;
  w.nodes = get_nodes(ctx, (size_t)n);
  int rc = w.nodes ? 0 : fail(ctx, AGILE_E_CUDA, "node allocation failed");
  if (!rc) rc = launch(ctx, w, (uint32_t)((n + kCtaThreads - 1) / kCtaThreads), ctx->stream);
  if (!rc) rc = agile_sync(ctx, ctx->stream);
  return rc;
}

int agile_run_reads(agile_ctx* ctx, const uint64_t* keys, uint32_t tasks, uint32_t reads, uint32_t epochs,
                    int async_mode, uint64_t compute_ns, void* bufs, uint64_t* digest, uint64_t* epoch_t,
                    void* stream) {
  if (!ctx || !keys || !bufs || !digest || !epoch_t || !tasks || !reads || !epochs) return fail(ctx, AGILE_E_ARG, "bad reads args");
  if (reads > (uint32_t)ReadsWork::MAXR) return fail(ctx, AGILE_E_ARG, "reads_per_task > 64");
  CK(cudaSetDevice(ctx->device));
  ReadsWork w;
  w.keys = reinterpret_cast<const u64*>(keys);
  w.bufs = reinterpret_cast<uint4*>(bufs);
  w.digest = reinterpret_cast<u64*>(digest);
  w.epoch_t = reinterpret_cast<u64*>(epoch_t);
  w.tasks = tasks; w.reads = reads; w.epochs = epochs; w.async_mode = async_mode ? 1u : 0u;
  w.compute_ns = compute_ns;
  w.nodes = get_nodes(ctx, (size_t)tasks * 2 * reads, reinterpret_cast<cudaStream_t>(stream));
  if (!w.nodes) return fail(ctx, AGILE_E_CUDA, "node allocation failed");
  const uint32_t users = (tasks + kCtaThreads - 1) / kCtaThreads;
  const uint32_t cap = resident_ctas<ReadsWork>(ctx);
  if (users > cap)
    return fail(ctx, AGILE_E_ARG, "tasks exceed co-resident capacity for the epoch barrier");
  return launch(ctx, w, users, reinterpret_cast<cudaStream_t>(stream));
}

int agile_run_loop(agile_ctx* ctx, uint32_t conc, uint64_t warmup_ns, uint64_t measure_ns,
                   uint64_t max_per_task, void* bufs, uint64_t* counters, void* stream) {
  return agile_run_loop_rw(ctx, conc, warmup_ns, measure_ns, max_per_task, bufs, counters, 0, stream);
}

int agile_run_loop_rw(agile_ctx* ctx, uint32_t conc, uint64_t warmup_ns, uint64_t measure_ns,
                      uint64_t max_per_task, void* bufs, uint64_t* counters, int write, void* stream) {
  if (!ctx || !conc || !bufs || !counters) return fail(ctx, AGILE_E_ARG, "bad loop args");
  CK(cudaSetDevice(ctx->device));
  LoopWork w;
  w.write = write ? 1u : 0u;
  w.bufs = reinterpret_cast<uint4*>(bufs);
  w.counters = reinterpret_cast<unsigned long long*>(counters);
  w.conc = conc;
  w.ndev = ctx->d.num_devices;
  uint64_t nb = ctx->store_blocks[0];
  for (uint32_t i = 1; i < ctx->d.num_devices; ++i) nb = std::min<uint64_t>(nb, ctx->store_blocks[i]);
  w.num_blocks = nb;
  w.warmup_ns = warmup_ns;
  w.measure_ns = measure_ns;
  w.max_per_task = max_per_task ? max_per_task : ~0ull;
  w.nodes = get_nodes(ctx, conc, reinterpret_cast<cudaStream_t>(stream));
  if (!w.nodes) return fail(ctx, AGILE_E_CUDA, "node allocation failed");
  const uint32_t users = (conc + kCtaThreads - 1) / kCtaThreads;
  return launch(ctx, w, users, reinterpret_cast<cudaStream_t>(stream));
}

int agile_run_gather(agile_ctx* ctx, const uint64_t* keys, uint32_t tasks, uint32_t epochs, uint32_t gathers,
                     int async_mode, uint64_t compute_ns, uint32_t* values, uint64_t* epoch_t, void* stream) {
  if (!ctx || !keys || !values || !epoch_t || !tasks || !epochs || !gathers) return fail(ctx, AGILE_E_ARG, "bad gather args");
  CK(cudaSetDevice(ctx->device));
  GatherWork w;
  w.keys = reinterpret_cast<const u64*>(keys);
  w.values = values;
  w.epoch_t = reinterpret_cast<u64*>(epoch_t);
  w.tasks = tasks; w.epochs = epochs; w.gathers = gathers; w.async_mode = async_mode ? 1u : 0u;
  w.compute_ns = compute_ns;
  const uint32_t users = (tasks + kCtaThreads - 1) / kCtaThreads;
  const uint32_t cap = resident_ctas<GatherWork>(ctx);
  if (users > cap)
    return fail(ctx, AGILE_E_ARG, "tasks exceed co-resident capacity for the epoch barrier");
  return launch(ctx, w, users, reinterpret_cast<cudaStream_t>(stream));
}

static uint32_t embbag_users(agile_ctx* ctx) { return resident_ctas<EmbBagWork>(ctx); }

// common launch of K5: geometry checks, then one AGILE run (user_ctas != 0: a bounded side run)
static int embbag_launch(agile_ctx* ctx, EmbBagWork& w, const int64_t* idx, const int64_t* offsets, uint8_t* out,
                         uint64_t* counters, uint32_t B, uint32_t T, uint32_t L, uint32_t D, uint32_t pd,
                         uint32_t user_ctas, int prefetch_only, void* stream) {
  if (T == 0) return fail(ctx, AGILE_E_ARG, "no tables");
  if (!offsets && L > 4096) return fail(ctx, AGILE_E_ARG, "pooling factor L must be <= 4096");
  if (D == 0 || D > 128 || D % 4 || (1024u % D) != 0) return fail(ctx, AGILE_E_ARG, "D must divide 1024, be a multiple of 4 and <= 128");
  if ((uint64_t)B * T >= (1ull << 31) || (!offsets && (uint64_t)B * T * L >= (1ull << 40)))
    return fail(ctx, AGILE_E_ARG, "too many bags");
  CK(cudaSetDevice(ctx->device));
  w.idx = reinterpret_cast<const long long*>(idx);
  w.offsets = reinterpret_cast<const long long*>(offsets);
  w.out = out;
  w.lookups_miss = reinterpret_cast<u64*>(counters);
  w.B = B; w.T = T; w.L = offsets ? 0 : L; w.D = D;
  w.t_magic = T > 1 ? ~0ull / T + 1 : 0;
  w.pd = pd;
  uint32_t rpp = kBlockBytes / (D * 4), sh = 0;
  while ((1u << sh) < rpp) ++sh;
  w.rows_per_page_shift = sh;
  w.prefetch_only = prefetch_only ? 1u : 0u;
  const uint32_t full = embbag_users(ctx);
  const uint32_t users = user_ctas ? std::min(user_ctas, full) : full;
  w.nwarps_total = users * kCtaWarps;
  if ((uint64_t)B * T == 0) return 0;
  return launch(ctx, w, users, reinterpret_cast<cudaStream_t>(stream), user_ctas != 0);
}

int agile_embbag_grid(agile_ctx* ctx, uint32_t* user_ctas, uint32_t* infra_ctas) {
  if (!ctx) return AGILE_E_ARG;
  if (user_ctas) *user_ctas = embbag_users(ctx);
  if (infra_ctas) *infra_ctas = ctx->d.n_engine_ctas + ctx->d.n_service_ctas;
  return 0;
}

int agile_embbag(agile_ctx* ctx, const int64_t* idx, const uint64_t* table_key0, const int64_t* table_rows,
                 float* out, uint64_t* counters, uint32_t B, uint32_t T, uint32_t L, uint32_t D,
                 uint32_t out_b_stride, uint32_t out_t_stride, uint32_t prefetch_distance, void* stream) {
  return agile_embbag_ctas(ctx, idx, table_key0, table_rows, out, counters, B, T, L, D, out_b_stride, out_t_stride,
                           prefetch_distance, 0, stream);
}

int agile_embbag_ctas(agile_ctx* ctx, const int64_t* idx, const uint64_t* table_key0, const int64_t* table_rows,
                      float* out, uint64_t* counters, uint32_t B, uint32_t T, uint32_t L, uint32_t D,
                      uint32_t out_b_stride, uint32_t out_t_stride, uint32_t prefetch_distance, uint32_t user_ctas,
                      void* stream) {
  if (!ctx || !idx || !table_key0 || !table_rows || !out || !counters) return fail(ctx, AGILE_E_ARG, "null embbag arg");
  EmbBagWork w{};
  w.table_key0 = reinterpret_cast<const u64*>(table_key0);
  w.table_rows = reinterpret_cast<const long long*>(table_rows);
  w.out_row_bytes = (u64)(out_b_stride ? out_b_stride : T * D) * 4;
  w.out_t_bytes = (out_t_stride ? out_t_stride : D) * 4;
  return embbag_launch(ctx, w, idx, nullptr, reinterpret_cast<uint8_t*>(out), counters, B, T, L, D, prefetch_distance,
                       user_ctas, 0, stream);
}

int agile_embbag_sharded(agile_ctx* ctx, const int64_t* idx, const int64_t* offsets, const agile_table_shard* tables,
                         void* out, uint64_t out_row_bytes, uint64_t* counters, uint32_t B, uint32_t T, uint32_t L,
                         uint32_t D, uint32_t prefetch_distance, uint32_t user_ctas, int mode, void* stream) {
  if (!ctx || !idx || !tables || !counters || (mode == 0 && !out)) return fail(ctx, AGILE_E_ARG, "null embbag arg");
  if (mode != 0 && mode != 1) return fail(ctx, AGILE_E_ARG, "mode must be 0 (pool) or 1 (prefetch only)");
  if (mode == 0 && (out_row_bytes % 16)) return fail(ctx, AGILE_E_ARG, "out_row_bytes must be a multiple of 16");
  EmbBagWork w{};
  w.tabs = reinterpret_cast<const TabDesc*>(tables);
  w.out_row_bytes = out_row_bytes;
  return embbag_launch(ctx, w, idx, offsets, reinterpret_cast<uint8_t*>(out), counters, B, T, L, D,
                       prefetch_distance, user_ctas, mode, stream);
}

int agile_embbag_prefetch(agile_ctx* ctx, const int64_t* idx, const uint64_t* table_key0, const int64_t* table_rows,
                          uint64_t* counters, uint32_t B, uint32_t T, uint32_t L, uint32_t D, uint32_t user_ctas,
                          void* stream) {
  if (!ctx || !idx || !table_key0 || !table_rows || !counters) return fail(ctx, AGILE_E_ARG, "null prefetch arg");
  EmbBagWork w{};
  w.table_key0 = reinterpret_cast<const u64*>(table_key0);
  w.table_rows = reinterpret_cast<const long long*>(table_rows);
  return embbag_launch(ctx, w, idx, nullptr, nullptr, counters, B, T, L, D, 0, user_ctas, 1, stream);
}

// ------------------------------------------------------------------ graph drivers (K6 / K7)
}  // extern "C"

namespace {

template <class T>
T* scratch(agile_ctx* ctx, const char* name, size_t count) {
  auto& e = ctx->scratch[name];
  const size_t bytes = std::max<size_t>(count * sizeof(T), 256);
  if (e.second < bytes) {
    if (e.first) { cudaDeviceSynchronize(); cudaFree(e.first); }
    e.first = nullptr;
    e.second = 0;
    if (cudaMalloc(&e.first, bytes) != cudaSuccess) return nullptr;
    e.second = bytes;
  }
  return reinterpret_cast<T*>(e.first);
}

// deg[i] = out-degree of frontier vertex i (deg[n] = 0), for the exclusive scan into eoff
__global__ void frontier_degree_kernel(const long long* row_ptr, const int* f, uint32_t n, long long* deg,
                                       uint32_t v0) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= n; i += (uint64_t)gridDim.x * blockDim.x)
    deg[i] = i < n ? row_ptr[f[i] - (int)v0 + 1] - row_ptr[f[i] - (int)v0] : 0;
}

__global__ void popc_kernel(const uint32_t* bits, uint32_t nw, uint32_t* cnt) {
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nw; w += (uint64_t)gridDim.x * blockDim.x)
    cnt[w] = __popc(bits[w]);
}

// next frontier in ascending vertex order from the discovery bitmap
__global__ void compact_kernel(const uint32_t* bits, const uint32_t* cnt, const uint32_t* pos, uint32_t nw, int* out,
                               uint32_t* n_out) {
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nw; w += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t b = bits[w];
    uint32_t p = pos[w];
    while (b) {
      const int k = __ffs(b) - 1;
      b &= b - 1;
      out[p++] = (int)(w * 32 + k);
    }
    if (w == nw - 1) *n_out = pos[w] + cnt[w];
  }
}

__global__ void fill_f32_kernel(float* y, uint64_t n, float v) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) y[i] = v;
}

// rows crossing chunk boundaries: the chunk where the row starts walks the following chunks'
// partials in chunk order (deterministic), then writes y
__global__ void spmv_fixup_kernel(const long long* row_ptr, const uint32_t* last_row, const double* part_first,
                                  const double* part_last, uint64_t nch, uint64_t E, float alpha, float beta, float* y) {
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < nch; c += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t r = last_row[c];
    if (r == 0xffffffffu) continue;
    const long long rend = row_ptr[r + 1];
    double s = part_last[c];
    for (uint64_t c2 = c + 1; c2 < nch; ++c2) {
      s += part_first[c2];
      const uint64_t ce = (c2 + 1) * SpmvWork::kChunk;
      const long long e1 = (long long)(ce < E ? ce : E);
      if (rend <= e1) break;
    }
    y[r] = (float)((double)alpha * s + (double)beta);
  }
}

uint32_t grid_for(uint64_t n) { return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148 * 16)); }

}  // namespace

extern "C" {

int agile_bfs(agile_ctx* ctx, const int64_t* row_ptr, uint32_t V, uint32_t source, uint64_t col_key0, int32_t* level,
              uint32_t prefetch_distance, uint64_t* stats, void* stream) {
  if (!ctx || !row_ptr || !level || !V) return fail(ctx, AGILE_E_ARG, "null bfs arg");
  if (source >= V) return fail(ctx, AGILE_E_ARG, "bfs source out of range");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const uint32_t nw = (V + 31) / 32;
  int* fa = scratch<int>(ctx, "bfs.fa", V);
  int* fb = scratch<int>(ctx, "bfs.fb", V);
  long long* deg = scratch<long long>(ctx, "bfs.deg", (size_t)V + 1);
  long long* eoff = scratch<long long>(ctx, "bfs.eoff", (size_t)V + 1);
  uint32_t* visited = scratch<uint32_t>(ctx, "bfs.visited", nw);
  uint32_t* next_bits = scratch<uint32_t>(ctx, "bfs.next", nw);
  uint32_t* wcnt = scratch<uint32_t>(ctx, "bfs.wcnt", nw);
  uint32_t* wpos = scratch<uint32_t>(ctx, "bfs.wpos", nw);
  uint32_t* nnext = scratch<uint32_t>(ctx, "bfs.nnext", 1);
  uint64_t* counters = scratch<uint64_t>(ctx, "bfs.counters", 2);
  if (!fa || !fb || !deg || !eoff || !visited || !next_bits || !wcnt || !wpos || !nnext || !counters)
    return fail(ctx, AGILE_E_CUDA, "bfs scratch allocation failed");
  size_t tb1 = 0, tb2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb1, deg, eoff, (int64_t)V + 1);
  cub::DeviceScan::ExclusiveSum(nullptr, tb2, wcnt, wpos, (int64_t)nw);
  void* tmp = scratch<uint8_t>(ctx, "bfs.cubtmp", std::max(tb1, tb2));
  if (!tmp) return fail(ctx, AGILE_E_CUDA, "bfs scratch allocation failed");
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, st));
  CK(cudaMemsetAsync(level, 0xff, (size_t)V * 4, st));   // -1 = unreached
  CK(cudaMemsetAsync(visited, 0, (size_t)nw * 4, st));
  CK(cudaMemsetAsync(counters, 0, 16, st));
  const int zero = 0;
  const uint32_t sbit = 1u << (source & 31);
  CK(cudaMemcpyAsync(level + source, &zero, 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(visited + source / 32, &sbit, 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(fa, &source, 4, cudaMemcpyHostToDevice, st));
  const uint32_t cap = resident_ctas<BfsWork>(ctx);
  const uint32_t full = cap;
  uint32_t n = 1, levels = 0;
  int cur = 0;
  while (n) {
    frontier_degree_kernel<<<grid_for((uint64_t)n + 1), 256, 0, st>>>(reinterpret_cast<const long long*>(row_ptr), fa, n, deg, 0u);
    size_t tb = tb1;
    CK(cub::DeviceScan::ExclusiveSum(tmp, tb, deg, eoff, (int64_t)n + 1, st));
    CK(cudaMemsetAsync(next_bits, 0, (size_t)nw * 4, st));
    BfsWork w;
    w.row_ptr = reinterpret_cast<const long long*>(row_ptr);
    w.v0 = 0;
    w.frontier = fa;
    w.eoff = eoff;
    w.n = n;
    w.visited = visited;
    w.next_bits = next_bits;
    w.level = level;
    w.cur = cur;
    w.col_key0 = col_key0;
    w.pd = prefetch_distance;
    w.counters = reinterpret_cast<u64*>(counters);
    // small frontiers need few warps (8 edges-chunks per CTA); the grid never exceeds residency
    const uint64_t est = (uint64_t)n * 64 / BfsWork::kChunk + 1;
    const uint32_t users = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(full, (est + kCtaWarps - 1) / kCtaWarps));
    int rc = launch(ctx, w, users, st);
    if (rc) return rc;
    popc_kernel<<<grid_for(nw), 256, 0, st>>>(next_bits, nw, wcnt);
    tb = tb2;
    CK(cub::DeviceScan::ExclusiveSum(tmp, tb, wcnt, wpos, (int64_t)nw, st));
    compact_kernel<<<grid_for(nw), 256, 0, st>>>(next_bits, wcnt, wpos, nw, fb, nnext);
    CK(cudaMemcpyAsync(&n, nnext, 4, cudaMemcpyDeviceToHost, st));
    rc = agile_sync(ctx, st);
    if (rc) return rc;
    std::swap(fa, fb);
    ++cur;
    ++levels;
  }
  CK(cudaEventRecord(e1, st));
  uint64_t cnt[2] = {0, 0};
  CK(cudaMemcpyAsync(cnt, counters, 16, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (stats) {
    stats[0] = levels;
    stats[1] = cnt[0];
    stats[2] = cnt[1];
    stats[3] = (uint64_t)((double)ms * 1e6);
  }
  return 0;
}

int agile_spmv(agile_ctx* ctx, const int64_t* row_ptr, uint32_t V, uint64_t E, uint64_t col_key0, uint64_t val_key0,
               const float* x, float* y, float alpha, float beta, uint32_t prefetch_distance, uint64_t* counters,
               void* stream) {
  return agile_spmv_rows(ctx, row_ptr, V, E, V, col_key0, val_key0, x, y, alpha, beta, prefetch_distance, counters,
                         stream);
}

int agile_spmv_rows(agile_ctx* ctx, const int64_t* row_ptr, uint32_t n_rows, uint64_t e_end, uint32_t x_len,
                    uint64_t col_key0, uint64_t val_key0, const float* x, float* y, float alpha, float beta,
                    uint32_t prefetch_distance, uint64_t* counters, void* stream) {
  if (!ctx || !row_ptr || !x || !y || !counters || !n_rows || !x_len) return fail(ctx, AGILE_E_ARG, "null spmv arg");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const uint64_t nch = (e_end + SpmvWork::kChunk - 1) / SpmvWork::kChunk;
  double* pf = scratch<double>(ctx, "spmv.first", nch);
  double* pl = scratch<double>(ctx, "spmv.last", nch);
  uint32_t* lr = scratch<uint32_t>(ctx, "spmv.lastrow", nch);
  if (!pf || !pl || !lr) return fail(ctx, AGILE_E_CUDA, "spmv scratch allocation failed");
  fill_f32_kernel<<<grid_for(n_rows), 256, 0, st>>>(y, n_rows, beta);   // rows without edges: alpha * 0 + beta
  if (!nch) return 0;
  CK(cudaMemsetAsync(lr, 0xff, nch * 4, st));
  SpmvWork w;
  w.row_ptr = reinterpret_cast<const long long*>(row_ptr);
  w.V = n_rows;
  w.nx = x_len;
  w.E = e_end;
  w.x = x;
  w.y = y;
  w.alpha = alpha;
  w.beta = beta;
  w.col_key0 = col_key0;
  w.val_key0 = val_key0;
  w.part_first = pf;
  w.part_last = pl;
  w.last_row = lr;
  w.pd = prefetch_distance;
  w.counters = reinterpret_cast<u64*>(counters);
  const uint32_t cap = resident_ctas<SpmvWork>(ctx);
  const uint32_t full = cap;
  const uint32_t users = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(full, (nch + kCtaWarps - 1) / kCtaWarps));
  int rc = launch(ctx, w, users, st);
  if (rc) return rc;
  spmv_fixup_kernel<<<grid_for(nch), 256, 0, st>>>(reinterpret_cast<const long long*>(row_ptr), lr, pf, pl, nch,
                                                     e_end, alpha, beta, y);
  CK(cudaGetLastError());
  return 0;
}

int agile_bfs_level(agile_ctx* ctx, const int64_t* row_ptr, uint32_t v0, const int32_t* frontier, uint32_t n,
                    uint32_t* visited, uint32_t* next_bits, int32_t* level, int32_t cur, uint64_t col_key0,
                    uint32_t prefetch_distance, uint64_t* counters, void* stream) {
  if (!ctx || !row_ptr || !visited || !next_bits || !level || !counters || (n && !frontier))
    return fail(ctx, AGILE_E_ARG, "null bfs_level arg");
  if (!n) return 0;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  long long* deg = scratch<long long>(ctx, "bfsl.deg", (size_t)n + 1);
  long long* eoff = scratch<long long>(ctx, "bfsl.eoff", (size_t)n + 1);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, deg, eoff, (int64_t)n + 1);
  void* tmp = scratch<uint8_t>(ctx, "bfsl.cubtmp", tb);
  if (!deg || !eoff || !tmp) return fail(ctx, AGILE_E_CUDA, "bfs_level scratch allocation failed");
  frontier_degree_kernel<<<grid_for((uint64_t)n + 1), 256, 0, st>>>(reinterpret_cast<const long long*>(row_ptr),
                                                                     frontier, n, deg, v0);
  CK(cub::DeviceScan::ExclusiveSum(tmp, tb, deg, eoff, (int64_t)n + 1, st));
  BfsWork w;
  w.row_ptr = reinterpret_cast<const long long*>(row_ptr);
  w.v0 = v0;
  w.frontier = frontier;
  w.eoff = eoff;
  w.n = n;
  w.visited = visited;
  w.next_bits = next_bits;
  w.level = level;
  w.cur = cur;
  w.col_key0 = col_key0;
  w.pd = prefetch_distance;
  w.counters = reinterpret_cast<u64*>(counters);
  const uint32_t full = resident_ctas<BfsWork>(ctx);
  const uint64_t est = (uint64_t)n * 64 / BfsWork::kChunk + 1;
  const uint32_t users = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(full, (est + kCtaWarps - 1) / kCtaWarps));
  return launch(ctx, w, users, st);
}

}  // extern "C"

// Device alias of a pinned, device-mapped host output buffer (nullptr: pageable, or
// AGILE_E2E_DIRECT_OUT=0): the host-buffer entries then let K5 store the pooled rows into it.
static float* mapped_host_out(float* out) {
  const char* ev = getenv("AGILE_E2E_DIRECT_OUT");
  if (ev && ev[0] == '0') return nullptr;
  cudaPointerAttributes pa{};
  float* r = nullptr;
  if (cudaPointerGetAttributes(&pa, out) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer)
    r = reinterpret_cast<float*>(pa.devicePointer);
  cudaGetLastError();   // clear a lookup failure of a pageable pointer
  return r;
}

extern "C" {

int agile_embbag_host_submit(agile_ctx* ctx, const int64_t* idx, const uint64_t* table_key0,
                             const int64_t* table_rows, float* out, uint64_t* counters, uint32_t B, uint32_t T,
                             uint32_t L, uint32_t D, uint32_t prefetch_distance, int slot) {
  if (!ctx || !idx || !out || slot < 0 || slot > 1) return fail(ctx, AGILE_E_ARG, "bad embbag_host_submit arg");
  CK(cudaSetDevice(ctx->device));
  auto& h = ctx->hs[slot];
  if (h.busy) return fail(ctx, AGILE_E_ARG, "slot busy: agile_embbag_host_wait it first");
  if (!h.st) {
    CK(cudaStreamCreateWithFlags(&h.st, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&h.ran, cudaEventDisableTiming));
    CK(cudaHostAlloc(&h.h_cnt, 16, cudaHostAllocDefault));
  }
  const size_t n_idx = (size_t)B * T * L * 8, n_out = (size_t)B * T * D * 4, n_tab = (size_t)T * 8;
  const size_t need = n_idx + n_out + 2 * n_tab + 16 + 256;
  if (h.bytes < need) {
    if (h.d) { cudaStreamSynchronize(h.st); cudaFree(h.d); }
    CK(cudaMalloc(&h.d, need));
    h.bytes = need;
  }
  uint8_t* base = reinterpret_cast<uint8_t*>(h.d);
  int64_t* d_idx = reinterpret_cast<int64_t*>(base);
  float* d_out = reinterpret_cast<float*>(base + n_idx);
  uint64_t* d_key = reinterpret_cast<uint64_t*>(base + n_idx + n_out);
  int64_t* d_rows = reinterpret_cast<int64_t*>(base + n_idx + n_out + n_tab);
  uint64_t* d_cnt = reinterpret_cast<uint64_t*>(base + n_idx + n_out + 2 * n_tab);
  // inputs ride in while the other slot's run is on the device; the run itself waits for the
  // previous run (one context: runs never overlap), its output leaves while the next run starts
  CK(cudaMemcpyAsync(d_idx, idx, n_idx, cudaMemcpyHostToDevice, h.st));
  CK(cudaMemcpyAsync(d_key, table_key0, n_tab, cudaMemcpyHostToDevice, h.st));
  CK(cudaMemcpyAsync(d_rows, table_rows, n_tab, cudaMemcpyHostToDevice, h.st));
  CK(cudaMemsetAsync(d_cnt, 0, 16, h.st));
  if (ctx->last_slot >= 0) CK(cudaStreamWaitEvent(h.st, ctx->hs[ctx->last_slot].ran, 0));
  // Pinned (device-mapped) output: the kernel stores each pooled bag straight into host memory as
  // it finishes — 512 B posted writes spread over the run — instead of a 27 MB copy-engine
  // download after it, whose upstream burst slows the next run's page fills by about its own
  // length (pipelined e2e step 3.02-3.12 ms against 3.32-3.53 staged, profiles/
  // e2e_direct_out_ab_r02q.txt).  Pageable output, or AGILE_E2E_DIRECT_OUT=0: device staging + D2H.
  float* kout = mapped_host_out(out);
  const bool direct = kout != nullptr;
  if (!direct) kout = d_out;
  int rc = agile_embbag(ctx, d_idx, d_key, d_rows, kout, d_cnt, B, T, L, D, 0, 0, prefetch_distance, h.st);
  if (rc) return rc;
  CK(cudaEventRecord(h.ran, h.st));
  ctx->last_slot = slot;
  if (!direct) CK(cudaMemcpyAsync(out, d_out, n_out, cudaMemcpyDeviceToHost, h.st));
  CK(cudaMemcpyAsync(h.h_cnt, d_cnt, 16, cudaMemcpyDeviceToHost, h.st));
  h.user_cnt = counters;
  h.busy = true;
  return 0;
}

int agile_embbag_host_wait(agile_ctx* ctx, int slot) {
  if (!ctx || slot < 0 || slot > 1) return fail(ctx, AGILE_E_ARG, "bad slot");
  auto& h = ctx->hs[slot];
  if (!h.busy) return 0;
  h.busy = false;
  int rc = agile_sync(ctx, h.st);
  if (!rc && h.user_cnt) { h.user_cnt[0] += h.h_cnt[0]; h.user_cnt[1] += h.h_cnt[1]; }
  return rc;
}

int agile_embbag_host(agile_ctx* ctx, const int64_t* idx, const uint64_t* table_key0, const int64_t* table_rows,
                      float* out, uint64_t* counters, uint32_t B, uint32_t T, uint32_t L, uint32_t D,
                      uint32_t prefetch_distance) {
  if (!ctx || !idx || !out) return fail(ctx, AGILE_E_ARG, "null embbag_host arg");
  CK(cudaSetDevice(ctx->device));
  const size_t n_idx = (size_t)B * T * L * 8, n_out = (size_t)B * T * D * 4, n_tab = (size_t)T * 8;
  const size_t need = n_idx + n_out + 2 * n_tab + 16 + 256;
  if (ctx->d_stage_bytes < need) {
    if (ctx->d_stage) cudaFree(ctx->d_stage);
    CK(cudaMalloc(&ctx->d_stage, need));
    ctx->d_stage_bytes = need;
  }
  uint8_t* base = reinterpret_cast<uint8_t*>(ctx->d_stage);
  int64_t* d_idx = reinterpret_cast<int64_t*>(base);
  float* d_out = reinterpret_cast<float*>(base + n_idx);
  uint64_t* d_key = reinterpret_cast<uint64_t*>(base + n_idx + n_out);
  int64_t* d_rows = reinterpret_cast<int64_t*>(base + n_idx + n_out + n_tab);
  uint64_t* d_cnt = reinterpret_cast<uint64_t*>(base + n_idx + n_out + 2 * n_tab);
  cudaStream_t st = ctx->stream;
  CK(cudaMemcpyAsync(d_idx, idx, n_idx, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_key, table_key0, n_tab, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_rows, table_rows, n_tab, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(d_cnt, 0, 16, st));
  float* kout = mapped_host_out(out);   // pinned output: the kernel stores into it directly
  int rc = agile_embbag(ctx, d_idx, d_key, d_rows, kout ? kout : d_out, d_cnt, B, T, L, D, 0, 0, prefetch_distance, st);
  if (rc) return rc;
  if (!kout) CK(cudaMemcpyAsync(out, d_out, n_out, cudaMemcpyDeviceToHost, st));
  uint64_t cnt[2] = {0, 0};
  CK(cudaMemcpyAsync(cnt, d_cnt, 16, cudaMemcpyDeviceToHost, st));
  rc = agile_sync(ctx, st);
  if (!rc && counters) { counters[0] += cnt[0]; counters[1] += cnt[1]; }
  return rc;
}

}  // extern "C"
