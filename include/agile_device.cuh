// agile_device.cuh — public device API of the B200 AGILE path for third-party CUDA kernels: the
// three access methods of the paper's Listing 1, mirroring the reference's
// AgileApi (gpu_api.py:107-278):
//
//   Method 1  ctrl.prefetch(active, dev, blk)             AgileApi.prefetch      gpu_api.py:139-155
//   Method 2  ctrl.asyncRead(active, dev, blk, buf)       AgileApi.async_read    gpu_api.py:164-190
//             ctrl.wait(active, buf)                      AgileApi.wait          gpu_api.py:233-248
//             ctrl.asyncWrite(active, dev, blk, buf)      AgileApi.async_write   gpu_api.py:192-227
//   Method 3  ctrl.get<T>(active, dev, idx)               AgileApi.array_get     gpu_api.py:250-278
//
// Every verb is WARP-COLLECTIVE, as the reference's warp lockstep (gpu_api.py:40-54, prefetch_skip
// 157-162): all 32 lanes call it, each with its own request or active = false; lanes with the same
// block coalesce (lowest lane leads), misses are claimed and submitted warp-aggregated, nobody
// holds a lock or pin while waiting.
//
// A third-party kernel is the user grid of one AGILE run:
//   host:    agile::prepare_user(kernel)             // load the module before the infra grid spins
//            agile_user_run_begin(ctx, stream, n_ctas, n_bufs, &devctx, &launch, &nodes)
//            agile::launch_user(kernel, n_ctas, stream, devctx, launch, ...your args...)
//            agile_user_run_end(ctx, stream)
//   device:  __global__ void kernel(const __grid_constant__ agile::DevCtx c, const agile::Launch L, ...) {
//              agile::UserRun run(c, L);           // users_started / user_done bookkeeping
//              agile::AgileCtrl ctrl(c);
//              ...
//            }
// The kernel runs with blockDim = agile::kCtaThreads (256); `nodes` holds n_bufs AgileBuf barriers
// for asyncRead / asyncWrite (one per outstanding buffer).
#pragma once
#include <cuda_runtime.h>
#include "../paper_2504_19365_b200/csrc/agile_core.cuh"

namespace agile {

// AgileBuf (gpu_api.py:28-38): a 4 KiB user buffer and its transaction barrier
struct AgileBufPtr {
  WaitNode* node;
  uint4* data;
  __device__ __forceinline__ bool ready() const { return ld_acquire(&node->done) != 0; }
};

// bookkeeping every user CTA of a run performs (agile_user_kernel does the same)
struct UserRun {
  const DevCtx& c;
  u32 n;
  __device__ UserRun(const DevCtx& ctx, const Launch& L) : c(ctx), n(L.n_user_ctas) {
    if (threadIdx.x == 0) {
      const u32 prev = atomicAdd(&c.run->users_started, 1u);
      // the infra grid left before this grid could start beside it (see agile_user_kernel)
      if ((prev & kInfraGaveUp) && !c.solo_ok) set_error(c, E_LIVELOCK, 1, __LINE__);
    }
    __syncthreads();
  }
  __device__ ~UserRun() { user_done(c, n); }
};

class AgileCtrl {
 public:
  __device__ explicit AgileCtrl(const DevCtx& c)
      : c_(c), who_(WHO_USER | (blockIdx.x * kCtaThreads + threadIdx.x)), sq_(blockIdx.x * kCtaWarps + (threadIdx.x >> 5)) {}

  // Method 1: pull (dev, blk) toward the cache without waiting
  __device__ void prefetch(bool active, u32 dev, u64 blk) {
    prefetch_warp(c_, active, make_key(dev, blk), who_, sq_, false);
  }
  // Method 2: start filling buf from (dev, blk); check buf.ready() or wait() before reading it
  __device__ void asyncRead(bool active, u32 dev, u64 blk, AgileBufPtr buf) {
    async_read_warp(c_, active, make_key(dev, blk), buf.node, buf.data, who_, sq_);
  }
  __device__ bool wait(bool active, AgileBufPtr buf) { return wait_nodes_warp(c_, active, buf.node); }
  // Method 2: publish a whole block from buf; buf is reusable on return, wait(buf) = durable
  __device__ void asyncWrite(bool active, u32 dev, u64 blk, AgileBufPtr buf) {
    async_write_warp(c_, active, make_key(dev, blk), buf.node, buf.data, who_, sq_);
  }
  // Method 3: element idx of device dev viewed as an array of T (sizeof(T) divides 4096)
  template <class T>
  __device__ T get(bool active, u32 dev, u64 idx) {
    static_assert(kBlockBytes % sizeof(T) == 0, "element size must divide the block size");
    const u64 byte_off = idx * sizeof(T);
    const u64 key = make_key(dev, byte_off >> kBlockShift);
    const u32 off = (u32)(byte_off & (kBlockBytes - 1));
    T val{};
    bool pend = active;
    Spin sp;
    while (__any_sync(FULL, pend)) {
      const Req r = access_warp(c_, pend, key, true, who_, sq_, false);
      const bool pinned = pend && (r.kind == R_HIT || r.kind == R_FILLING || r.kind == R_MISS);
      u32 wp = __ballot_sync(FULL, pinned);
      Spin s2;
      while (wp) {
        bool rd = false;
        if ((wp >> lane_id()) & 1u) {
          const u64 w = ld_acquire(&c_.tags[r.line]);
          rd = tw_state(w) == ST_READY || tw_state(w) == ST_MODIFIED;
        }
        wp &= ~__ballot_sync(FULL, rd);
        if (wp && !s2.again(c_, 512, __LINE__)) break;
      }
      if (pinned) {
        val = *reinterpret_cast<const volatile T*>(line_ptr(c_, r.line) + off);
        unpin_line(c_, r.line, 1);
      }
      pend = pend && r.kind == R_RETRY;
      if (aborted(c_)) break;
      if (__any_sync(FULL, pend) && !sp.again(c_, 1024, __LINE__)) break;
    }
    return val;
  }

 private:
  const DevCtx& c_;
  u32 who_, sq_;
};

// Host helper: load a user kernel's module BEFORE agile_user_run_begin.  With lazy module loading
// the first launch of a kernel loads its module, and loading while the run's infra grid already
// spins can wait for the device to drain — the two grids would then never overlap.
template <class... KArgs>
cudaError_t prepare_user(void (*kernel)(KArgs...)) {
  cudaFuncAttributes a{};
  return cudaFuncGetAttributes(&a, kernel);
}

// Host helper: launch a third-party user kernel as the PDL dependent of the run's infra grid
// (it starts once every engine and service CTA is resident).
template <class... KArgs, class... Args>
cudaError_t launch_user(void (*kernel)(KArgs...), unsigned n_ctas, cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_ctas);
  cfg.blockDim = dim3(kCtaThreads);
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

}  // namespace agile
