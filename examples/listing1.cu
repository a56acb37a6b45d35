// The paper's Listing 1 as a third-party kernel over the public device API
// (include/agile_device.cuh): every thread prefetches one block (Method 1), async-reads another
// into its own AgileBuf, waits and publishes a digest, writes the buffer back to a third block
// (Method 2), and reads one u32 through the array view (Method 3).  Built by build() into
// examples/libagile_listing1.so; tests/test_gpu_device_api.py drives it through ctypes.
#include <cstdint>
#include "../include/agile_b200.h"
#include "../include/agile_device.cuh"

namespace {

__global__ void listing1_kernel(const __grid_constant__ agile::DevCtx c, const agile::Launch L, uint32_t n,
                                uint64_t nblk, uint4* bufs, agile::WaitNode* nodes, unsigned long long* digest,
                                uint32_t* got, int do_write) {
  agile::UserRun run(c, L);
  agile::AgileCtrl ctrl(c);
  for (uint32_t t0 = blockIdx.x * blockDim.x; t0 < n; t0 += gridDim.x * blockDim.x) {
    const uint32_t t = t0 + threadIdx.x;
    const bool act = t < n;
    // Method 1: AGILE prefetch
    ctrl.prefetch(act, 0, act ? (t * 7ull) % nblk : 0);
    // Method 2: AGILE async_issue
    agile::AgileBufPtr buf{nodes + (act ? t : 0), bufs + (uint64_t)(act ? t : 0) * 256};
    ctrl.asyncRead(act, 0, act ? (uint64_t)t % nblk : 0, buf);
    ctrl.wait(act, buf);
    if (act) digest[t] = *reinterpret_cast<const unsigned long long*>(buf.data);
    __syncwarp();
    if (do_write) {
      ctrl.asyncWrite(act, 0, act ? nblk - 1 - (t % nblk) : 0, buf);
      ctrl.wait(act, buf);
    }
    // Method 3: AGILE array-like synchronous API
    const uint32_t v = ctrl.get<uint32_t>(act, 0, act ? (uint64_t)t * 1029ull % (nblk * 1024) : 0);
    if (act) got[t] = v;
  }
}

}  // namespace

extern "C" int listing1_run(agile_ctx* ctx, uint32_t n, uint64_t nblk, void* bufs, uint64_t* digest, uint32_t* got,
                            int do_write, void* stream) {
  const uint32_t ctas = (n + agile::kCtaThreads - 1) / agile::kCtaThreads < 64 ? (n + agile::kCtaThreads - 1) / agile::kCtaThreads : 64;
  if (agile::prepare_user(listing1_kernel) != cudaSuccess) return -1;
  agile::DevCtx dc;
  agile::Launch L;
  void* nodes = nullptr;
  int rc = agile_user_run_begin(ctx, stream, ctas, n, &dc, sizeof(dc), &L, sizeof(L), &nodes);
  if (rc) return rc;
  cudaError_t e = agile::launch_user(listing1_kernel, ctas, reinterpret_cast<cudaStream_t>(stream), dc, L, n, nblk,
                                     reinterpret_cast<uint4*>(bufs), reinterpret_cast<agile::WaitNode*>(nodes),
                                     reinterpret_cast<unsigned long long*>(digest), got, do_write);
  if (e != cudaSuccess) return -1;
  return agile_user_run_end(ctx, stream);
}
