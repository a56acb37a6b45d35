// Probe (GPU-box tool): can the TMA bulk-copy engine (cp.async.bulk) move 4 KiB pages from a
// host-pinned GPU-mapped store into HBM, and at what rate, vs the register-staged warp copy the
// device engine (K4) uses?  Random pages of an 8 GiB pinned store -> distinct 4 KiB HBM slots.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/probe_bulk tools/probe_bulk.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull; x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull; x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// register path: one warp moves one page per iteration, P pages in flight (8 x 16 B per lane each)
template <int P>
__global__ void reg_copy(const uint4* __restrict__ src, uint4* dst, uint64_t npages, uint64_t ndst, int iters) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  for (int it = 0; it < iters; it += P) {
    uint4 v[P][8];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const uint64_t pg = mix(w * 1000003ull + it + p) % npages;
#pragma unroll
      for (int k = 0; k < 8; ++k) v[p][k] = __ldcg(src + pg * 256 + lane + 32 * k);
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const uint64_t d = (w * iters + it + p) % ndst;
#pragma unroll
      for (int k = 0; k < 8; ++k) __stcs(dst + d * 256 + lane + 32 * k, v[p][k]);
    }
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// bulk path: one thread per CTA runs an S-stage ring of 4 KiB smem pages: global(host) -> smem
// with an mbarrier complete_tx, then smem -> global (HBM) as a bulk group
template <int S>
__global__ void bulk_copy(const uint8_t* __restrict__ src, uint8_t* dst, uint64_t npages, uint64_t ndst, int iters) {
  extern __shared__ __align__(128) uint8_t stage[];
  __shared__ __align__(8) uint64_t bar[S];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t phase = 0;   // bit s: parity of stage s
  const uint64_t cta = blockIdx.x;
  auto load = [&](int it) {
    const int s = it % S;
    const uint64_t pg = mix(cta * 1000003ull + it) % npages;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 4096;" :: "r"(smem_u32(&bar[s])) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];"
                 :: "r"(smem_u32(stage + s * 4096)), "l"(src + pg * 4096), "r"(smem_u32(&bar[s])) : "memory");
  };
  for (int it = 0; it < S && it < iters; ++it) load(it);
  for (int it = 0; it < iters; ++it) {
    const int s = it % S;
    // wait for stage s's bytes
    uint32_t done = 0;
    const uint32_t par = (phase >> s) & 1u;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(smem_u32(&bar[s])), "r"(par) : "memory");
    phase ^= 1u << s;
    const uint64_t d = (cta * iters + it) % ndst;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 4096;"
                 :: "l"(dst + d * 4096), "r"(smem_u32(stage + s * 4096)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // the store must have read stage s before the load of iteration it + S overwrites it
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    if (it + S < iters) load(it + S);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  const uint64_t gib = argc > 1 ? atoll(argv[1]) : 8;
  const uint64_t npages = (gib << 30) >> 12;
  const uint64_t ndst = (4ull << 30) >> 12;
  uint8_t* h;
  CK(cudaHostAlloc(&h, gib << 30, cudaHostAllocMapped));
  for (uint64_t i = 0; i < (gib << 30); i += 4096) h[i] = (uint8_t)(i >> 12);
  uint8_t* hd;
  CK(cudaHostGetDevicePointer(&hd, h, 0));
  uint8_t* d;
  CK(cudaMalloc(&d, ndst << 12));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  // register path (the K4 engine's page move)
  for (int warps : {256, 1024, 4096}) {
    const int iters = 64;
    reg_copy<4><<<warps / 8, 256>>>((const uint4*)hd, (uint4*)d, npages, ndst, iters);
    CK(cudaEventRecord(a));
    reg_copy<4><<<warps / 8, 256>>>((const uint4*)hd, (uint4*)d, npages, ndst, iters);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    const double bytes = (double)warps * iters * 4096;
    printf("{\"path\": \"register\", \"warps\": %d, \"pages_in_flight\": %d, \"GBps\": %.2f}\n", warps, warps * 4, bytes / ms / 1e6);
  }
  // bulk path
  for (int ctas : {sms, 2 * sms, 4 * sms}) {
    for (int S : {4, 8, 16}) {
      const int iters = 128;
      auto run = [&]() {
        const size_t sm = (size_t)S * 4096;
        if (S == 4) bulk_copy<4><<<ctas, 32, sm>>>(hd, d, npages, ndst, iters);
        if (S == 8) bulk_copy<8><<<ctas, 32, sm>>>(hd, d, npages, ndst, iters);
        if (S == 16) bulk_copy<16><<<ctas, 32, sm>>>(hd, d, npages, ndst, iters);
      };
      CK(cudaFuncSetAttribute(bulk_copy<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 4096));
      run();
      CK(cudaGetLastError());
      CK(cudaEventRecord(a));
      run();
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      const double bytes = (double)ctas * iters * 4096;
      printf("{\"path\": \"bulk\", \"ctas\": %d, \"stages\": %d, \"pages_in_flight\": %d, \"GBps\": %.2f}\n", ctas, S, ctas * S,
             bytes / ms / 1e6);
    }
  }
  // correctness spot check: one bulk page
  CK(cudaMemset(d, 0, 4096));
  bulk_copy<4><<<1, 32, 4 * 4096>>>(hd, d, 1, 1, 1);
  CK(cudaDeviceSynchronize());
  uint8_t chk[4096];
  CK(cudaMemcpy(chk, d, 4096, cudaMemcpyDeviceToHost));
  int ok = memcmp(chk, h, 4096) == 0;
  printf("{\"bulk_bytes_match\": %d}\n", ok);
  return 0;
}
