// Step-0 probe: host link roofline for the page store.
// Measures pinned H2D memcpy bandwidth, zero-copy kernel read bandwidth
// (sequential 16 B loads) and random 4 KiB page gathers over mapped host
// memory, plus cudaHostAlloc cost per GiB.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <chrono>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void seq_read(const int4* __restrict__ src, size_t n, int4* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    int4 v = src[i];
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}

// one warp per page: 32 lanes x 8 x 16 B = 4 KiB, copy into HBM destination
__global__ void page_gather(const int4* __restrict__ src, int4* __restrict__ dst, const uint32_t* pages,
                            int npages, int dst_pages) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  int nw = (gridDim.x * blockDim.x) >> 5;
  for (int p = warp; p < npages; p += nw) {
    const int4* s = src + (size_t)pages[p] * 256;
    int4* d = dst + (size_t)(p % dst_pages) * 256;
    int4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = s[lane + 32 * k];
#pragma unroll
    for (int k = 0; k < 8; ++k) d[lane + 32 * k] = v[k];
  }
}

int main(int argc, char** argv) {
  size_t gib = argc > 1 ? atoll(argv[1]) : 4;
  size_t bytes = gib << 30;
  auto t0 = std::chrono::steady_clock::now();
  void* h = nullptr;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  auto t1 = std::chrono::steady_clock::now();
  printf("cudaHostAlloc %zu GiB: %.3f s\n", gib, std::chrono::duration<double>(t1 - t0).count());
  memset(h, 1, bytes);
  auto t2 = std::chrono::steady_clock::now();
  printf("memset host %zu GiB: %.3f s\n", gib, std::chrono::duration<double>(t2 - t1).count());
  void* dh = nullptr;
  CK(cudaHostGetDevicePointer(&dh, h, 0));
  void* d = nullptr;
  size_t dbytes = (size_t)1 << 30;
  CK(cudaMalloc(&d, dbytes));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  float ms;
  // memcpy H2D 1 GiB
  for (int it = 0; it < 3; ++it) {
    CK(cudaEventRecord(a));
    CK(cudaMemcpyAsync(d, h, dbytes, cudaMemcpyHostToDevice));
    CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("memcpy H2D 1 GiB: %.3f ms = %.2f GB/s\n", ms, dbytes / ms / 1e6);
  }
  for (int it = 0; it < 2; ++it) {
    CK(cudaEventRecord(a));
    CK(cudaMemcpyAsync(h, d, dbytes, cudaMemcpyDeviceToHost));
    CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("memcpy D2H 1 GiB: %.3f ms = %.2f GB/s\n", ms, dbytes / ms / 1e6);
  }
  int4* sink; CK(cudaMalloc(&sink, 64));
  int grids[] = {148, 296, 592, 1184, 2368};
  for (int g : grids) {
    for (int bs : {256, 1024}) {
      CK(cudaEventRecord(a));
      seq_read<<<g, bs>>>((const int4*)dh, dbytes / 16, sink);
      CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
      CK(cudaGetLastError());
      CK(cudaEventElapsedTime(&ms, a, b));
      printf("zero-copy seq read grid %d x %d: %.2f GB/s\n", g, bs, dbytes / ms / 1e6);
    }
  }
  // random 4 KiB page gather
  size_t store_pages = bytes / 4096;
  int npages = 1 << 18;
  uint32_t* hp = (uint32_t*)malloc(npages * 4);
  uint64_t x = 88172645463325252ull;
  for (int i = 0; i < npages; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; hp[i] = x % store_pages; }
  uint32_t* dp; CK(cudaMalloc(&dp, npages * 4));
  CK(cudaMemcpy(dp, hp, npages * 4, cudaMemcpyHostToDevice));
  int dst_pages = dbytes / 4096;
  for (int g : grids) {
    for (int bs : {128, 256, 512}) {
      CK(cudaEventRecord(a));
      page_gather<<<g, bs>>>((const int4*)dh, (int4*)d, dp, npages, dst_pages);
      CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
      CK(cudaGetLastError());
      CK(cudaEventElapsedTime(&ms, a, b));
      printf("zero-copy 4KiB gather grid %d x %d: %.2f GB/s = %.2f MIOPS\n", g, bs,
             (double)npages * 4096 / ms / 1e6, npages / ms / 1e3);
    }
  }
  // HBM copy for reference
  void* d2; CK(cudaMalloc(&d2, dbytes));
  CK(cudaEventRecord(a));
  CK(cudaMemcpyAsync(d2, d, dbytes, cudaMemcpyDeviceToDevice));
  CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
  CK(cudaEventElapsedTime(&ms, a, b));
  printf("D2D copy 1 GiB: %.2f GB/s (r+w)\n", 2.0 * dbytes / ms / 1e6);
  int v = 0;
  CK(cudaDeviceGetAttribute(&v, cudaDevAttrPageableMemoryAccess, 0));
  printf("pageableMemoryAccess=%d\n", v);
  CK(cudaDeviceGetAttribute(&v, cudaDevAttrCanUseHostPointerForRegisteredMem, 0));
  printf("canUseHostPointerForRegisteredMem=%d\n", v);
  CK(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, 0));
  printf("SMs=%d\n", v);
  CK(cudaDeviceGetAttribute(&v, cudaDevAttrConcurrentKernels, 0));
  printf("concurrentKernels=%d\n", v);
  return 0;
}
