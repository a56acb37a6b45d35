// %globaltimer update granularity probe (GPU-box tool): one thread spins ~200 us, recording every
// change of %globaltimer with clock64; prints the histogram of update steps in ns.
#include <cstdio>
#include <map>
__global__ void k(unsigned long long* out, int n) {
  unsigned long long last, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(last));
  int i = 0;
  long long c0 = clock64();
  while (i < n && clock64() - c0 < 2000000) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t != last) { out[i++] = t - last; last = t; }
  }
  out[n] = i;
}
int main() {
  const int n = 4096;
  unsigned long long* d; cudaMalloc(&d, (n + 1) * 8);
  unsigned long long h[n + 1];
  for (int rep = 0; rep < 2; ++rep) {
    k<<<1, 1>>>(d, n);
    cudaMemcpy(h, d, (n + 1) * 8, cudaMemcpyDeviceToHost);
    std::map<unsigned long long, int> hist;
    for (unsigned long long i = 0; i < h[n]; ++i) hist[h[i]]++;
    printf("rep %d: %llu updates;", rep, h[n]);
    int shown = 0;
    for (auto& kv : hist) { if (shown++ < 12) printf(" %lluns x%d", kv.first, kv.second); }
    printf("\n");
  }
  return 0;
}
