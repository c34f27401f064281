// Pointer-chase latency microbenchmark (B200): cycles per dependent 4-byte load
// for working sets from 1 MB (L2) to 2 GB (HBM). One thread, random cyclic
// permutation at 128-byte granularity.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void chase(const unsigned* __restrict__ next, unsigned start, int iters, unsigned long long* out, unsigned* sink) {
  unsigned p = start;
  for (int i = 0; i < 64; ++i) p = next[p];  // warm TLB / caches a bit
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = next[p];
  long long t1 = clock64();
  out[0] = (unsigned long long)(t1 - t0);
  *sink = p;
}

int main() {
  const size_t sizes_mb[] = {1, 8, 32, 64, 96, 128, 256, 1024, 2048};
  unsigned long long* d_out; unsigned* d_sink;
  cudaMalloc(&d_out, 8); cudaMalloc(&d_sink, 4);
  for (size_t mb : sizes_mb) {
    size_t n = mb * (1 << 20) / 4, stride = 32;  // 128-byte lines
    size_t lines = n / stride;
    std::vector<unsigned> perm(lines);
    for (size_t i = 0; i < lines; ++i) perm[i] = (unsigned)i;
    std::mt19937_64 g(1);
    std::shuffle(perm.begin(), perm.end(), g);
    std::vector<unsigned> h(n, 0);
    for (size_t i = 0; i < lines; ++i) h[(size_t)perm[i] * stride] = perm[(i + 1) % lines] * (unsigned)stride;
    unsigned* d; cudaMalloc(&d, n * 4);
    cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
    int iters = 20000;
    // first pass warms L2, second measures
    for (int rep = 0; rep < 2; ++rep) chase<<<1, 1>>>(d, perm[0] * (unsigned)stride, iters, d_out, d_sink);
    unsigned long long cyc; cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
    printf("%6zu MB: %.1f cycles/load\n", mb, (double)cyc / iters);
    cudaFree(d);
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock rate attr %d kHz\n", clk);
  return 0;
}
