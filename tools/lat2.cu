// Are kernel-parameter (constant bank) reads on the critical path slow?
// Variant A: pointers as plain params. Variant B: pointers inside a by-value
// struct read after the first load (like DevModel). Variant C: B but the
// struct fields are read before the first load (hoisted).
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

struct M { const int4* pad0; const int4* pad1; const int* pad2; const float* pad3; const int* pad4;
           const int4* table; int slots; int S, V, order; unsigned long long* bad; };

__global__ void kA(const int* __restrict__ states, const int4* __restrict__ table, int slots, long long* out, int* sink) {
  const int b = blockIdx.x, lane = threadIdx.x & 31;
  long long t0 = clock64();
  int s = __shfl_sync(0xffffffffu, lane == 0 ? __ldg(&states[b]) : 0, 0);
  long long t1 = clock64();
  int4 x = make_int4(0, 0, 0, 0);
  if (lane < slots) x = __ldg(table + (size_t)s * slots + lane);
  int v = __shfl_sync(0xffffffffu, x.x + x.y, 0);
  long long t2 = clock64();
  if (lane == 0) { out[b * 2] = t1 - t0; out[b * 2 + 1] = t2 - t1; sink[b] = v; }
}
__global__ void kB(M m, const int* __restrict__ states, long long* out, int* sink) {
  const int b = blockIdx.x, lane = threadIdx.x & 31;
  long long t0 = clock64();
  int s = __shfl_sync(0xffffffffu, lane == 0 ? __ldg(&states[b]) : 0, 0);
  long long t1 = clock64();
  int4 x = make_int4(0, 0, 0, 0);
  if (lane < m.slots) x = __ldg(m.table + (size_t)s * m.slots + lane);
  int v = __shfl_sync(0xffffffffu, x.x + x.y, 0);
  long long t2 = clock64();
  if (lane == 0) { out[b * 2] = t1 - t0; out[b * 2 + 1] = t2 - t1; sink[b] = v; }
}

int main() {
  const int S = 627559, slots = 6, B = 1024;
  std::vector<int4> h((size_t)S * slots);
  for (size_t i = 0; i < h.size(); ++i) h[i] = make_int4((int)i, 1, 2, 3);
  std::vector<int> st(B);
  std::mt19937 g(1);
  for (auto& x : st) x = g() % S;
  int4* dt; int* ds; long long* dout; int* sink;
  cudaMalloc(&dt, h.size() * 16); cudaMalloc(&ds, st.size() * 4); cudaMalloc(&dout, B * 16); cudaMalloc(&sink, B * 4);
  cudaMemcpy(dt, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(ds, st.data(), st.size() * 4, cudaMemcpyHostToDevice);
  M m{}; m.table = dt; m.slots = slots; m.S = S;
  std::vector<long long> out(B * 2);
  auto rep = [&](const char* name, int nb) {
    cudaMemcpy(out.data(), dout, nb * 16, cudaMemcpyDeviceToHost);
    std::vector<long long> a, c;
    for (int i = 0; i < nb; ++i) { a.push_back(out[i * 2]); c.push_back(out[i * 2 + 1]); }
    std::sort(a.begin(), a.end()); std::sort(c.begin(), c.end());
    printf("%s B=%4d: first load med %lld | second load med %lld (max %lld) cycles\n", name, nb, a[nb / 2], c[nb / 2], c.back());
  };
  for (int nb : {128, 1024}) for (int r = 0; r < 2; ++r) {
    kA<<<nb, 32>>>(ds, dt, slots, dout, sink); cudaDeviceSynchronize(); rep("plain params ", nb);
    kB<<<nb, 32>>>(m, ds, dout, sink); cudaDeviceSynchronize(); rep("struct params", nb);
  }
  return 0;
}
