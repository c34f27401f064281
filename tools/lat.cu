// Latency of the advance kernel's first two dependent loads, isolated:
// lane 0 loads states[b]; lanes 0..5 load the 96-byte record table[state].
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void k(const int* __restrict__ states, const int4* __restrict__ table, int slots,
                  long long* out, int* sink) {
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

int main() {
  const int S = 627559, slots = 6, B = 1024;
  std::vector<int4> h((size_t)S * slots);
  for (size_t i = 0; i < h.size(); ++i) h[i] = make_int4((int)i, 1, 2, 3);
  std::vector<int> st(B * 16);
  std::mt19937 g(1);
  for (auto& x : st) x = g() % S;
  int4* dt; int* ds; long long* dout; int* sink;
  cudaMalloc(&dt, h.size() * 16); cudaMalloc(&ds, st.size() * 4); cudaMalloc(&dout, B * 16); cudaMalloc(&sink, B * 4);
  cudaMemcpy(dt, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(ds, st.data(), st.size() * 4, cudaMemcpyHostToDevice);
  std::vector<long long> out(B * 2);
  for (int nb : {128, 1024}) {
    for (int rep = 0; rep < 3; ++rep) {
      k<<<nb, 32>>>(ds, dt, slots, dout, sink);
      cudaMemcpy(out.data(), dout, nb * 16, cudaMemcpyDeviceToHost);
      std::vector<long long> a, c;
      for (int i = 0; i < nb; ++i) { a.push_back(out[i * 2]); c.push_back(out[i * 2 + 1]); }
      std::sort(a.begin(), a.end()); std::sort(c.begin(), c.end());
      printf("B=%4d rep %d: states load med %lld max %lld | record load med %lld max %lld cycles\n", nb, rep,
             a[nb / 2], a.back(), c[nb / 2], c.back());
    }
  }
  return 0;
}
