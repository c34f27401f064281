// Streaming floor of the persistent CTC decode's frame reads (B rows x T frames
// x (V+1) f32, each row contiguous): (a) the decode's producer/consumer TMA ring
// with a no-op or plain-argmax consumer, (b) W warps per row each loading and
// reducing its own frames with plain coalesced loads (frame-parallel).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stream_frames tools/stream_frames.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>
#include <climits>

constexpr int NC = 1025;
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(phase) : "memory");
  } while (!done);
}
__device__ __forceinline__ uint32_t fkey(float v) {
  const uint32_t u = __float_as_uint(v);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ int warp_argmax(const float* v33) {
  const int lane = threadIdx.x & 31;
  float m = v33[0];
  for (int j = 1; j < 33; ++j) m = fmaxf(m, v33[j]);
  const uint32_t k = __reduce_max_sync(~0u, fkey(m));
  const float M = __uint_as_float((k & 0x80000000u) ? (k ^ 0x80000000u) : ~k);
  int c = INT_MAX;
  for (int j = 32; j >= 0; --j) if (v33[j] == M) c = lane + 32 * j;
  return (int)__reduce_min_sync(~0u, (uint32_t)c);
}

// (a) ring: 2 warps per row, R rows per CTA
template <int MODE>
__global__ void ring_kernel(const float* x, int B, int T, int depth, int* out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int R = blockDim.x >> 6, wid = threadIdx.x >> 5, w = wid % R, lane = threadIdx.x & 31;
  const bool producer = wid >= R;
  const size_t lb = ((size_t)NC * 4 + 16 + 15) / 16 * 16;
  unsigned char* base = smem + (size_t)w * (256 + depth * lb);
  uint64_t* full = reinterpret_cast<uint64_t*>(base);
  uint64_t* empty = full + 16;
  float* ring = reinterpret_cast<float*>(base + 256);
  const int row = blockIdx.x * R + w;
  if (!producer && lane == 0) {
    for (int i = 0; i < depth; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + i)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(empty + i)));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (row >= B) return;
  const float* r0 = x + (size_t)row * T * NC;
  if (producer) {
    int slot = 0; uint32_t ph = 0;
    for (int t = 0; t < T; ++t) {
      if (t >= depth) mbar_wait(empty + slot, ph);
      const float* src = r0 + (size_t)t * NC;
      uintptr_t s = (uintptr_t)src, lo = (s + 15) & ~(uintptr_t)15, hi = (s + NC * 4) & ~(uintptr_t)15;
      if (lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + slot)), "r"((uint32_t)(hi - lo)) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(ring + slot * (lb / 4) + 4)), "l"(lo), "r"((uint32_t)(hi - lo)), "r"(smem_u32(full + slot)) : "memory");
      }
      if (++slot == depth) { slot = 0; if (t >= depth) ph ^= 1; }
    }
    return;
  }
  int slot = 0; uint32_t ph = 0; int acc = 0;
  for (int t = 0; t < T; ++t) {
    mbar_wait(full + slot, ph);
    const float* b = ring + slot * (lb / 4) + 4;
    if (MODE == 1) {
      float v[33];
      for (int j = 0; j < 33; ++j) { int c = lane + 32 * j; v[j] = c < NC - 8 ? b[c] : -1e30f; }
      acc += warp_argmax(v);
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + slot)) : "memory");
    if (++slot == depth) { slot = 0; ph ^= 1; }
  }
  if (lane == 0) out[row] = acc;
}

__device__ __forceinline__ uint32_t fkey0(float v) { return fkey(v + 0.0f); }
__device__ __forceinline__ uint32_t nkey(float v) { return v == v ? fkey0(v) : 0u; }
// top two (+ third) of 33 keys per lane: VAR 0 = select-chain lowest column, 1 = tree min
template <int VAR>
__device__ __forceinline__ uint32_t top2(uint32_t (&k)[33]) {
  const int lane = threadIdx.x & 31;
  auto lane_max = [&]() {
    uint32_t t[33];
    for (int j = 0; j < 33; ++j) t[j] = k[j];
    for (int d = 1; d < 33; d *= 2)
      for (int j = 0; j + d < 33; j += 2 * d) t[j] = max(t[j], t[j + d]);
    return __reduce_max_sync(~0u, t[0]);
  };
  auto lowest = [&](uint32_t K) {
    if (VAR == 0) {
      uint32_t cm = 0xffffffffu;
      for (int j = 32; j >= 0; --j) cm = k[j] == K ? (uint32_t)(lane + 32 * j) : cm;
      return __reduce_min_sync(~0u, cm);
    }
    uint32_t t[33];
    for (int j = 0; j < 33; ++j) t[j] = k[j] == K ? (uint32_t)(lane + 32 * j) : 0xffffffffu;
    for (int d = 1; d < 33; d *= 2)
      for (int j = 0; j + d < 33; j += 2 * d) t[j] = min(t[j], t[j + d]);
    return __reduce_min_sync(~0u, t[0]);
  };
  auto drop = [&](uint32_t C) { for (int j = 0; j < 33; ++j) k[j] = lane + 32 * j == (int)C ? 0u : k[j]; };
  const uint32_t K1 = lane_max(); const uint32_t C1 = lowest(K1); drop(C1);
  const uint32_t K2 = lane_max(); const uint32_t C2 = lowest(K2); drop(C2);
  const uint32_t K3 = lane_max();
  return K1 ^ C1 ^ K2 ^ C2 ^ K3;
}
template <int VAR, int LISTS>
__global__ void sum_kernel(const float* x, int B, int T, int* out) {
  const int W = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31, row = blockIdx.x;
  const float* r0 = x + (size_t)row * T * NC;
  for (int t = w; t < T; t += W) {
    const float* f = r0 + (size_t)t * NC;
    uint32_t k[33], kz[33];
    for (int j = 0; j < 33; ++j) { int c = lane + 32 * j; float v = c < NC - 1 ? __ldcs(f + c) : __int_as_float(0x7fc00000); k[j] = nkey(v); kz[j] = nkey(__fmaf_rn(0.3f, (float)j, v)); }
    uint32_t a = top2<VAR>(k);
    if (LISTS == 2) a ^= top2<VAR>(kz);
    if (lane == 0) out[(size_t)row * T + t] = a;
  }
}

// (b) W warps per row (one CTA per row), warp w takes frames w, w+W, ...
__global__ void par_kernel(const float* x, int B, int T, int* out) {
  const int W = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31, row = blockIdx.x;
  const float* r0 = x + (size_t)row * T * NC;
  for (int t = w; t < T; t += W) {
    const float* f = r0 + (size_t)t * NC;
    float v[33];
    for (int j = 0; j < 33; ++j) { int c = lane + 32 * j; v[j] = c < NC ? __ldcs(f + c) : -1e30f; }
    const int a = warp_argmax(v);
    if (lane == 0) out[(size_t)row * T + t] = a;
  }
}

int main() {
  const int B = 256, T = 500;
  float* x; int* out;
  cudaMalloc(&x, (size_t)B * T * NC * 4);
  cudaMalloc(&out, (size_t)B * T * 4);
  std::vector<float> h((size_t)B * T * NC);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)((i * 2654435761u) % 1000) * 1e-3f;
  cudaMemcpy(x, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](auto f) { f(); cudaDeviceSynchronize(); float best = 1e9;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best; } return best; };
  const double bytes = (double)B * T * NC * 4;
  for (int R : {1, 2}) for (int depth : {4, 8, 16}) for (int mode : {0, 1}) {
    const size_t lb = ((size_t)NC * 4 + 16 + 15) / 16 * 16, sm = (size_t)R * (256 + depth * lb);
    auto k = mode ? ring_kernel<1> : ring_kernel<0>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    float ms = timeit([&] { k<<<(B + R - 1) / R, 64 * R, sm>>>(x, B, T, depth, out); });
    printf("ring R=%d depth=%2d %s: %.4f ms  %.0f GB/s  (%s)\n", R, depth, mode ? "argmax" : "noop  ", ms, bytes / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  }
  for (int W : {1, 2, 4, 8, 16}) {
    float ms = timeit([&] { par_kernel<<<B, 32 * W>>>(x, B, T, out); });
    printf("parallel W=%2d: %.4f ms  %.0f GB/s\n", W, ms, bytes / ms / 1e6);
  }
  for (int B2 : {1, 256}) for (int W : {1, 4, 8}) {
    float ms0 = timeit([&] { sum_kernel<0, 1><<<B2, 32 * W>>>(x, B2, T, out); });
    float ms1 = timeit([&] { sum_kernel<1, 1><<<B2, 32 * W>>>(x, B2, T, out); });
    float ms2 = timeit([&] { sum_kernel<1, 2><<<B2, 32 * W>>>(x, B2, T, out); });
    float msa = timeit([&] { par_kernel<<<B2, 32 * W>>>(x, B2, T, out); });
    printf("summary B=%3d W=%d: argmax %.4f ms, top2 chain %.4f ms, top2 tree %.4f ms, two lists %.4f ms\n", B2, W, msa, ms0, ms1, ms2);
  }
  return 0;
}
