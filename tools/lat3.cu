// What makes the advance kernel's first dependent loads slow? Variants of
// the same two-load chain (states[b] -> record[state]) as the kernel does it.
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

__device__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
template <bool kPdl, bool kBig, bool kTma = false>
__global__ void k(const int* __restrict__ states, const int4* __restrict__ table, int slots, long long* out, int* sink) {
  extern __shared__ __align__(16) int smem[];
  __shared__ __align__(8) unsigned long long bar;
  const int b = blockIdx.x, lane = threadIdx.x & 31;
  if (kTma && threadIdx.x == 32) {
    const unsigned bb = smem_u32(&bar), bytes = 4096;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bb) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(2u * bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(smem)), "l"(table), "r"(bytes), "r"(bb) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(smem + 1024)), "l"(table + 256), "r"(bytes), "r"(bb) : "memory");
  }
  if (kPdl) { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); asm volatile("griddepcontrol.wait;" ::: "memory"); }
  if (threadIdx.x >= 32) {
    if (kBig && !kTma) smem[threadIdx.x] = threadIdx.x;
    __syncthreads();
    if (kTma) { unsigned done = 0; do { asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(smem_u32(&bar)) : "memory"); } while (!done); }
    return;
  }
  long long t0 = clock64();
  int s = __shfl_sync(0xffffffffu, lane == 0 ? __ldg(&states[b]) : 0, 0);
  long long t1 = clock64();
  int4 x = make_int4(0, 0, 0, 0);
  if (lane < slots) x = __ldg(table + (size_t)s * slots + lane);
  int v = __shfl_sync(0xffffffffu, x.x + x.y, 0);
  long long t2 = clock64();
  if (lane == 0) { out[b * 2] = t1 - t0; out[b * 2 + 1] = t2 - t1; sink[b] = v; }
  __syncthreads();
  if (kTma) { unsigned done = 0; do { asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(smem_u32(&bar)) : "memory"); } while (!done); }
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
  std::vector<long long> out(B * 2);
  auto run = [&](const char* name, auto kern, int threads, size_t smem, bool pdl, int nb) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nb); cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = smem; cfg.stream = 0;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr; cfg.numAttrs = pdl ? 1 : 0;
    for (int r = 0; r < 3; ++r) cudaLaunchKernelEx(&cfg, kern, (const int*)ds, (const int4*)dt, slots, dout, sink);
    cudaDeviceSynchronize();
    cudaMemcpy(out.data(), dout, nb * 16, cudaMemcpyDeviceToHost);
    std::vector<long long> a, c;
    for (int i = 0; i < nb; ++i) { a.push_back(out[i * 2]); c.push_back(out[i * 2 + 1]); }
    std::sort(a.begin(), a.end()); std::sort(c.begin(), c.end());
    printf("%-34s B=%4d: states %5lld (max %5lld) | record %5lld (max %5lld)  err=%s\n", name, nb, a[nb / 2], a.back(),
           c[nb / 2], c.back(), cudaGetErrorString(cudaGetLastError()));
  };
  for (int nb : {128, 1024}) {
    run("32 thr, no smem, no pdl", k<false, false>, 32, 0, false, nb);
    run("256 thr, no smem, no pdl", k<false, false>, 256, 0, false, nb);
    run("256 thr, 20KB smem, no pdl", k<false, true>, 256, 20 * 1024, false, nb);
    run("256 thr, 20KB smem, pdl attr+wait", k<true, true>, 256, 20 * 1024, true, nb);
    run("256 thr, 20KB, pdl, TMA prologue", k<true, true, true>, 256, 20 * 1024, true, nb);
  }
  return 0;
}
