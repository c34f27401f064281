// Store-phase floor of a CTA-per-SM advance layout: grid = ceil(B / rpc) CTAs
// of W warps, rpc rows per CTA (one 8 KiB row buffer each), each row built
// (simulated: `spin` cycles) before griddepcontrol.wait and stored by TMA bulk
// stores after it — issued by each row's warp, or all by thread 0 after a CTA
// barrier. Residency is set with padding shared memory.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store_floor2 store_floor2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void store_row(char* dst, const unsigned char* row) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(row)), "r"(4096)
               : "memory");
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + 4096),
               "r"(smem_u32(row + 4096)), "r"(4096)
               : "memory");
}

__global__ void k_cta(char* out, int B, int rpc, int spin, int by_cta) {
  extern __shared__ __align__(16) unsigned char smem[];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, W = blockDim.x >> 5;
  const int r0 = blockIdx.x * rpc;
  for (int i = w; i < rpc; i += W) {  // "build" row i
    unsigned char* row = smem + (size_t)i * 8192;
    const long long t0 = clock64();
    while (clock64() - t0 < spin) {
    }
    for (int j = lane; j < 2048; j += 32) reinterpret_cast<int*>(row)[j] = j + i;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (by_cta) __syncthreads(); else __syncwarp();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (by_cta) {
    if (threadIdx.x == 0) {
      for (int i = 0; i < rpc && r0 + i < B; ++i) store_row(out + (size_t)(r0 + i) * 8192, smem + (size_t)i * 8192);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncthreads();
  } else {
    if (lane == 0) {
      for (int i = w; i < rpc && r0 + i < B; i += W) store_row(out + (size_t)(r0 + i) * 8192, smem + (size_t)i * 8192);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
  }
}

float run(int B, int rpc, int W, size_t smem, int spin, int by_cta, int n, char* buf, size_t nbuf) {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (smem < (size_t)rpc * 8192) smem = (size_t)rpc * 8192;
  cudaFuncSetAttribute(k_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = (B + rpc - 1) / rpc;
  cfg.blockDim = 32 * W;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const size_t per = (size_t)B * 8192;
  const int nrot = (int)(nbuf / per);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < n; ++i) cudaLaunchKernelEx(&cfg, k_cta, buf + (size_t)(i % nrot) * per, B, rpc, spin, by_cta);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(s);
  return best * 1e3f / n;
}

int main() {
  const size_t nbuf = (size_t)640 << 20;
  char* buf;
  cudaMalloc(&buf, nbuf);
  cudaMemset(buf, 0, nbuf);
  printf("B rpc W smemKB spin by_cta us/launch GB/s\n");
  for (int B : {1024, 4096}) {
    for (int rpc : {4, 7, 8}) {
      for (int W : {4, 8}) {
        if (W > rpc) continue;
        for (size_t smem : {(size_t)0, (size_t)100 << 10, (size_t)200 << 10})
          for (int spin : {0, 2000})
            for (int by_cta = 0; by_cta < 2; ++by_cta) {
              const float us = run(B, rpc, W, smem, spin, by_cta, 400, buf, nbuf);
              printf("%5d %2d %2d %4zu %5d %d %7.3f %7.0f\n", B, rpc, W, smem >> 10, spin, by_cta, us,
                     B * 8192.0 / us / 1e3);
            }
      }
    }
  }
  cudaFree(buf);
  return 0;
}
