// Floor of the advance call's store phase on this GPU: back-to-back dependent
// (PDL) kernels in a CUDA graph that do nothing but write B rows of 8 KiB
// (scores + next, V = 1024) from shared memory by TMA bulk stores after
// griddepcontrol.wait, outputs rotating over > 4x L2. Grid shapes: one warp
// per row and per CTA (the advance kernel's), R rows per CTA, a persistent
// grid of 148 CTAs; with and without the wait.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store_floor store_floor.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// rows_per_warp rows handled by each warp in turn; R warps per CTA
__global__ void k_store(char* out, int B, int dep, int rows_per_warp) {
  extern __shared__ __align__(16) unsigned char smem[];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, R = blockDim.x >> 5;
  unsigned char* row = smem + (size_t)w * 8192;
  for (int i = lane; i < 2048; i += 32) reinterpret_cast<int*>(row)[i] = i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (dep) asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int k = 0; k < rows_per_warp; ++k) {
    const int r = (blockIdx.x * R + w) * rows_per_warp + k;
    if (r >= B) break;
    if (lane == 0) {
      char* dst = out + (size_t)r * 8192;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(row)),
                   "r"(4096)
                   : "memory");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + 4096),
                   "r"(smem_u32(row + 4096)), "r"(4096)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

float run(int B, int grid, int warps, int rpw, int dep, bool pdl, int n, char* buf, size_t nbuf, size_t smem_min = 0) {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  size_t smem = (size_t)warps * 8192;
  if (smem < smem_min) smem = smem_min;
  cudaFuncSetAttribute(k_store, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = 32 * warps;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  const size_t per = (size_t)B * 8192;
  const int nrot = (int)(nbuf / per);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < n; ++i) cudaLaunchKernelEx(&cfg, k_store, buf + (size_t)(i % nrot) * per, B, dep, rpw);
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
  const int n = 400;
  printf("B grid warps rows/warp smemKB pdl wait us/launch GB/s\n");
  for (int B : {1024, 4096}) {
    struct Shape { int grid, warps, rpw; size_t smem; } shapes[] = {
        {B, 1, 1, 8192}, {B, 1, 1, 14 << 10}, {B, 1, 1, 28 << 10}, {B, 1, 1, 56 << 10},
        {B / 2, 1, 2, 8192}, {B / 2, 1, 2, 28 << 10}, {B / 4, 1, 4, 8192}, {B / 4, 1, 4, 28 << 10},
        {148, 1, (B + 147) / 148, 8192}, {148, 1, (B + 147) / 148, 56 << 10}, {148, 1, (B + 147) / 148, 110 << 10},
        {296, 1, (B + 295) / 296, 8192}, {296, 1, (B + 295) / 296, 56 << 10}};
    for (auto sh : shapes)
      for (int mode = 1; mode < 3; ++mode) {
        const bool pdl = mode > 0;
        const int dep = mode == 2;
        const float us = run(B, sh.grid, sh.warps, sh.rpw, dep, pdl, n, buf, nbuf, sh.smem);
        printf("%5d %5d %2d %3d %4zu %d %d %7.3f %7.0f\n", B, sh.grid, sh.warps, sh.rpw, sh.smem >> 10, (int)pdl, dep,
               us, B * 8192.0 / us / 1e3);
      }
  }
  cudaFree(buf);
  return 0;
}
