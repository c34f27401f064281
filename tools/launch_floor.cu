// Per-launch floor of back-to-back dependent kernels in a CUDA graph on this
// GPU: an (almost) empty kernel, with and without programmatic dependent
// launch, at the advance kernel's grid shape. nvcc -arch=sm_100a -o launch_floor launch_floor.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_pdl(const int* in, int* out, int dep) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (dep) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) out[blockIdx.x] = in[blockIdx.x] + 1;
}

float run(int grid, int block, size_t smem, bool pdl, int dep, int n) {
  int *in, *out;
  cudaMalloc(&in, 1 << 20);
  cudaMalloc(&out, 1 << 20);
  cudaMemset(in, 0, 1 << 20);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaFuncSetAttribute(k_pdl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < n; ++i) cudaLaunchKernelEx(&cfg, k_pdl, (const int*)in, out, dep);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaFree(in);
  cudaFree(out);
  cudaStreamDestroy(s);
  return ms * 1e3f / n;
}

int main() {
  const int n = 400;
  printf("grid block smem pdl wait us/launch\n");
  for (int pdl = 0; pdl < 2; ++pdl)
    for (int dep = 0; dep < 2; ++dep) {
      if (!pdl && !dep) continue;
      printf("147 224 69K %d %d %.3f\n", pdl, dep, run(147, 224, 69 * 1024, pdl, dep, n));
      printf("147 224  0K %d %d %.3f\n", pdl, dep, run(147, 224, 0, pdl, dep, n));
      printf("  1  32  0K %d %d %.3f\n", pdl, dep, run(1, 32, 0, pdl, dep, n));
      printf("512 256 78K %d %d %.3f\n", pdl, dep, run(512, 256, 78 * 1024, pdl, dep, n));
    }
  return 0;
}
