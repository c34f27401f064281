// Synthetic transducer joint on the GPU — INPUT GENERATION ONLY (no part of the
// NGPU-LM method): stands in for the neural joint network of the label-looping
// driver (SPEC.md:276-283 SyntheticScorer, splitmix64 of SPEC.md:348). Row b is
// the joint output for (frame[b], u[b], last[b]):
//   h = seed; for x in (t, u, last + 1): h = splitmix64(h ^ x)
//   x = float((splitmix64(h ^ v) >> 40) * 2^-24); x = fl32(x + blank_bias) at v == blank
//   out[b, v] = x * temperature
// Unnormalized scores (greedy decisions only depend on their order), every
// value exact in float32 for a power-of-two temperature, so the CPU twins
// (synth.synthetic_joint_raw, the oracle's own copy) produce identical bits.
#include <cstdint>
#include <cuda_runtime.h>

namespace {
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void joint_kernel(uint64_t seed, int32_t B, const int32_t* frame, const int32_t* u, const int32_t* last,
                             int32_t ncols, int32_t blank, float blank_bias, float temperature, float* out,
                             int64_t row_stride) {
  const int32_t b = blockIdx.y;
  if (b >= B) return;
  uint64_t h = seed;
  h = splitmix64(h ^ (uint64_t)(int64_t)frame[b]);
  h = splitmix64(h ^ (uint64_t)(int64_t)u[b]);
  h = splitmix64(h ^ (uint64_t)(int64_t)(last[b] + 1));
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < ncols; v += gridDim.x * blockDim.x) {
    const uint64_t r = splitmix64(h ^ (uint64_t)v) >> 40;
    float x = (float)r * 5.9604644775390625e-08f;
    if (v == blank) x = __fadd_rn(x, blank_bias);
    out[(size_t)b * row_stride + v] = __fmul_rn(x, temperature);
  }
}
}  // namespace

extern "C" int synth_joint(uint64_t seed, int32_t B, const int32_t* frame, const int32_t* u, const int32_t* last,
                           int32_t ncols, int32_t blank, float blank_bias, float temperature, float* out,
                           int64_t row_stride, void* stream) {
  if (B <= 0) return 0;
  dim3 grid((ncols + 255) / 256, B);
  joint_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(seed, B, frame, u, last, ncols, blank, blank_bias, temperature, out,
                                                                row_stride);
  return (int)cudaGetLastError();
}
