// Debug build only (NGPULM_PHASE_TIMING, tools/*timing*.py): the phase-stamp
// accessors and a dependent-load probe. Compiled only through unity_timing.cu.
#include "kcommon.cuh"

namespace ngpulm {
#ifdef NGPULM_PHASE_TIMING
// lat3-style probe on the model's own data: states[b] -> chain record, by warp 0.
__global__ void probe_kernel(DevModel m, const int32_t* __restrict__ states, long long* out) {
  const int b = blockIdx.x, lane = threadIdx.x & 31;
  long long t0 = clock64();
  const int32_t st = __shfl_sync(kFull, lane == 0 ? __ldg(&states[b]) : 0, 0);
  long long t1 = clock64();
  int4 x = make_int4(0, 0, 0, 0);
  if (lane < m.chain_slots) x = __ldg(reinterpret_cast<const int4*>(m.chain) + (size_t)st * m.chain_slots + lane);
  const int v = __shfl_sync(kFull, x.x + x.y, 0);
  long long t2 = clock64();
  if (lane == 0) { out[b * 3] = t1 - t0; out[b * 3 + 1] = t2 - t1; out[b * 3 + 2] = v; }
}
extern "C" int ngpulm_debug_probe(const DevModel* m, const int32_t* states, int32_t B, long long* out_dev) {
  probe_kernel<<<B, 32>>>(*m, states, out_dev);
  return (int)cudaDeviceSynchronize();
}
extern "C" int ngpulm_debug_skip(int bits) { return (int)cudaMemcpyToSymbol(g_skip, &bits, sizeof bits); }
extern "C" int ngpulm_debug_phases(unsigned long long* host, int n) {
  const int e = (int)cudaMemcpyFromSymbol(host, g_phase, sizeof(unsigned long long) * (size_t)n);
  void* p = nullptr;
  cudaGetSymbolAddress(&p, g_phase);
  cudaMemset(p, 0, sizeof(g_phase));  // rows a launch does not stamp read as 0 next time
  cudaDeviceSynchronize();
  return e;
}
#endif
}  // namespace ngpulm
