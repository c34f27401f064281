// Debug build (NGPULM_PHASE_TIMING): all kernels in one translation unit, so the
// phase-stamp buffer (g_phase, kcommon.cuh) is one object for every kernel.
#include "advance.cu"
#include "decode.cu"
#include "fused.cu"
#include "debug.cu"
