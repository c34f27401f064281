// NGPU-LM hot path for sm_100a: batched full-vocabulary query (Algorithm 1,
// PAPER.md:54-89) and the fused greedy shallow-fusion step.
//
// Design: one CTA per batch row, 256 threads.
//  1. one thread walks the row's back-off chain (Algorithm 1 lines 72, 81-82):
//     one 16-byte StateRec per level, acc_boff accumulated left to right in
//     float (R10); the root is never loaded (its arcs are [0, V)).
//  2. all threads scatter the non-root levels' arcs into shared memory: pass 1
//     takes, per token, the lowest level index with an arc (= the first level
//     Algorithm 1 would fill, lines 77-79) with a shared-memory atomicMin; pass
//     2 writes that level's acc + weight and target.
//  3. the root level is dense: every remaining token takes
//     acc_root + root_w[v] and root_to[v]; the row leaves in 16-byte streaming
//     stores (advance) or feeds a warp-shuffle argmax (fused step), so the LM
//     row of the fused step never touches HBM.
// No tensor cores: this is gather/scatter + store bandwidth.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <cmath>

#include "ngpulm_internal.h"

namespace ngpulm {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxL = NGPULM_MAX_ORDER;
constexpr uint32_t kNone = 0xFFFFFFFFu;

struct RowCtl {
  int32_t beg[kMaxL];      // first arc of level i
  int32_t pre[kMaxL + 1];  // prefix count of arcs over levels
  float acc[kMaxL];        // acc_boff when level i is visited
  float acc_root;          // acc_boff at the root level
  float fin;               // final weight of the row's state (AED)
  int32_t nlev;            // non-root levels
  int32_t bad;             // invalid state id / corrupted chain
  int32_t state;
  int32_t prevc;           // CTC: previous frame's column
};

// Algorithm 1 lines 67-82 for one row, serial by nature (pointer chase).
__device__ __forceinline__ void walk_chain(const DevModel& m, int32_t s, RowCtl& c) {
  c.state = s;
  c.acc_root = 0.f;
  c.nlev = 0;
  c.pre[0] = 0;
  if (s < 0 || s >= m.S) { c.bad = 1; return; }
  float acc = 0.f;
  int32_t n = 0, pre = 0;
  const int4* rec = reinterpret_cast<const int4*>(m.srec);
  for (; n < kMaxL && s != 0; ++n) {
    const int4 r = __ldg(rec + s);  // {arc_begin, arc_end, boff_to, boff_w}
    c.beg[n] = r.x;
    c.pre[n] = pre;
    c.acc[n] = acc;
    pre += r.y - r.x;
    acc = __fadd_rn(acc, __int_as_float(r.w));  // acc_boff += boff_weights[state]
    s = r.z;                                     // state = boff_to_states[state]
  }
  c.pre[n] = pre;
  c.nlev = n;
  c.acc_root = acc;
  c.bad = (s != 0) ? 2 : 0;
}

// Non-root levels -> shared-memory overrides; first (highest-order) level wins.
__device__ __forceinline__ void scatter_levels(const DevModel& m, const RowCtl& c, uint32_t* lvl,
                                               float* ovr_s, int32_t* ovr_n) {
  const int32_t T = c.pre[c.nlev];
  for (int32_t j = threadIdx.x; j < T; j += kThreads) {
    int L = 0;
    while (j >= c.pre[L + 1]) ++L;
    const int32_t a = c.beg[L] + (j - c.pre[L]);
    atomicMin(&lvl[__ldg(&m.arc_tok[a])], (uint32_t)L);
  }
  __syncthreads();
  for (int32_t j = threadIdx.x; j < T; j += kThreads) {
    int L = 0;
    while (j >= c.pre[L + 1]) ++L;
    const int32_t a = c.beg[L] + (j - c.pre[L]);
    const int32_t tok = __ldg(&m.arc_tok[a]);
    if (lvl[tok] == (uint32_t)L) {
      ovr_s[tok] = __fadd_rn(c.acc[L], __ldg(&m.arc_w[a]));  // acc_boff + arc_weights
      ovr_n[tok] = __ldg(&m.arc_to[a]);
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void init_lvl(uint32_t* lvl, int32_t V) {
  for (int32_t v = threadIdx.x; v < V; v += kThreads) lvl[v] = kNone;
}

// ---------------------------------------------------------------- advance
template <bool kVec4>
__global__ void __launch_bounds__(kThreads) advance_kernel(DevModel m, const int32_t* __restrict__ states,
                                                           float* __restrict__ scores,
                                                           int32_t* __restrict__ next,
                                                           float* __restrict__ final_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int32_t V = m.V;
  uint32_t* lvl = reinterpret_cast<uint32_t*>(smem);
  float* ovr_s = reinterpret_cast<float*>(lvl + V);
  int32_t* ovr_n = reinterpret_cast<int32_t*>(ovr_s + V);
  __shared__ RowCtl c;
  const int32_t b = blockIdx.x;
  if (threadIdx.x == 0) {
    walk_chain(m, __ldg(&states[b]), c);
    if (c.bad) atomicMin(m.bad_row, (unsigned long long)b);
    if (final_out) final_out[b] = c.bad ? __int_as_float(0x7fc00000) : __ldg(&m.final_w[c.state]);
  }
  init_lvl(lvl, V);
  __syncthreads();
  float* srow = scores + (size_t)b * V;
  int32_t* nrow = next + (size_t)b * V;
  if (c.bad) {
    for (int32_t v = threadIdx.x; v < V; v += kThreads) { srow[v] = __int_as_float(0x7fc00000); nrow[v] = -1; }
    return;
  }
  scatter_levels(m, c, lvl, ovr_s, ovr_n);
  const float acc_root = c.acc_root;
  if (kVec4) {
    const float4* rw4 = reinterpret_cast<const float4*>(m.arc_w);  // root arcs = [0, V)
    const int4* rt4 = reinterpret_cast<const int4*>(m.arc_to);
    for (int32_t q = threadIdx.x; q < V / 4; q += kThreads) {
      const uint4 l = reinterpret_cast<const uint4*>(lvl)[q];
      const float4 rw = __ldg(rw4 + q);
      const int4 rt = __ldg(rt4 + q);
      const int32_t v = q * 4;
      float4 o;
      int4 n;
      o.x = l.x != kNone ? ovr_s[v + 0] : __fadd_rn(acc_root, rw.x);
      o.y = l.y != kNone ? ovr_s[v + 1] : __fadd_rn(acc_root, rw.y);
      o.z = l.z != kNone ? ovr_s[v + 2] : __fadd_rn(acc_root, rw.z);
      o.w = l.w != kNone ? ovr_s[v + 3] : __fadd_rn(acc_root, rw.w);
      n.x = l.x != kNone ? ovr_n[v + 0] : rt.x;
      n.y = l.y != kNone ? ovr_n[v + 1] : rt.y;
      n.z = l.z != kNone ? ovr_n[v + 2] : rt.z;
      n.w = l.w != kNone ? ovr_n[v + 3] : rt.w;
      __stcs(reinterpret_cast<float4*>(srow) + q, o);
      __stcs(reinterpret_cast<int4*>(nrow) + q, n);
    }
  } else {
    for (int32_t v = threadIdx.x; v < V; v += kThreads) {
      const bool hit = lvl[v] != kNone;
      __stcs(srow + v, hit ? ovr_s[v] : __fadd_rn(acc_root, __ldg(&m.arc_w[v])));
      __stcs(nrow + v, hit ? ovr_n[v] : __ldg(&m.arc_to[v]));
    }
  }
}

// ---------------------------------------------------------------- final
__global__ void final_kernel(DevModel m, const int32_t* __restrict__ states, int32_t B,
                             float* __restrict__ out) {
  const int32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int32_t s = __ldg(&states[b]);
  if (s < 0 || s >= m.S) {
    out[b] = __int_as_float(0x7fc00000);
    atomicMin(m.bad_row, (unsigned long long)b);
    return;
  }
  out[b] = __ldg(&m.final_w[s]);
}

// ---------------------------------------------------------------- fused greedy step
// (value, column) order: larger value first, then lower column (R14).
__device__ __forceinline__ bool better(float v2, int32_t c2, float v, int32_t c) {
  return v2 > v || (v2 == v && c2 < c);
}

__device__ __forceinline__ void block_argmax(float& v, int32_t& c, float* sv, int32_t* sc) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int32_t c2 = __shfl_xor_sync(0xffffffffu, c, o);
    if (better(v2, c2, v, c)) { v = v2; c = c2; }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { sv[warp] = v; sc[warp] = c; }
  __syncthreads();
  if (warp == 0) {
    v = lane < kWarps ? sv[lane] : -INFINITY;
    c = lane < kWarps ? sc[lane] : INT_MAX;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float v2 = __shfl_xor_sync(0xffffffffu, v, o);
      const int32_t c2 = __shfl_xor_sync(0xffffffffu, c, o);
      if (better(v2, c2, v, c)) { v = v2; c = c2; }
    }
    if (lane == 0) { sv[kWarps] = v; sc[kWarps] = c; }
  }
  __syncthreads();
  v = sv[kWarps];
  c = sc[kWarps];
}

template <int kMode>
__global__ void __launch_bounds__(kThreads) fused_kernel(DevModel m, const float* __restrict__ logits,
                                                         int64_t row_stride, int32_t* __restrict__ states,
                                                         int32_t* __restrict__ prev,
                                                         const uint8_t* __restrict__ active, float lambda,
                                                         int32_t sp, int32_t* __restrict__ tokens_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int32_t V = m.V, ncols = V + 1;
  uint32_t* lvl = reinterpret_cast<uint32_t*>(smem);
  float* ovr_s = reinterpret_cast<float*>(lvl + V);
  int32_t* ovr_n = reinterpret_cast<int32_t*>(ovr_s + V);
  __shared__ RowCtl c;
  __shared__ float sv[kWarps + 1];
  __shared__ int32_t sc[kWarps + 1];
  const int32_t b = blockIdx.x;
  if (active && !__ldg(&active[b])) {
    if (threadIdx.x == 0) tokens_out[b] = -1;
    return;
  }
  const float* row = logits + (size_t)b * row_stride;
  if (threadIdx.x == 0) {
    walk_chain(m, states[b], c);
    if (c.bad) atomicMin(m.bad_row, (unsigned long long)b);
    if (kMode == NGPULM_CTC) c.prevc = prev[b];
    if (kMode == NGPULM_AED) c.fin = c.bad ? 0.f : __ldg(&m.final_w[c.state]);
  }
  init_lvl(lvl, V);
  if (kMode == NGPULM_RNNT) {
    // stage 1: standard greedy prediction over all V+1 columns
    float bv = -INFINITY;
    int32_t bc = INT_MAX;
    for (int32_t col = threadIdx.x; col < ncols; col += kThreads) {
      const float a = __ldg(&row[col]);
      if (better(a, col, bv, bc)) { bv = a; bc = col; }
    }
    block_argmax(bv, bc, sv, sc);  // includes __syncthreads: c is visible after it
    if (c.bad) {
      if (threadIdx.x == 0) tokens_out[b] = -1;
      return;
    }
    if (bc == sp) {                // blank is retained: no LM work, state unchanged
      if (threadIdx.x == 0) tokens_out[b] = sp;
      return;
    }
  } else {
    __syncthreads();
    if (c.bad) {
      if (threadIdx.x == 0) tokens_out[b] = -1;
      return;
    }
  }
  scatter_levels(m, c, lvl, ovr_s, ovr_n);
  const float acc_root = c.acc_root;
  const int32_t pc = (kMode == NGPULM_CTC) ? c.prevc : -2;
  float bv = -INFINITY;
  int32_t bc = INT_MAX;
  for (int32_t col = threadIdx.x; col < ncols; col += kThreads) {
    const float a = __ldg(&row[col]);
    float val;
    if (col == sp) {
      if (kMode == NGPULM_RNNT) continue;                  // stage 2: non-blank only
      val = (kMode == NGPULM_AED) ? __fmaf_rn(lambda, c.fin, a) : a;  // eos <-> final / blank raw
    } else if (kMode == NGPULM_CTC && col == pc) {
      val = a;                                             // repeated token: not rescored
    } else {
      const int32_t v = col < sp ? col : col - 1;
      const float lm = lvl[v] != kNone ? ovr_s[v] : __fadd_rn(acc_root, __ldg(&m.arc_w[v]));
      val = __fmaf_rn(lambda, lm, a);                      // asr + lambda * lm, one rounding
    }
    if (better(val, col, bv, bc)) { bv = val; bc = col; }
  }
  block_argmax(bv, bc, sv, sc);
  if (threadIdx.x == 0) {
    if (bc < 0 || bc >= ncols) { tokens_out[b] = -1; return; }  // all-NaN row (unspecified)
    tokens_out[b] = bc;
    if (bc == sp) {
      if (kMode == NGPULM_CTC) prev[b] = -1;
      return;
    }
    if (kMode == NGPULM_CTC && bc == pc) return;            // collapsed: no LM advance
    const int32_t v = bc < sp ? bc : bc - 1;
    states[b] = lvl[v] != kNone ? ovr_n[v] : __ldg(&m.arc_to[v]);
    if (kMode == NGPULM_CTC) prev[b] = bc;
  }
}

size_t row_smem(int32_t V) { return (size_t)V * 12; }

int set_smem(const void* fn, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  return (int)cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace

int max_vocab_supported() {
  return (int)((227 * 1024 - (int)sizeof(RowCtl) - 2 * 64) / 12) & ~3;
}

int launch_advance(const DevModel& m, const int32_t* states, int32_t B, float* scores, int32_t* next,
                   float* final_out, void* stream) {
  const size_t sm = row_smem(m.V);
  const bool vec = (m.V % 4 == 0) && ((uintptr_t)scores % 16 == 0) && ((uintptr_t)next % 16 == 0);
  cudaStream_t st = (cudaStream_t)stream;
  if (vec) {
    if (int e = set_smem((const void*)advance_kernel<true>, sm)) return e;
    advance_kernel<true><<<B, kThreads, sm, st>>>(m, states, scores, next, final_out);
  } else {
    if (int e = set_smem((const void*)advance_kernel<false>, sm)) return e;
    advance_kernel<false><<<B, kThreads, sm, st>>>(m, states, scores, next, final_out);
  }
  return (int)cudaGetLastError();
}

int launch_final(const DevModel& m, const int32_t* states, int32_t B, float* out, void* stream) {
  final_kernel<<<(B + 255) / 256, 256, 0, (cudaStream_t)stream>>>(m, states, B, out);
  return (int)cudaGetLastError();
}

int launch_fused(const DevModel& m, int32_t mode, const float* logits, int64_t row_stride, int32_t B,
                 int32_t* states, int32_t* prev, const uint8_t* active, float lambda, int32_t blank,
                 int32_t* tokens_out, void* stream) {
  const size_t sm = row_smem(m.V);
  cudaStream_t st = (cudaStream_t)stream;
  switch (mode) {
    case NGPULM_CTC:
      if (int e = set_smem((const void*)fused_kernel<NGPULM_CTC>, sm)) return e;
      fused_kernel<NGPULM_CTC><<<B, kThreads, sm, st>>>(m, logits, row_stride, states, prev, active, lambda,
                                                        blank, tokens_out);
      break;
    case NGPULM_RNNT:
      if (int e = set_smem((const void*)fused_kernel<NGPULM_RNNT>, sm)) return e;
      fused_kernel<NGPULM_RNNT><<<B, kThreads, sm, st>>>(m, logits, row_stride, states, prev, active, lambda,
                                                         blank, tokens_out);
      break;
    default:
      if (int e = set_smem((const void*)fused_kernel<NGPULM_AED>, sm)) return e;
      fused_kernel<NGPULM_AED><<<B, kThreads, sm, st>>>(m, logits, row_stride, states, prev, active, lambda,
                                                        blank, tokens_out);
      break;
  }
  return (int)cudaGetLastError();
}

}  // namespace ngpulm
