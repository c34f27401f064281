// Whole-utterance greedy CTC decoding with shallow fusion in one launch
// for sm_100a, and its launcher.
#include "kcommon.cuh"

namespace ngpulm {
namespace {

// ---------------------------------------------------------------- persistent CTC decode
// One launch decodes whole utterances: T fused CTC steps per
// row, identical to T launches of the fused step with active = (t < len).
// Two warps per row, warp-specialised:
//  * the consumer warp decides the frames. The row's LM scores are rebuilt in
//    shared memory only when its state changes (an emission: blanks and
//    repeats do not advance the LM) and are cached in registers
//    (lane i: columns i, i+32, ...) across the frames in between;
//  * the producer warp streams the row's frames through a ring of
//    shared-memory buffers ahead of the consumer: the aligned interior of a
//    frame by one bulk copy (TMA, L2 evict-first: logits are read once, the
//    trie should stay in L2), the <= 3 columns on each side by 4-byte
//    cp.async, all tracked by the slot's "full" mbarrier; the consumer frees a
//    slot through its "empty" mbarrier.
constexpr int kRingMax = 8;

__host__ __device__ constexpr size_t lbuf_bytes(int32_t V) { return align16((size_t)(V + 1) * 4 + 16); }
// per row: row_s | row_n | levels | 2 mbarriers | full [kRingMax] | empty [kRingMax] | ring buffers [depth]
__host__ __device__ constexpr size_t dslice_bytes(int32_t V, int32_t order, int depth) {
  return wslice_bytes(V, order, 0) + 2 * kRingMax * 8 + (size_t)depth * lbuf_bytes(V);
}
// CTA: root weights [V] | root targets [V] | mbarrier | R slices
__host__ __device__ constexpr size_t dcta_smem(int32_t V, int32_t order, int R, int depth) {
  return 2 * align16((size_t)V * 4) + 16 + (size_t)R * dslice_bytes(V, order, depth);
}

// The row of state `st` into s.row_s / s.row_n (Algorithm 1, as in
// advance_warp_kernel), root level from the CTA's shared copies. Returns the
// row scalars (r.bad: invalid state, nothing written).
struct NoStamp {
  __device__ void operator()(int) const {}
};

template <bool kTable, bool kPacked, typename F = NoStamp>
__device__ __forceinline__ Row build_row_warp(const DevModel& m, const WSlice& s, const float* root_w,
                                              const int32_t* root_to, int32_t st, F stamp = F()) {
  constexpr int kW = 8;
  const int lane = threadIdx.x & 31;
  WLevel lv;
  int32_t nslots;
  const Row r = warp_row_src<kTable>(m, ValState{st}, s, lv, nslots);
  stamp(1);
  if (r.bad) return r;
  Window<kW, kPacked> a;
  load_window<kW, kPacked>(m, s, lv, r.nlev, 0, nslots, a);
  {  // root level while the gathers fly: acc_root + root weight, root targets
    const float4* w4 = reinterpret_cast<const float4*>(root_w);
    const int4* t4 = reinterpret_cast<const int4*>(root_to);
    float4* s4 = reinterpret_cast<float4*>(s.row_s);
    int4* n4 = reinterpret_cast<int4*>(s.row_n);
    const float ar = r.acc_root;
    for (int32_t q = lane; q < m.V / 4; q += 32) {
      float4 y = w4[q];
      y.x = __fadd_rn(ar, y.x);
      y.y = __fadd_rn(ar, y.y);
      y.z = __fadd_rn(ar, y.z);
      y.w = __fadd_rn(ar, y.w);
      s4[q] = y;
      n4[q] = t4[q];
    }
  }
  __syncwarp();
  stamp(7);
  for (int32_t k0 = 0; k0 < nslots;) {
    write_window<kW, kPacked>(s, a, k0, nslots, m.pk_bits);
    k0 += kW;
    if (k0 < nslots) load_window<kW, kPacked>(m, s, lv, r.nlev, k0, nslots, a);
  }
  __syncwarp();
  stamp(8);
  return r;
}

constexpr int kDecodeMaxRows = 4;  // rows per CTA (2 warps each): 256 threads, up to 255 registers

template <bool kTable, bool kPacked, bool kNoLM = false>
__global__ void __launch_bounds__(64 * kDecodeMaxRows, 1)
    ctc_decode_kernel(DevModel m, const float* __restrict__ logits, int64_t row_stride, int64_t frame_stride,
                      int32_t B, int32_t T, const int32_t* __restrict__ lengths, int32_t* __restrict__ states,
                      int32_t* __restrict__ prev, float lambda, int32_t sp, int32_t depth,
                      int32_t* __restrict__ frames_out, int32_t* __restrict__ emit_out,
                      int32_t* __restrict__ emit_len) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int32_t V = m.V, ncols = V + 1;
  const int lane = threadIdx.x & 31, R = blockDim.x >> 6;  // R consumer warps, then R producer warps
  const int wid = threadIdx.x >> 5, w = wid % R;
  const bool producer = wid >= R;
  const size_t rb = align16((size_t)V * 4);
  float* root_w = reinterpret_cast<float*>(smem);
  int32_t* root_to = reinterpret_cast<int32_t*>(smem + rb);
  uint64_t* cbar = reinterpret_cast<uint64_t*>(smem + 2 * rb);
  unsigned char* base = smem + 2 * rb + 16 + (size_t)w * dslice_bytes(V, m.order, depth);
  const WSlice s = wcarve(base, V, m.order, 0);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + wslice_bytes(V, m.order, 0));
  uint64_t* empty = full + kRingMax;
  float* ring = reinterpret_cast<float*>(base + wslice_bytes(V, m.order, 0) + 2 * kRingMax * 8);
  const size_t lstride = lbuf_bytes(V) / 4;
  const int32_t row = (int32_t)blockIdx.x * R + w;
  pdl_trigger();
  // the root level once per CTA (immutable model data: before the wait)
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(cbar)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(cbar)), "r"((uint32_t)V * 8u)
                 : "memory");
    bulk_g2s(root_w, m.arc_w, (uint32_t)V * 4u, cbar);
    bulk_g2s(root_to, m.arc_to, (uint32_t)V * 4u, cbar);
  }
  if (!producer && lane == 0) {
    for (int i = 0; i < depth; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + i)) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(empty + i)) : "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();  // barrier inits visible to every warp
  pdl_wait();
  if (row >= B) {
    if (threadIdx.x == 0) mbar_wait(cbar, 0);  // no exit with the CTA's bulk copy in flight
    return;
  }
  int32_t len = T;
  if (lengths) len = min(T, max(0, __ldg(&lengths[row])));
  constexpr bool nolm = kNoLM;  // plain greedy CTC (no LM, states == nullptr): its own instantiation
  int32_t st = nolm ? 0 : __ldg(&states[row]);
  const bool bad = st < 0 || st >= m.S;
  const int32_t run = bad ? 0 : len;  // an invalid state decides nothing (token -1 every frame)
  const float* lrow0 = logits + (size_t)row * row_stride;
  if (producer) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    int32_t slot = 0;
    uint32_t phase = 0;  // parity of the slot's previous use
    for (int32_t t = 0; t < run; ++t) {
      if (t >= depth) mbar_wait(empty + slot, phase);  // the consumer is done with frame t - depth
      issue_frame(lrow0 + (size_t)t * frame_stride, ncols, ring + (size_t)slot * lstride, full + slot, pol);
      if (++slot == depth) { slot = 0; if (t >= depth) phase ^= 1u; }
    }
    if (threadIdx.x == R * 32) mbar_wait(cbar, 0);
    return;
  }
  int32_t pc = __ldg(&prev[row]);
  int32_t* fout = frames_out ? frames_out + (size_t)row * T : nullptr;
  int32_t* eout = emit_out ? emit_out + (size_t)row * T : nullptr;
  if (bad && len > 0 && lane == 0) atomicMin(m.bad_row, (unsigned long long)row);
  mbar_wait(cbar, 0);
#ifdef NGPULM_PHASE_TIMING
  // debug build: cycles per phase, per row: 0 first build, 1 rebuild: record,
  // 2 logits wait, 3 decide, 4 rebuild: LM registers, 5 rebuild count,
  // 6 frames, 7 rebuild: gathers + root, 8 rebuild: writes, 9 SM id
  long long ck[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long c0 = clock64(), c1;
#define DSTAMP(i) do { c1 = clock64(); ck[i] += c1 - c0; c0 = c1; } while (0)
  auto stamp = [&](int i) { DSTAMP(i); };
#else
#define DSTAMP(i) do { } while (0)
  NoStamp stamp;
#endif
  float lm[kMaxColsPerLane];
  auto rebuild = [&](int32_t state) {
    if (nolm) {
#pragma unroll
      for (int j = 0; j < kMaxColsPerLane; ++j) lm[j] = 0.f;
      return;
    }
    build_row_warp<kTable, kPacked>(m, s, root_w, root_to, state, stamp);
#pragma unroll
    for (int j = 0; j < kMaxColsPerLane; ++j) {
      const int32_t col = lane + 32 * j;
      lm[j] = (col < ncols && col != sp) ? s.row_s[col - (col > sp)] : 0.f;  // blank: 0 (fused value = asr)
    }
  };
  if (run > 0) rebuild(st);
  DSTAMP(0);
  int32_t nemit = 0;
  int32_t slot = 0;
  uint32_t phase = 0;
  const float* lrow = lrow0;
  for (int32_t t = 0; t < run; ++t, lrow += frame_stride) {
    mbar_wait(full + slot, phase);
    DSTAMP(2);
    const float* buf = ring + (size_t)slot * lstride;
    const int32_t h = (int32_t)((reinterpret_cast<uintptr_t>(lrow) & 15) / 4);
    // fused values (R13, R19): prev column raw, every other column
    // fmaf(lambda, lm, asr) — the blank column too, with lm = 0 there, which
    // is exactly asr for finite lambda. Argmax (R14) in two passes: the
    // largest value (NaN ignored), then the lowest column holding it.
    float val[kMaxColsPerLane], mx[kMaxColsPerLane];
    const float* bp = buf + h + lane;
#pragma unroll
    for (int j = 0; j < kMaxColsPerLane; ++j) {
      const int32_t col = lane + 32 * j;
      float x = __int_as_float(0x7fc00000);  // past the last column: NaN, never selected
      if (col < ncols) x = bp[32 * j];
      val[j] = col == pc ? x : __fmaf_rn(lambda, lm[j], x);
      mx[j] = val[j];
    }
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + slot)) : "memory");
    if (++slot == depth) { slot = 0; phase ^= 1u; }
#pragma unroll
    for (int d = 1; d < kMaxColsPerLane; d *= 2)
#pragma unroll
      for (int j = 0; j + d < kMaxColsPerLane; j += 2 * d) mx[j] = fmaxf(mx[j], mx[j + d]);
    const float lmax = mx[0] == mx[0] ? mx[0] : -INFINITY;
    const uint32_t kmax = __reduce_max_sync(kFull, fkey(lmax));
    const float M = __uint_as_float((kmax & 0x80000000u) ? (kmax ^ 0x80000000u) : ~kmax);
    int32_t cm[kMaxColsPerLane];
#pragma unroll
    for (int j = 0; j < kMaxColsPerLane; ++j) cm[j] = val[j] == M ? lane + 32 * j : INT_MAX;
#pragma unroll
    for (int d = 1; d < kMaxColsPerLane; d *= 2)
#pragma unroll
      for (int j = 0; j + d < kMaxColsPerLane; j += 2 * d) cm[j] = min(cm[j], cm[j + d]);
    const int32_t bc = (int32_t)__reduce_min_sync(kFull, (uint32_t)cm[0]);
    int32_t tok = -1;
    bool moved = false;
    if (bc >= 0 && bc < ncols) {
      tok = bc;
      if (bc == sp) {
        pc = -1;
      } else if (bc != pc) {  // an emission: LM advance (a repeat of prev is collapsed)
        const int32_t ns = nolm ? 0 : s.row_n[bc < sp ? bc : bc - 1];
        if (lane == 0 && eout) eout[nemit] = bc;
        ++nemit;
        pc = bc;
        moved = ns != st;
        st = ns;
      }
    }
    if (lane == 0 && fout) fout[t] = tok;
    DSTAMP(3);
#ifdef NGPULM_PHASE_TIMING
    if (g_skip & 16) moved = false;
    ck[5] += moved;
    ck[6] += 1;
#endif
    if (moved) rebuild(st);
    DSTAMP(4);
  }
#ifdef NGPULM_PHASE_TIMING
  if (lane == 0 && row < 16384) {
    for (int i = 0; i < 9; ++i) g_phase[row * 16 + i] = (unsigned long long)ck[i];
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    g_phase[row * 16 + 9] = sm;
  }
#endif
#undef DSTAMP
  // frames past the row's length (and every frame of an invalid row): -1
  if (fout)
    for (int32_t t = run + lane; t < T; t += 32) fout[t] = -1;
  if (lane == 0) {
    if (!nolm) states[row] = st;
    prev[row] = pc;
    if (emit_len) emit_len[row] = nemit;
  }
}

}  // namespace

int launch_ctc_decode(const DevModel& m, const float* logits, int64_t row_stride, int64_t frame_stride, int32_t B,
                      int32_t T, const int32_t* lengths, int32_t* states, int32_t* prev, float lambda, int32_t blank,
                      int32_t* frames_out, int32_t* emit_out, int32_t* emit_len, void* stream) {
  if (m.V % 4 != 0 || m.V > 1024) return (int)cudaErrorNotSupported;
  int R = (B + 147) / 148;
  R = R < 1 ? 1 : (R > kDecodeMaxRows ? kDecodeMaxRows : R);
  int depth = kRingMax;
  while (depth > 2 && dcta_smem(m.V, m.order, R, depth) > 227 * 1024) --depth;
  while (R > 1 && dcta_smem(m.V, m.order, R, depth) > 227 * 1024) --R;
  const size_t sm = dcta_smem(m.V, m.order, R, depth);
  const dim3 g((B + R - 1) / R), b(64 * R);
  const bool pk = m.arc_q != nullptr && m.adv_kind == NGPULM_ADVANCE_AUTO, table = m.chain != nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  if (states == nullptr)
    return launch(ctc_decode_kernel<true, true, true>, g, b, sm, st, m, logits, row_stride, frame_stride, B, T,
                  lengths, states, prev, lambda, blank, depth, frames_out, emit_out, emit_len);
#define NGPULM_DECODE_LAUNCH(TB, P)                                                                                  \
  return launch(ctc_decode_kernel<TB, P>, g, b, sm, st, m, logits, row_stride, frame_stride, B, T, lengths, states, \
                prev, lambda, blank, depth, frames_out, emit_out, emit_len)
  if (table) { if (pk) NGPULM_DECODE_LAUNCH(true, true); NGPULM_DECODE_LAUNCH(true, false); }
  if (pk) NGPULM_DECODE_LAUNCH(false, true);
  NGPULM_DECODE_LAUNCH(false, false);
#undef NGPULM_DECODE_LAUNCH
}

}  // namespace ngpulm
