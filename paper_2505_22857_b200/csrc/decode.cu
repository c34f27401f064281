// Whole-utterance greedy CTC decoding with shallow fusion in one launch
// for sm_100a, and its launcher.
#include <cfloat>

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

// a frame slot: V+1 columns + the slack of a 16-byte-aligned cover (issue_frame_cover)
__host__ __device__ constexpr size_t lbuf_bytes(int32_t V) { return align16((size_t)(V + 1) * 4 + 32); }
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

template <bool kTable, bool kPacked, typename F = NoStamp, bool kTiny = false>
__device__ __forceinline__ Row build_row_warp(const DevModel& m, const WSlice& s, const float* root_w,
                                              const int32_t* root_to, int32_t st, F stamp = F()) {
  constexpr int kW = 8;
  const int lane = threadIdx.x & 31;
  WLevel lv;
  int32_t nslots;
  const Row r = warp_row_src<kTable, NoOp, ValState, kTiny>(m, ValState{st}, s, lv, nslots);
  stamp(1);
  if (r.bad) return r;
  Window<kW, kPacked> a;
  load_window<kW, kPacked, kTiny>(m, s, lv, r.nlev, 0, nslots, a);
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
    if (k0 < nslots) load_window<kW, kPacked, kTiny>(m, s, lv, r.nlev, k0, nslots, a);
  }
  __syncwarp();
  stamp(8);
  return r;
}

constexpr int kDecodeMaxRows = 4;  // rows per CTA (2 warps each): 256 threads, up to 255 registers

template <bool kTable, bool kPacked, bool kNoLM = false, bool kTiny = false>
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
  unsigned char* sm0 = smem + (kTiny ? tiny_copy_bytes(m.tiny_chain_bytes, m.tiny_arcq_bytes) : 0);
  float* root_w = reinterpret_cast<float*>(sm0);
  int32_t* root_to = reinterpret_cast<int32_t*>(sm0 + rb);
  uint64_t* cbar = reinterpret_cast<uint64_t*>(sm0 + 2 * rb);
  unsigned char* base = sm0 + 2 * rb + 16 + (size_t)w * dslice_bytes(V, m.order, depth);
  WSlice s = wcarve(base, V, m.order, 0);
  if (kTiny) {  // the tiny LM resident in the CTA's shared memory (tiny_copy_issue)
    s.chain_s = reinterpret_cast<const int4*>(smem);
    s.st_q = reinterpret_cast<int4*>(smem + align16((size_t)m.tiny_chain_bytes));
  }
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
    if (kTiny) tiny_copy_issue(m, smem);
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
    if (threadIdx.x == 0) {  // no exit with the CTA's bulk copies in flight
      mbar_wait(cbar, 0);
      if (kTiny) mbar_wait(tiny_bar(smem, m), 0);
    }
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
      issue_frame_cover(lrow0 + (size_t)t * frame_stride, ncols, ring + (size_t)slot * lstride, full + slot, pol, logits,
                        logits + (size_t)(B - 1) * row_stride + (size_t)(T - 1) * frame_stride + ncols);
      if (++slot == depth) { slot = 0; if (t >= depth) phase ^= 1u; }
    }
    cp_async_settle();
    if (threadIdx.x == R * 32) mbar_wait(cbar, 0);
    return;
  }
  int32_t pc = __ldg(&prev[row]);
  int32_t* fout = frames_out ? frames_out + (size_t)row * T : nullptr;
  int32_t* eout = emit_out ? emit_out + (size_t)row * T : nullptr;
  if (bad && len > 0 && lane == 0) atomicMin(m.bad_row, (unsigned long long)row);
  mbar_wait(cbar, 0);
  if (kTiny) mbar_wait(tiny_bar(smem, m), 0);
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
    build_row_warp<kTable, kPacked, decltype(stamp), kTiny>(m, s, root_w, root_to, state, stamp);
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
    release_slot(empty + slot);
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

// ---------------------------------------------------------------- bound-pruned persistent CTC decode
// The same decisions as ctc_decode_kernel (T fused CTC steps, PAPER.md:139;
// R13, R14, R17, R19) without building the LM row and scanning all V+1
// columns after every emission. One CTA (2 + kSumWarps warps) per row:
//  * producer: streams the frames through a TMA ring (as ctc_decode_kernel);
//  * summary warps (frame t -> warp t % kSumWarps; frame-parallel, LM-free):
//    the blank column's raw value xb and the two largest raw token values
//    with their columns and the third value (x1 c1, x2 c2, x3);
//  * decider: walks the frames in order with the state s, its chain record,
//    ub(s) (load-time bound: every score of the row of s is <= ub(s)) and the
//    chain's arcs staged in shared memory by TMA (one bulk copy per level,
//    slot layout). For lambda >= 0 a token v has fused value
//    fmaf(lambda, lm, x[v]) <= fmaf(lambda, ub(s), x[v]) (monotone rounding),
//    so every token outside a candidate set C is below
//    fmaf(lambda, ub(s), largest raw value outside C).
//    Level 0: C = {} (the repeated column pc, raw, and the blank, raw, are
//    exact): the better of them wins if it beats that bound strictly — no LM
//    value is needed. Level 1: C = {c1, c2}: their exact fused values from the
//    staged arcs (the highest-order level holding the token wins, Algorithm 1
//    lines 77-79; else the root level) against the bound with x3. Level 2
//    (no strict winner): the exact step of ctc_decode_kernel over the full
//    row, built in shared memory from the staged arcs and kept while the
//    state stays.
// Every decision is the full argmax's (tested bit-exact against the oracle
// and ctc_decode_kernel); plain greedy (states == nullptr) is the summaries'
// raw argmax.
#ifndef NGPULM_SUM_WARPS
#define NGPULM_SUM_WARPS 4
#endif
#ifndef NGPULM_DECODE_BOUND
#define NGPULM_DECODE_BOUND 0
#endif
constexpr int kSumWarps = NGPULM_SUM_WARPS;
constexpr int kStageSlots = 16;  // staged arc slots (32 quads each) per row; beyond: global gathers at level 2
constexpr int kRing2 = 8;        // frames in flight per row

struct FrameSum {  // per frame, LM-free (32 B)
  float xb, x1, x2, x3;
  int32_t c1, c2, pad0, pad1;  // columns of x1, x2 (-1: none)
};

__host__ __device__ constexpr size_t stage2_bytes(bool packed) { return (size_t)kStageSlots * 32 * (packed ? 32 : 48); }
// root_w | root_to | cbar | WSlice | full, empty, sfull [kRing2] | sbar | sums [kRing2] | ring [kRing2] | stage
__host__ __device__ constexpr size_t d2_smem(int32_t V, int32_t order, bool packed) {
  return 2 * align16((size_t)V * 4) + 16 + wslice_bytes(V, order, 0) + 3 * kRing2 * 8 + 16 +
         kRing2 * sizeof(FrameSum) + (size_t)kRing2 * lbuf_bytes(V) + stage2_bytes(packed);
}

__device__ __forceinline__ float unkey(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k ^ 0x80000000u) : ~k);
}
// NaN: 0, below every value; -0 and +0 share a key
__device__ __forceinline__ uint32_t nkey(float v) { return v == v ? fkey(v + 0.0f) : 0u; }

// The two largest values of a row held in registers (lane i: columns i + 32 j;
// NaN never taken) with their columns (lowest column among equal values; -1:
// none) and the third value (-inf: none): three rounds of a lane max tree and
// a warp max, the winning column dropped after each.
__device__ __forceinline__ void top2(float (&v)[kMaxColsPerLane], float& M1, int32_t& C1, float& M2, int32_t& C2,
                                     float& M3) {
  const int lane = threadIdx.x & 31;
#pragma unroll 1
  for (int r = 0; r < 3; ++r) {
    float t[kMaxColsPerLane];
#pragma unroll
    for (int j = 0; j < kMaxColsPerLane; ++j) t[j] = v[j];
#pragma unroll
    for (int d = 1; d < kMaxColsPerLane; d *= 2)
#pragma unroll
      for (int j = 0; j + d < kMaxColsPerLane; j += 2 * d) t[j] = fmaxf(t[j], t[j + d]);
    const uint32_t K = __reduce_max_sync(kFull, nkey(t[0]));
    const float M = K ? unkey(K) : -INFINITY;
    if (r == 2) { M3 = M; break; }
    uint32_t cm = 0xffffffffu;
#pragma unroll
    for (int j = kMaxColsPerLane - 1; j >= 0; --j) cm = (K && v[j] == M) ? (uint32_t)(lane + 32 * j) : cm;
    const int32_t C = (int32_t)__reduce_min_sync(kFull, cm);
    if (r == 0) { M1 = M; C1 = C; } else { M2 = M; C2 = C; }
#pragma unroll
    for (int j = 0; j < kMaxColsPerLane; ++j) v[j] = lane + 32 * j == C ? __int_as_float(0x7fc00000) : v[j];
  }
}

template <bool kPacked, bool kNoLM>
__global__ void __launch_bounds__(32 * (2 + kSumWarps), 2)
    ctc_decode2_kernel(DevModel m, const float* __restrict__ logits, int64_t row_stride, int64_t frame_stride,
                       int32_t B, int32_t T, const int32_t* __restrict__ lengths, int32_t* __restrict__ states,
                       int32_t* __restrict__ prev, float lambda, int32_t sp, int32_t* __restrict__ frames_out,
                       int32_t* __restrict__ emit_out, int32_t* __restrict__ emit_len) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int32_t V = m.V, ncols = V + 1;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;  // 0 decider, 1 producer, 2.. summaries
  const size_t rb = align16((size_t)V * 4);
  float* root_w = reinterpret_cast<float*>(smem);
  int32_t* root_to = reinterpret_cast<int32_t*>(smem + rb);
  uint64_t* cbar = reinterpret_cast<uint64_t*>(smem + 2 * rb);
  unsigned char* p = smem + 2 * rb + 16;
  const WSlice s = wcarve(p, V, m.order, 0);
  p += wslice_bytes(V, m.order, 0);
  uint64_t* full = reinterpret_cast<uint64_t*>(p);
  uint64_t* empty = full + kRing2;
  uint64_t* sfull = empty + kRing2;
  uint64_t* sbar = sfull + kRing2;
  p += 3 * kRing2 * 8 + 16;
  FrameSum* sums = reinterpret_cast<FrameSum*>(p);
  p += kRing2 * sizeof(FrameSum);
  float* ring = reinterpret_cast<float*>(p);
  const size_t lstride = lbuf_bytes(V) / 4;
  p += (size_t)kRing2 * lbuf_bytes(V);
  unsigned char* stage = p;
  constexpr int kSQ = kStageSlots * 32;  // staged quads
  const int32_t row = (int32_t)blockIdx.x;
  pdl_trigger();
  if (threadIdx.x == 0) {  // root level (immutable model data: before the wait) and the barriers
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(cbar)) : "memory");
    for (int i = 0; i < kRing2; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + i)) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(smem_u32(empty + i)) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(sfull + i)) : "memory");
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(sbar)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(cbar)), "r"((uint32_t)V * 8u)
                 : "memory");
    bulk_g2s(root_w, m.arc_w, (uint32_t)V * 4u, cbar);
    bulk_g2s(root_to, m.arc_to, (uint32_t)V * 4u, cbar);
  }
  __syncthreads();
  pdl_wait();
  int32_t len = T;
  if (lengths) len = min(T, max(0, __ldg(&lengths[row])));
  int32_t st = kNoLM ? 0 : __ldg(&states[row]);
  const bool bad = st < 0 || st >= m.S;
  const int32_t run = bad ? 0 : len;
  const float* lrow0 = logits + (size_t)row * row_stride;
  auto frame_buf = [&](int32_t t) {  // column c of frame t at [c]
    const float* lrow = lrow0 + (size_t)t * frame_stride;
    return ring + (size_t)(t % kRing2) * lstride + (reinterpret_cast<uintptr_t>(lrow) & 15) / 4;
  };
  if (wid == 1) {  // ---- producer
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (int32_t t = 0; t < run; ++t) {
      const int32_t slot = t % kRing2;
      if (t >= kRing2) mbar_wait(empty + slot, (uint32_t)(t / kRing2 - 1) & 1u);
      issue_frame_cover(lrow0 + (size_t)t * frame_stride, ncols, ring + (size_t)slot * lstride, full + slot, pol, logits,
                        logits + (size_t)(B - 1) * row_stride + (size_t)(T - 1) * frame_stride + ncols);
    }
    cp_async_settle();
    return;
  }
  mbar_wait(cbar, 0);
  if (wid >= 2) {  // ---- summary warps
    for (int32_t t = wid - 2; t < run; t += kSumWarps) {
      const int32_t slot = t % kRing2;
      mbar_wait(full + slot, (uint32_t)(t / kRing2) & 1u);
      const float* fb = frame_buf(t);
      float v[kMaxColsPerLane];
#pragma unroll
      for (int j = 0; j < kMaxColsPerLane; ++j) {
        const int32_t col = lane + 32 * j;
        v[j] = (col < ncols && col != sp) ? fb[col] : __int_as_float(0x7fc00000);
      }
      float x1, x2, x3;
      int32_t c1, c2;
      top2(v, x1, c1, x2, c2, x3);
      if (lane == 0) {
        float4* d4 = reinterpret_cast<float4*>(sums + slot);
        d4[0] = make_float4(fb[sp], x1, x2, x3);
        d4[1] = make_float4(__int_as_float(c1), __int_as_float(c2), 0.f, 0.f);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(sfull + slot)) : "memory");
      }
      release_slot(empty + slot);
    }
    return;
  }
  // ---- decider
  int32_t pc = __ldg(&prev[row]);
  int32_t* fout = frames_out ? frames_out + (size_t)row * T : nullptr;
  int32_t* eout = emit_out ? emit_out + (size_t)row * T : nullptr;
  if (bad && len > 0 && lane == 0) atomicMin(m.bad_row, (unsigned long long)row);
  WLevel lv;
  int32_t nslots = 0, nlev = 0, row_state = -1;
  float acc_root = 0.f, ub = 0.f;
  bool staged = false, spend = false;
  uint32_t nst = 0;  // stagings issued
  auto stage_wait = [&]() {
    if (spend) { mbar_wait(sbar, (nst - 1u) & 1u); spend = false; }
  };
#ifdef NGPULM_PHASE_TIMING
  // debug build: per row 0 summary waits, 1 level 0, 2 lookups (incl. staging wait), 3 staging wait,
  // 4 level-2 builds, 5 level-2 argmax, 6 state loads, 7 output; counts 8 level0, 9 level1, 10 level2,
  // 11 builds, 12 state loads
  long long ck[13] = {0};
  long long tk0 = clock64(), tk1;
#define D2STAMP(i) do { tk1 = clock64(); ck[i] += tk1 - tk0; tk0 = tk1; } while (0)
#define D2COUNT(i) do { ck[i] += 1; } while (0)
#else
#define D2STAMP(i) do { } while (0)
#define D2COUNT(i) do { } while (0)
#endif
  const bool fast = !kNoLM && lambda >= 0.f && lambda <= FLT_MAX;
  bool need_state = !kNoLM && run > 0;
  int32_t nemit = 0;
  for (int32_t t = 0; t < run; ++t) {
    if (need_state) {  // the decider's view of st: chain record, ub(st), arcs staged by TMA
      need_state = false;
      float uv = 0.f;
      const Row r = warp_row_src<true>(m, ValState{st}, s, lv, nslots, [&] {
        if (lane == 0) uv = __ldg(m.lm_ub + st);
      });
      nlev = r.nlev;
      acc_root = r.acc_root;
      ub = __shfl_sync(kFull, uv, 0);
      staged = nslots <= kStageSlots;
      if (staged) {
        stage_wait();        // no copy for the previous state still landing
        proxy_fence_warp();  // the staging area's generic reads before the async overwrite
        const int32_t nq = (lane >= 1 && lane <= nlev) ? (lv.info & 0xffff) : 0;
        const uint32_t bytes = __reduce_add_sync(kFull, (uint32_t)nq * (kPacked ? 32u : 48u));
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(sbar)), "r"(bytes)
                       : "memory");
        __syncwarp();
        if (nq > 0) {
          const size_t q0 = (size_t)(lv.info >> 16) * 32;  // the level's first slot
          if (kPacked) {
            bulk_g2s(stage + q0 * 32, static_cast<const unsigned char*>(m.arc_q) + (size_t)lv.qbase * 32,
                     (uint32_t)nq * 32u, sbar);
          } else {
            bulk_g2s(stage + q0 * 16, m.arc_tok + (size_t)lv.qbase * 4, (uint32_t)nq * 16u, sbar);
            bulk_g2s(stage + (kSQ + q0) * 16, m.arc_w + (size_t)lv.qbase * 4, (uint32_t)nq * 16u, sbar);
            bulk_g2s(stage + (2 * kSQ + q0) * 16, m.arc_to + (size_t)lv.qbase * 4, (uint32_t)nq * 16u, sbar);
          }
        }
        ++nst;
        spend = true;
      }
      D2COUNT(12);
      D2STAMP(6);
    }
    const int32_t slot = t % kRing2;
    const uint32_t ph = (uint32_t)(t / kRing2) & 1u;
    mbar_wait(sfull + slot, ph);
    mbar_wait(full + slot, ph);  // (already complete: the summary warp saw it) the frame's bytes for this warp
    D2STAMP(0);
    const float* fb = frame_buf(t);
    const float4 s0 = reinterpret_cast<const float4*>(sums + slot)[0];
    const int4 s1 = reinterpret_cast<const int4*>(sums + slot)[1];
    float bv = -INFINITY;  // the best exactly valued (value, column) so far (R14 order)
    int32_t bc = INT_MAX, ns = st;
    bool got = false;
    if (kNoLM) {  // plain greedy: every column raw
      if (better(s0.x, sp, bv, bc)) { bv = s0.x; bc = sp; }
      if (s1.x >= 0 && better(s0.y, s1.x, bv, bc)) { bv = s0.y; bc = s1.x; }
      got = true;
    } else if (fast) {
      if (better(s0.x, sp, bv, bc)) { bv = s0.x; bc = sp; }  // blank: fmaf(lambda, 0, x) == x
      if (pc >= 0) {                                          // the repeated column: raw (R17)
        const float xp = fb[pc];
        if (better(xp, pc, bv, bc)) { bv = xp; bc = pc; }
      }
      if (bv > __fmaf_rn(lambda, ub, s1.x != pc ? s0.y : s0.z)) {
        got = true;  // level 0
        D2COUNT(8);
        D2STAMP(1);
      } else if (staged) {
        D2STAMP(1);
        // level 1: the exact fused values of c1, c2 (pc excluded: its value is raw)
        const int32_t ca = s1.x == pc ? -1 : s1.x, cb = (s1.y == pc || s1.y == s1.x) ? -1 : s1.y;
        const int32_t va = ca < 0 ? -1 : ca - (ca > sp), vb = cb < 0 ? -1 : cb - (cb > sp);
        stage_wait();
        D2STAMP(3);
        const uint32_t tmask = kPacked ? (1u << m.pk_bits) - 1u : 0xffffffffu;
        uint32_t ka = 0u, kb = 0u;  // the last (highest-order) hit: (slot << 7 | lane << 2 | j) + 1
#pragma unroll 2
        for (int32_t k = 0; k < nslots; ++k) {
          const int32_t L = nlev - 1 - __popc(__ballot_sync(kFull, lv.eslot <= k));
          const int32_t info = __shfl_sync(kFull, lv.info, L + 1);
          if ((k - (info >> 16)) * 32 + lane < (info & 0xffff)) {
            const int4 q = reinterpret_cast<const int4*>(stage)[kPacked ? 2 * (k * 32 + lane) : k * 32 + lane];
            const uint32_t tk[4] = {(uint32_t)q.x & tmask, (uint32_t)q.y & tmask, (uint32_t)q.z & tmask,
                                    (uint32_t)q.w & tmask};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint32_t key = (uint32_t)((k << 7) | (lane << 2) | j) + 1u;
              if (tk[j] == (uint32_t)va) ka = key;
              if (tk[j] == (uint32_t)vb) kb = key;
            }
          }
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int32_t col = c ? cb : ca, vt = c ? vb : va;
          const uint32_t kk = __reduce_max_sync(kFull, c ? kb : ka);
          if (col < 0) continue;
          float lmv;
          int32_t nxv;
          if (kk) {
            const uint32_t pos = kk - 1u;
            const int32_t k = (int32_t)(pos >> 7), qi = k * 32 + (int32_t)((pos >> 2) & 31u), j = (int32_t)(pos & 3u);
            const int32_t L = nlev - 1 - __popc(__ballot_sync(kFull, lv.eslot <= k));
            const float acc = __shfl_sync(kFull, lv.acc, L + 1);
            float w;
            if (kPacked) {
              nxv = (int32_t)(reinterpret_cast<const uint32_t*>(stage)[qi * 8 + j] >> m.pk_bits);
              w = reinterpret_cast<const float*>(stage)[qi * 8 + 4 + j];
            } else {
              w = reinterpret_cast<const float*>(stage + (size_t)kSQ * 16)[qi * 4 + j];
              nxv = reinterpret_cast<const int32_t*>(stage + (size_t)2 * kSQ * 16)[qi * 4 + j];
            }
            lmv = __fadd_rn(acc, w);  // acc_boff + arc weight (Alg. 1 line 74)
          } else {
            lmv = __fadd_rn(acc_root, root_w[vt]);  // the root level
            nxv = root_to[vt];
          }
          const float fv = __fmaf_rn(lambda, lmv, fb[col]);
          if (better(fv, col, bv, bc)) { bv = fv; bc = col; ns = nxv; }
        }
        if (bv > __fmaf_rn(lambda, ub, s0.w)) { got = true; D2COUNT(9); }  // level 1
        D2STAMP(2);
      }
    }
    if (!got) {  // level 2: the exact step over the full row (ctc_decode_kernel's frame)
      D2COUNT(10);
      if (row_state != st) {
        if (kPacked && staged) {  // the row from the staged arcs: root level, then the levels in slot order
          stage_wait();
          {
            const float4* w4 = reinterpret_cast<const float4*>(root_w);
            const int4* t4 = reinterpret_cast<const int4*>(root_to);
            float4* s4 = reinterpret_cast<float4*>(s.row_s);
            int4* n4 = reinterpret_cast<int4*>(s.row_n);
            for (int32_t q = lane; q < V / 4; q += 32) {
              float4 y = w4[q];
              y.x = __fadd_rn(acc_root, y.x);
              y.y = __fadd_rn(acc_root, y.y);
              y.z = __fadd_rn(acc_root, y.z);
              y.w = __fadd_rn(acc_root, y.w);
              s4[q] = y;
              n4[q] = t4[q];
            }
          }
          __syncwarp();
          const uint32_t tmask = (1u << m.pk_bits) - 1u;
#pragma unroll 1
          for (int32_t k = 0; k < nslots; ++k) {  // slot order = level order, lowest order first (Alg. 1 lines 77-79)
            const int32_t L = nlev - 1 - __popc(__ballot_sync(kFull, lv.eslot <= k));
            const int32_t info = __shfl_sync(kFull, lv.info, L + 1);
            const float acc = __shfl_sync(kFull, lv.acc, L + 1);
            if ((k - (info >> 16)) * 32 + lane < (info & 0xffff)) {
              const int4 q = reinterpret_cast<const int4*>(stage)[2 * (k * 32 + lane)];
              const float4 w = reinterpret_cast<const float4*>(stage)[2 * (k * 32 + lane) + 1];
              const int32_t qq[4] = {q.x, q.y, q.z, q.w};
              const float ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const uint32_t x = (uint32_t)qq[j];
                s.row_s[x & tmask] = __fadd_rn(acc, ww[j]);
                s.row_n[x & tmask] = (int32_t)(x >> m.pk_bits);
              }
            }
            __syncwarp();
          }
          __syncwarp();
        } else {
          build_row_warp<true, kPacked>(m, s, root_w, root_to, st);
        }
        row_state = st;
        D2COUNT(11);
      }
      D2STAMP(4);
      float val[kMaxColsPerLane];
#pragma unroll
      for (int j = 0; j < kMaxColsPerLane; ++j) {
        const int32_t col = lane + 32 * j;
        float x = __int_as_float(0x7fc00000);  // past the last column: NaN, never selected
        float lmv = 0.f;                        // blank: 0
        if (col < ncols) {
          x = fb[col];
          if (col != sp) lmv = s.row_s[col - (col > sp)];
        }
        val[j] = col == pc ? x : __fmaf_rn(lambda, lmv, x);
      }
      bc = warp_argmax_cols(val);
      if (bc >= 0 && bc < ncols && bc != sp && bc != pc) ns = s.row_n[bc < sp ? bc : bc - 1];
      D2STAMP(5);
    }
    int32_t tok = -1;
    if (bc >= 0 && bc < ncols) {
      tok = bc;
      if (bc == sp) {
        pc = -1;
      } else if (bc != pc) {  // an emission: LM advance (a repeat of prev is collapsed)
        if (lane == 0 && eout) eout[nemit] = bc;
        ++nemit;
        pc = bc;
        if (!kNoLM && ns != st) { st = ns; need_state = true; }
      }
    }
    if (lane == 0 && fout) fout[t] = tok;
    release_slot(empty + slot);
    D2STAMP(7);
  }
#ifdef NGPULM_PHASE_TIMING
  if (lane == 0 && row < 16384)
    for (int i = 0; i < 13; ++i) g_phase[row * 16 + i] = (unsigned long long)ck[i];
#endif
#undef D2STAMP
#undef D2COUNT
  stage_wait();  // no bulk copy in flight at exit
  if (fout)
    for (int32_t t = run + lane; t < T; t += 32) fout[t] = -1;
  if (lane == 0) {
    if (!kNoLM) states[row] = st;
    prev[row] = pc;
    if (emit_len) emit_len[row] = nemit;
  }
}

// ---------------------------------------------------------------- segment-parallel exact CTC decode
// A row's decisions form one chain (frame t needs the LM state and prev after
// frame t-1), ~290 emissions long at configs[2], each emission a dependent
// record -> arcs -> row rebuild. The chain is cut into K segments decoded at
// once (pass 1): segment 0 from the row's true start; segment k >= 1 from the
// root state and no prev, kSegWarm frames before its first frame (an n-gram
// state is the suffix of the last N-1 emitted tokens, so the warm-up usually
// reaches the true trajectory before the segment starts). Pass 2 (one CTA per
// row) re-decides every boundary at once, one warp each, from the state
// recorded before it (the previous segment's last record) until its decision
// and state equal the records at the same frame — decisions depend only on
// (state, prev) and the frame, so from there on the records are one run of the
// decision process; a segment that never meets is re-decided to its end. A
// boundary whose recorded start its predecessor's fix-up rewrote is re-done in
// order by warp 0 (each warp keeps the start it used), which then turns the
// per-frame decisions into the emission list, the final state and prev.
// Every output is therefore exactly ctc_decode_kernel's (tested bit-exact).
// Records: frames_out holds the decisions, emit_out (row stride T) the state
// after every frame until the end of pass 2 overwrites it with the emissions.
// One warp per chain with its own TMA ring (lane 0 refills a slot right after
// the warp has read it), so a segment costs one warp's registers.
#ifndef NGPULM_SEG_CTAS
#define NGPULM_SEG_CTAS 2  // resident CTAs per SM (kSegRows chains each): the chains one launch holds at once
#endif
#ifndef NGPULM_SEG_MIN_FRAMES
#define NGPULM_SEG_MIN_FRAMES 64  // fewest frames per segment
#endif
#ifndef NGPULM_SEG_EXPT
#define NGPULM_SEG_EXPT 0  // timing experiments only (tools/): bit 0 no proxy fence, bit 1 no pass-1 records
#endif
#ifndef NGPULM_SEG_MERGED
#define NGPULM_SEG_MERGED 0  // 1: both passes in one launch (one CTA per row; measured 0.322 vs 0.305 ms: the
                             // pass-2 code spills registers into the pass-1 loop); 0: two launches
#endif
#ifndef NGPULM_SEG_RW_REGS
#define NGPULM_SEG_RW_REGS 1  // root weights: 1 in registers (33 per lane; 0.305 vs 0.323 ms), 0 read from the CTA copy
#endif
#ifndef NGPULM_SEG_RING
#define NGPULM_SEG_RING 2
#endif
constexpr int kSegRing = NGPULM_SEG_RING;  // frames in flight per chain
#ifndef NGPULM_SEG_WARM
#define NGPULM_SEG_WARM 16
#endif
constexpr int kSegWarm = NGPULM_SEG_WARM;  // warm-up frames before a segment >= 1
#ifndef NGPULM_SEG_ROWS
#define NGPULM_SEG_ROWS 4
#endif
constexpr int kSegRows = NGPULM_SEG_ROWS;  // chains (warps) per CTA, sharing the root-level copy
constexpr int kSegCtas = NGPULM_SEG_CTAS;

// A chain's row: arc-level entries only, tagged with the rebuild that wrote them
// ({acc_boff + weight, generation << 24 | next state} per token); a token without
// an entry of the current generation takes the root level (acc_root + root
// weight from the lane's registers, root target from the CTA's copy), so a
// rebuild writes only the arcs, not the V root entries.
__host__ __device__ constexpr size_t grow_bytes(int32_t V) { return align16((size_t)(V + 1) * 8); }
__host__ __device__ constexpr size_t sslice_bytes(int32_t V, int32_t order) {
  return grow_bytes(V) + levels_bytes(order) + 16 + align16(kSegRing * 8) +
         (size_t)kSegRing * lbuf_bytes(V);
}
// [tiny model copy] | root_w | root_to | cbar | pass-2 boundary starts [2 x 8] | R slices
// (row_g | levels | 2 bars | full[kSegRing] | ring)
constexpr int kSegHdr = 16 + 64;
__host__ __device__ constexpr size_t scta_smem(int32_t V, int32_t order, int R) {
  return 2 * align16((size_t)V * 4) + kSegHdr + (size_t)R * sslice_bytes(V, order);
}

// write_window into generation-tagged entries: row_g[token] = {acc_boff + weight,
// (generation << 24) | next state} (states < 2^24, generations 1..255).
template <int kW, bool kPacked>
__device__ __forceinline__ void write_window_gen(float2* row_g, const Window<kW, kPacked>& a, int32_t k0,
                                                 int32_t nslots, int32_t pk_bits, int32_t gen) {
  const uint32_t tmask = (1u << pk_bits) - 1u;
  const uint32_t gtag = (uint32_t)gen << 24;
#pragma unroll
  for (int g = 0; g < kW; g += 8) {
    if (g > 0 && k0 + g >= nslots) break;
#pragma unroll
    for (int u = g; u < g + 8; ++u) {
      if (u > g && k0 + u >= nslots) break;  // (uniform) past the row's last slot: nothing to write
      if (u > 0) __syncwarp();  // slots in level order: a lower order is done before a higher one
      const int32_t x[4] = {a.tok[u].x, a.tok[u].y, a.tok[u].z, a.tok[u].w};
      const float ww[4] = {a.w[u].x, a.w[u].y, a.w[u].z, a.w[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int32_t tk, nx;
        if (kPacked) {
          tk = (int32_t)((uint32_t)x[j] & tmask);
          nx = (int32_t)((uint32_t)x[j] >> pk_bits);
        } else {
          const int32_t t4[4] = {a.to[u].x, a.to[u].y, a.to[u].z, a.to[u].w};
          tk = x[j];
          nx = t4[j];
        }
        // acc_boff + arc_weights (Alg. 1 line 74), the arc's target
        row_g[tk] = make_float2(__fadd_rn(a.acc[u], ww[j]), __uint_as_float(gtag | (uint32_t)nx));
      }
    }
  }
  __syncwarp();
}

// The chain record of state `st` (chain table row: lane l < chain_slots holds
// slot l), loaded by an ordered (volatile) access so that it is in flight while
// the caller does other work before build_row_gen consumes it.
template <bool kTiny>
__device__ __forceinline__ int4 record_issue(const DevModel& m, const WSlice& s, int32_t st) {
  const int lane = threadIdx.x & 31;
  int4 x = make_int4(0, 0, 0, 0);
  if (st >= 0 && st < m.S && lane < m.chain_slots) {
    if (kTiny) {
      x = s.chain_s[(size_t)st * m.chain_slots + lane];
    } else {
      const int4* p = reinterpret_cast<const int4*>(m.chain) + (size_t)st * m.chain_slots + lane;
      asm volatile("ld.global.nc.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w) : "l"(p));
    }
  }
  return x;
}

// The arc levels of state `st` (record x from record_issue) into row_g with tag
// `gen` (Algorithm 1's levels 1..N-1; the root level stays implicit).
// Returns the row scalars (warp_row_src's, table mode).
template <bool kPacked, bool kTiny, typename F = NoStamp>
__device__ __forceinline__ Row build_row_gen(const DevModel& m, const WSlice& s, float2* row_g, int32_t st,
                                             const int4 x, int32_t gen, F stamp = F()) {
  constexpr int kW = 8;
  const int lane = threadIdx.x & 31;
  WLevel lv;
  lv.beg = 0; lv.qbase = 0; lv.info = 0; lv.eslot = INT_MAX; lv.acc = 0.f;
  Row r;
  r.state = st;
  r.bad = st < 0 || st >= m.S;
  r.nlev = 0; r.total = 0; r.acc_root = 0.f; r.fin = 0.f;
  if (r.bad) return r;
  r.nlev = __shfl_sync(kFull, x.x, 0);
  r.acc_root = __int_as_float(__shfl_sync(kFull, x.y, 0));
  r.fin = __int_as_float(__shfl_sync(kFull, x.z, 0));
  r.total = __shfl_sync(kFull, x.w, 0);
  if (lane >= 1 && lane <= r.nlev) {
    lv.beg = x.x;
    lv.acc = __int_as_float(x.z);
    lv.info = x.w;
    lv.eslot = (lv.info >> 16) + (((lv.info & 0xffff) + 31) >> 5);
  }
  lv.qbase = lv.beg >> 2;
  const int32_t nslots = r.nlev > 0 ? __shfl_sync(kFull, lv.eslot, 1) : 0;
  stamp(7);
  Window<kW, kPacked> a;
  load_window<kW, kPacked, kTiny>(m, s, lv, r.nlev, 0, nslots, a);
  for (int32_t k0 = 0; k0 < nslots;) {
    write_window_gen<kW, kPacked>(row_g, a, k0, nslots, m.pk_bits, gen);
    stamp(8);
    k0 += kW;
    if (k0 < nslots) load_window<kW, kPacked, kTiny>(m, s, lv, r.nlev, k0, nslots, a);
  }
  __syncwarp();
  stamp(9);
  return r;
}

// the first frame of segment k: segment 0 is [0, L0), segment k >= 1 [L0 + (k - 1) L, L0 + k L)
__device__ __forceinline__ int32_t seg_begin(int32_t k, int32_t L0, int32_t L) { return k == 0 ? 0 : L0 + (k - 1) * L; }

// The end of pass 2, per row (one warp): the emissions from the decisions (CTC
// collapse: a selection that is neither blank nor prev), the final state and
// prev; frames past the row's length -1; an invalid row as ctc_decode_kernel
// (bad-row word, nothing decided, state and prev unchanged).
__device__ __forceinline__ void compact_row(int32_t row, int32_t T, int32_t len, int32_t st0, int32_t sp,
                                            int32_t* frames_out, int32_t* rec, int32_t* states, int32_t* prev,
                                            int32_t* emit_len, unsigned long long* bad_row, bool bad) {
  const int lane = threadIdx.x & 31;
  int32_t* fo = frames_out + (size_t)row * T;
  int32_t* eo = rec + (size_t)row * T;
  if (bad) {
    for (int32_t t = lane; t < T; t += 32) fo[t] = -1;
    if (lane == 0) {
      if (len > 0) atomicMin(bad_row, (unsigned long long)row);
      if (emit_len) emit_len[row] = 0;
    }
    return;
  }
  const int32_t st_final = len > 0 ? eo[len - 1] : st0;  // the last record, read before eo is overwritten
  int32_t pc = prev[row], count = 0;
  __syncwarp();
  const uint32_t lt = (1u << lane) - 1u;
  constexpr int kU = 16;  // 32-frame blocks whose decisions are loaded at once (one memory latency per 512 frames)
  for (int32_t b0 = 0; b0 < len; b0 += 32 * kU) {
    int32_t fr[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int32_t t = b0 + 32 * u + lane;
      fr[u] = t < len ? fo[t] : -1;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
    const int32_t b = b0 + 32 * u;
    if (b >= len) break;
    const int32_t f = fr[u];
    const uint32_t valid = __ballot_sync(kFull, f >= 0);
    const uint32_t before = valid & lt;  // prev before frame t: the last selecting frame before it
    const int32_t fp = __shfl_sync(kFull, f, before ? 31 - __clz(before) : 0);
    const int32_t pcb = before ? (fp == sp ? -1 : fp) : pc;
    const bool emit = f >= 0 && f != sp && f != pcb;
    const uint32_t em = __ballot_sync(kFull, emit);
    if (emit) eo[count + __popc(em & lt)] = f;
    count += __popc(em);
    if (valid) {
      const int32_t fl = __shfl_sync(kFull, f, 31 - __clz(valid));
      pc = fl == sp ? -1 : fl;
    }
    }
  }
  for (int32_t t = len + lane; t < T; t += 32) fo[t] = -1;
  __syncwarp();
  if (lane == 0) {
    states[row] = st_final;
    prev[row] = pc;
    if (emit_len) emit_len[row] = count;
  }
}

// registers: as many as kSegCtas resident CTAs leave (65536 per SM, allocated in units of 8 per thread)
constexpr int kSegMaxReg = (65536 / (32 * kSegRows * kSegCtas)) / 8 * 8 > 255 ? 255
                                                                               : (65536 / (32 * kSegRows * kSegCtas)) / 8 * 8;
// kPass: 1 = pass 1 only (one warp per chain), 2 = pass 2 only (one CTA per row), 3 = both in one launch
// (one CTA per row, warp w decodes segment w, then the same CTA fixes the row's boundaries)
// kVc: the vocabulary size as a compile-time constant (1024, the workload's BPE vocabulary: the column
// predicates fold away), or 0 = m.V at run time
template <bool kTable, bool kPacked, bool kTiny, int kPass, int kVc = 0>
__global__ void __maxnreg__(kSegMaxReg)
    ctc_seg_kernel(DevModel m, const float* __restrict__ logits, int64_t row_stride, int64_t frame_stride,
                   int32_t B, int32_t T, int32_t K, int32_t L0, int32_t L, const int32_t* __restrict__ lengths,
                   int32_t* __restrict__ states, int32_t* __restrict__ prev, float lambda, int32_t sp,
                   int32_t* __restrict__ frames_out, int32_t* __restrict__ rec, int32_t* __restrict__ emit_len) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int32_t V = kVc ? kVc : m.V, ncols = V + 1;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, R = blockDim.x >> 5;
  const size_t rb = align16((size_t)V * 4);
  unsigned char* sm0 = smem + (kTiny ? tiny_copy_bytes(m.tiny_chain_bytes, m.tiny_arcq_bytes) : 0);
  float* root_w = reinterpret_cast<float*>(sm0);
  int32_t* root_to = reinterpret_cast<int32_t*>(sm0 + rb);
  uint64_t* cbar = reinterpret_cast<uint64_t*>(sm0 + 2 * rb);
  static_assert(kTable, "the segment decode reads the chain table");
  unsigned char* base = sm0 + 2 * rb + kSegHdr + (size_t)w * sslice_bytes(V, m.order);
  float2* row_g = reinterpret_cast<float2*>(base);
  WSlice s;
  {
    unsigned char* lp = base + grow_bytes(V);
    int32_t* l = reinterpret_cast<int32_t*>(lp);
    const int32_t Lc = level_cap(m.order);
    s.row_s = nullptr;
    s.row_n = nullptr;
    s.beg = l;
    s.pre = l + Lc;
    s.acc = reinterpret_cast<float*>(l + 2 * Lc + 1);
    s.bar = reinterpret_cast<uint64_t*>(lp + levels_bytes(m.order));
    s.abar = s.bar + 1;
    s.st_q = nullptr;
    s.chain_s = nullptr;
  }
  if (kTiny) {
    s.chain_s = reinterpret_cast<const int4*>(smem);
    s.st_q = reinterpret_cast<int4*>(smem + align16((size_t)m.tiny_chain_bytes));
  }
  uint64_t* full = s.bar + 2;
  float* ring = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(full) + align16(kSegRing * 8));
  const size_t lstride = lbuf_bytes(V) / 4;
  for (int32_t c = lane; c < V; c += 32) row_g[c] = make_float2(0.f, 0.f);  // generation 0: never current
  pdl_trigger();
  if (threadIdx.x == 0) {  // the root level (immutable model data: before the wait)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(cbar)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(cbar)), "r"((uint32_t)V * 8u)
                 : "memory");
    bulk_g2s(root_w, m.arc_w, (uint32_t)V * 4u, cbar);
    bulk_g2s(root_to, m.arc_to, (uint32_t)V * 4u, cbar);
    if (kTiny) tiny_copy_issue(m, smem);
  }
  if (lane == 0) {
    for (int i = 0; i < kSegRing; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + i)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  const int32_t chain = (int32_t)blockIdx.x * R + w;
  const int32_t row = kPass == 1 ? chain / K : (int32_t)blockIdx.x;  // passes 2 and 3: one row per CTA
  const int32_t k0 = kPass == 1 ? chain % K : (kPass == 3 ? w : 0);
  auto cta_exit = [&]() {  // no exit with the CTA's bulk copies in flight
    if (threadIdx.x == 0) {
      mbar_wait(cbar, 0);
      if (kTiny) mbar_wait(tiny_bar(smem, m), 0);
    }
  };
  if (row >= B) { cta_exit(); return; }
  pdl_wait();  // (pass 2 reads pass 1's records)
  int32_t len = T;
  if (lengths) len = min(T, max(0, __ldg(&lengths[row])));
  const int32_t st0 = states[row];  // (pass 2 rewrites it last, in compact_row)
  if (kPass == 1 && (st0 < 0 || st0 >= m.S || seg_begin(k0, L0, L) >= len)) { cta_exit(); return; }
  if (kPass != 1 && (st0 < 0 || st0 >= m.S)) {  // an invalid row decides nothing (as ctc_decode_kernel)
    if (w == 0) compact_row(row, T, len, st0, sp, frames_out, rec, states, prev, emit_len, m.bad_row, true);
    cta_exit();
    return;
  }
  mbar_wait(cbar, 0);
  if (kTiny) mbar_wait(tiny_bar(smem, m), 0);
  const float* lrow0 = logits + (size_t)row * row_stride;
  int32_t* fo = frames_out + (size_t)row * T;
  int32_t* ro = rec + (size_t)row * T;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  // the ring: frame number `idx` (counted over the warp's life) sits in slot idx % kSegRing
  uint32_t issued = 0, consumed = 0;
  int32_t next_t = 0, stop_t = 0;
  // the bytes the logits view spans (frame covers may read a few columns of the neighbouring frames)
  const float* lo_b = logits;
  const float* hi_b = logits + (size_t)(B - 1) * row_stride + (size_t)(T - 1) * frame_stride + ncols;
  auto issue_upto = [&]() {
    while (issued - consumed < (uint32_t)kSegRing && next_t < stop_t) {
      issue_frame_cover(lrow0 + (size_t)next_t * frame_stride, ncols, ring + (size_t)(issued % kSegRing) * lstride,
                        full + issued % kSegRing, pol, lo_b, hi_b);
      ++issued;
      ++next_t;
    }
  };
  auto take = [&](int32_t t) {  // wait for the next frame (t) of the ring; column c at [c]
    mbar_wait(full + consumed % kSegRing, (consumed / kSegRing) & 1u);  // (it tracks the edge cp.asyncs too)
    const float* lrow = lrow0 + (size_t)t * frame_stride;
    return ring + (size_t)(consumed % kSegRing) * lstride + (reinterpret_cast<uintptr_t>(lrow) & 15) / 4;
  };
  auto give = [&]() {  // the warp is done with the frame: its slot may be refilled
    if (!(NGPULM_SEG_EXPT & 1)) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    ++consumed;
  };
#ifdef NGPULM_PHASE_TIMING
  // debug build: per chain 0 rebuilds, 1 frame waits, 2 loads + refill issue, 3 decision, 4 records;
  // counts 5 frames, 6 rebuilds
  long long ck[11] = {0};
  long long tq0 = clock64(), tq1;
#define SSTAMP(i) do { tq1 = clock64(); ck[i] += tq1 - tq0; tq0 = tq1; } while (0)
#else
#define SSTAMP(i) do { } while (0)
#endif
  float lm[kMaxColsPerLane];  // the row's LM scores
#if NGPULM_SEG_RW_REGS
  float rw[kMaxColsPerLane];  // the root weights of the same columns
#pragma unroll
  for (int j = 0; j < kMaxColsPerLane; ++j) {
    const int32_t col = lane + 32 * j;
    rw[j] = (col < ncols && col != sp) ? root_w[col - (col > sp)] : 0.f;
  }
#define NGPULM_RW(j, tk) rw[j]
#else
#define NGPULM_RW(j, tk) root_w[tk]
#endif
  int32_t row_state = -1, gen = 0;
  auto finish_row = [&](int32_t st, const int4 x) {  // the row of st from its record x
#ifdef NGPULM_PHASE_TIMING
    ck[6] += 1;
#endif
    if (++gen == 256) {  // generations wrap: no entry may carry the new one
      __syncwarp();
      for (int32_t c = lane; c < V; c += 32) row_g[c].y = 0.f;
      __syncwarp();
      gen = 1;
    }
#ifdef NGPULM_PHASE_TIMING
    auto bstamp = [&](int i) { SSTAMP(i); };
#else
    NoStamp bstamp;
#endif
    const Row r = build_row_gen<kPacked, kTiny>(m, s, row_g, st, x, gen, bstamp);
    // branch-free, loads in groups of 11 columns (lane i: columns i + 32 j); out-of-row columns read token V-1
    static_assert(kMaxColsPerLane % 11 == 0, "groups of 11 columns");
#pragma unroll
    for (int g = 0; g < kMaxColsPerLane; g += 11) {
      float2 e[11];
      float rv[11];
#pragma unroll
      for (int u = 0; u < 11; ++u) {
        const int32_t col = lane + 32 * (g + u);
        const int32_t tk = min(col - (col > sp), V - 1);
        e[u] = row_g[tk];
        rv[u] = NGPULM_RW(g + u, tk);
      }
#pragma unroll
      for (int u = 0; u < 11; ++u) {
        const int32_t col = lane + 32 * (g + u);
        const float v = (__float_as_uint(e[u].y) >> 24) == (uint32_t)gen ? e[u].x : __fadd_rn(r.acc_root, rv[u]);
        lm[g + u] = (col < ncols && col != sp) ? v : 0.f;  // blank: 0 (fused value = asr)
      }
    }
    row_state = st;
  };
  auto ensure_row = [&](int32_t st) {
    if (row_state != st) finish_row(st, record_issue<kTiny>(m, s, st));
  };
  auto next_state = [&](int32_t tk) {  // the state after token tk from the row's state
    const uint32_t e = __float_as_uint(row_g[tk].y);
    const int32_t rt = root_to[tk];  // (both shared loads in flight at once)
    return (e >> 24) == (uint32_t)gen ? (int32_t)(e & 0xffffffu) : rt;
  };
  // the fused CTC decision of one frame (ctc_decode_kernel's, R13, R14, R17, R19); the frame's
  // slot is handed back (and refilled) as soon as its columns are in registers
  auto load_frame = [&](int32_t t, float (&val)[kMaxColsPerLane]) {  // frame t's columns into registers
    const float* bp = take(t) + lane;
    SSTAMP(1);
#pragma unroll
    for (int j = 0; j < kMaxColsPerLane; ++j) {
      const int32_t col = lane + 32 * j;
      val[j] = __int_as_float(0x7fc00000);
      if (col < ncols) val[j] = bp[32 * j];
    }
    give();
    issue_upto();
    SSTAMP(2);
  };
  auto decide = [&](float (&val)[kMaxColsPerLane], int32_t pc) {
    float mx[kMaxColsPerLane];
#pragma unroll
    for (int j = 0; j < kMaxColsPerLane; ++j) {
      const int32_t col = lane + 32 * j;
      val[j] = col == pc ? val[j] : __fmaf_rn(lambda, lm[j], val[j]);
      mx[j] = val[j];
    }
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
    return (int32_t)__reduce_min_sync(kFull, (uint32_t)cm[0]);
  };
  // one frame t: decision from (st, pc), then (st, pc) after it; returns the selected column or -1
  auto step = [&](int32_t t, int32_t& st, int32_t& pc) {
    SSTAMP(4);
    float val[kMaxColsPerLane];
    if (row_state != st) {  // a rebuild: the record load flies while the frame's columns are read
      const int4 x = record_issue<kTiny>(m, s, st);
      load_frame(t, val);
      finish_row(st, x);
      SSTAMP(0);
    } else {
      load_frame(t, val);
    }
    const int32_t bc = decide(val, pc);
    SSTAMP(3);
#ifdef NGPULM_PHASE_TIMING
    ck[5] += 1;
#endif
    if (bc < 0 || bc >= ncols) return -1;  // all-NaN frame: nothing changes
    if (bc == sp) {
      pc = -1;
    } else if (bc != pc) {  // an emission: LM advance
      st = next_state(bc < sp ? bc : bc - 1);
      pc = bc;
    }
    return bc;
  };
  if (kPass == 1 || (kPass == 3 && seg_begin(k0, L0, L) < len)) {  // ---- pass 1: segment k0
    const int32_t t0 = seg_begin(k0, L0, L), t1 = min(seg_begin(k0 + 1, L0, L), len);
    const int32_t tb = k0 == 0 ? 0 : max(0, t0 - kSegWarm);
    int32_t st = k0 == 0 ? st0 : 0, pc = k0 == 0 ? __ldg(&prev[row]) : -1;
    next_t = tb;
    stop_t = t1;
    issue_upto();
    int32_t my_tok = -1, my_st = 0;  // the records of frames t0 + 32 i + lane, stored 32 frames at a time
    for (int32_t t = tb; t < t1; ++t) {
      const int32_t tok = step(t, st, pc);
      if (t >= t0 && !(NGPULM_SEG_EXPT & 2)) {
        const int32_t i = (t - t0) & 31;
        if (lane == i) { my_tok = tok; my_st = st; }
        if (i == 31 || t == t1 - 1) {
          if (lane <= i) {
            fo[t - i + lane] = my_tok;
            ro[t - i + lane] = my_st;
          }
        }
      }
      SSTAMP(4);
    }
  }
  if (kPass == 3) __syncthreads();  // every segment of the row decoded: its records are visible to the CTA
  if (kPass != 1) {  // ---- pass 2: every boundary of the row at once (warp w: k = 1 + w, 1 + w + R, ...), then warp 0
    // re-does, in order, any boundary whose start its predecessor's fix-up rewrote, and compacts
    int32_t* used = reinterpret_cast<int32_t*>(sm0 + 2 * rb + 16);  // [k]: start state, [8 + k]: start prev
    const int32_t pc_row = __ldg(&prev[row]);
    // prev before t0: the last frame before t0 that selected a column (blank -> -1), else the row's prev
    auto prev_before = [&](int32_t t0) {
      int32_t pc = pc_row;
      for (int32_t b = t0 - 1; b >= 0; b -= 32) {
        const int32_t t = b - lane;
        const int32_t f = t >= 0 ? fo[t] : -1;
        const uint32_t hit = __ballot_sync(kFull, f >= 0);
        if (hit) {
          const int32_t fl = __shfl_sync(kFull, f, __ffs(hit) - 1);
          pc = fl == sp ? -1 : fl;
          break;
        }
      }
      return pc;
    };
    // re-decide segment k from (st, pc) at its first frame until the decision and the state meet the
    // records (any record sequence in the arrays is one continuous run of the decision process)
    auto fix = [&](int32_t k, int32_t st, int32_t pc) {
      const int32_t t0 = seg_begin(k, L0, L), t1 = min(seg_begin(k + 1, L0, L), len);
      const int32_t f_pre = t0 + lane < t1 ? fo[t0 + lane] : -1, s_pre = t0 + lane < t1 ? ro[t0 + lane] : -1;
      // frames still in the ring from the warp's previous meeting point: their slots are taken
      // back after this segment's row is built (they have landed by then)
      const uint32_t stale_end = issued;
      next_t = t0;
      stop_t = t1;
      issue_upto();
      ensure_row(st);
      while (consumed < stale_end) {
        take(0);
        give();
      }
      issue_upto();
      for (int32_t t = t0; t < t1; ++t) {
        const int32_t tok = step(t, st, pc);
#ifdef NGPULM_PHASE_TIMING
        if (lane == 0 && row < 4096) g_phase[(8192 + row) * 16 + k] += 1;  // fix-up frames of segment k
#endif
        const int32_t i = t - t0;
        const int32_t f_rec = i < 32 ? __shfl_sync(kFull, f_pre, i) : fo[t];
        const int32_t s_rec = i < 32 ? __shfl_sync(kFull, s_pre, i) : ro[t];
        const bool met = tok >= 0 && tok == f_rec && st == s_rec;  // same (state, prev) from here on
        if (!met && lane == 0) {
          fo[t] = tok;
          ro[t] = st;
        }
        __syncwarp();
        if (met) break;
      }
    };
    for (int32_t k = 1 + w; k < K; k += R) {
      const int32_t t0 = seg_begin(k, L0, L);
      if (t0 >= len) break;
      const int32_t st = ro[t0 - 1], pc = prev_before(t0);  // (the predecessor's fix-up may be rewriting them)
      if (lane == 0) {
        used[k] = st;
        used[8 + k] = pc;
      }
      fix(k, st, pc);
    }
    __syncthreads();  // every fix-up's records are visible to the CTA
    if (w == 0) {
      for (int32_t k = 1; k < K; ++k) {  // segments before k are final: k's true start decides
        const int32_t t0 = seg_begin(k, L0, L);
        if (t0 >= len) break;
        const int32_t st = ro[t0 - 1], pc = prev_before(t0);
        if (st != used[k] || pc != used[8 + k]) fix(k, st, pc);
      }
      __syncwarp();
      compact_row(row, T, len, st0, sp, frames_out, rec, states, prev, emit_len, m.bad_row, false);
    }
    while (consumed < issued) {  // frames issued past the last meeting point: let them land
      take(0);
      give();
    }
  }
  cp_async_settle();  // every edge cp.async of this warp has landed (the ring waits already implied it)
#ifdef NGPULM_PHASE_TIMING
  if (kPass != 2 && lane == 0 && chain < 16384)
    for (int i = 0; i < 11; ++i) g_phase[chain * 16 + i] = (unsigned long long)ck[i];
#endif
#undef SSTAMP
#undef NGPULM_RW
}

}  // namespace

int launch_ctc_decode(const DevModel& m, const float* logits, int64_t row_stride, int64_t frame_stride, int32_t B,
                      int32_t T, const int32_t* lengths, int32_t* states, int32_t* prev, float lambda, int32_t blank,
                      int32_t* frames_out, int32_t* emit_out, int32_t* emit_len, void* stream) {
  if (m.V % 4 != 0 || m.V > 1024) return (int)cudaErrorNotSupported;
  if (B <= 0) return 0;
  const bool pk = m.arc_q != nullptr && m.adv_kind == NGPULM_ADVANCE_AUTO, table = m.chain != nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  // plain greedy (no LM): the summary warps' raw argmax, frame-parallel. With an LM the default is
  // ctc_decode_kernel; the bound-pruned variant (NGPULM_DECODE_BOUND=1 builds) is exact too but its
  // single decider warp measured slower (configs[2]: 1.15 vs 0.69 ms).
  if (states == nullptr || (NGPULM_DECODE_BOUND && table)) {
    const size_t sm = d2_smem(m.V, m.order, pk);
    const dim3 g(B), b(32 * (2 + kSumWarps));
#define NGPULM_DECODE2(P, NOLM)                                                                                    \
  return launch(ctc_decode2_kernel<P, NOLM>, g, b, sm, st, m, logits, row_stride, frame_stride, B, T, lengths,     \
                states, prev, lambda, blank, frames_out, emit_out, emit_len)
    if (states == nullptr) NGPULM_DECODE2(true, true);
#if NGPULM_DECODE_BOUND
    if (pk) NGPULM_DECODE2(true, false);
    NGPULM_DECODE2(false, false);
#endif
#undef NGPULM_DECODE2
  }
  // segment-parallel exact decode: table mode, both record buffers given, enough frames per segment
  const size_t tinyb = pk && m.tiny_chain_bytes > 0 ? tiny_copy_bytes(m.tiny_chain_bytes, m.tiny_arcq_bytes) : 0;
#define NGPULM_SEG_VC(P, TI, PASS, VC, G, BL, SM)                                                                   \
  ((e = ensure_max_carveout((const void*)ctc_seg_kernel<true, P, TI, PASS, VC>)) != 0                                \
       ? e                                                                                                          \
       : launch(ctc_seg_kernel<true, P, TI, PASS, VC>, G, BL, SM, st, m, logits, row_stride, frame_stride, B, T, K,  \
                L0, L, lengths, states, prev, lambda, blank, frames_out, emit_out, emit_len))
#define NGPULM_SEG(P, TI, PASS, G, BL, SM) \
  (m.V == 1024 ? NGPULM_SEG_VC(P, TI, PASS, 1024, G, BL, SM) : NGPULM_SEG_VC(P, TI, PASS, 0, G, BL, SM))
  const bool seg_ok = table && frames_out && emit_out && kSegCtas > 0 && m.S <= (1 << 24);  // (24-bit states)
#if NGPULM_SEG_MERGED
  // one launch, one CTA per row, warp w decodes segment w and the CTA then fixes the row's boundaries:
  // a row's fix-ups start as soon as its own segments are done. K warps per CTA x ceil(B / 148) CTAs
  // per SM within the 8 warps per SM the register file holds (B <= 148: 8 segments, <= 296: 4, <= 592: 2)
  {
    const int cps = (B + 147) / 148;
    int K = 8 / cps;
    K = K > 8 ? 8 : K;
    if (K > T / NGPULM_SEG_MIN_FRAMES) K = T / NGPULM_SEG_MIN_FRAMES;
    if (seg_ok && K >= 2) {
      // every chain the same number of frames: segment 0 (no warm-up) kSegWarm frames longer
      const int32_t L = (T - kSegWarm + K - 1) / K, L0 = T - (K - 1) * L;
      const size_t sm0 = scta_smem(m.V, m.order, K);
      // the tiny-LM copy only where the CTAs of a wave still fit
      const bool tiny = tinyb > 0 && cps * (sm0 + tinyb + 1024) <= 228 * 1024;
      const size_t sm = sm0 + (tiny ? tinyb : 0);
      if (cps * (sm + 1024) <= 228 * 1024) {
        int e;
        const dim3 g(B), b(32 * K);
        if (tiny) return NGPULM_SEG(true, true, 3, g, b, sm);
        if (pk) return NGPULM_SEG(true, false, 3, g, b, sm);
        return NGPULM_SEG(false, false, 3, g, b, sm);
      }
    }
  }
#else
  // two launches: pass 1 (148 SMs x kSegCtas resident CTAs x kSegRows chains: one wave of chains), pass 2
  {
    int K = 148 * kSegCtas * kSegRows / B;
    K = K > 8 ? 8 : K;
    if (K > T / NGPULM_SEG_MIN_FRAMES) K = T / NGPULM_SEG_MIN_FRAMES;
    if (seg_ok && K >= 2) {
      const int32_t L = (T - kSegWarm + K - 1) / K, L0 = T - (K - 1) * L;
      const size_t sm0 = scta_smem(m.V, m.order, kSegRows);
      const bool tiny = tinyb > 0 && kSegCtas * (sm0 + tinyb + 1024) <= 228 * 1024;
      const size_t sm = sm0 + (tiny ? tinyb : 0);
      if (kSegCtas * (sm + 1024) <= 228 * 1024) {
        // pass 2: one CTA per row, one warp per boundary as far as 8 warps per SM (the register file) allow
        const int rows_per_sm = (B + 147) / 148;
        int w2 = 8 / rows_per_sm;
        w2 = w2 < 1 ? 1 : (w2 > K - 1 ? K - 1 : w2);
        const size_t sm2 = scta_smem(m.V, m.order, w2) + (tiny ? tinyb : 0);
        const dim3 b1(32 * kSegRows), g1((B * K + kSegRows - 1) / kSegRows), b2(32 * w2), g2(B);
        int e;
        if (tiny) e = NGPULM_SEG(true, true, 1, g1, b1, sm);
        else if (pk) e = NGPULM_SEG(true, false, 1, g1, b1, sm);
        else e = NGPULM_SEG(false, false, 1, g1, b1, sm);
        if (e) return e;
        if (tiny) return NGPULM_SEG(true, true, 2, g2, b2, sm2);
        if (pk) return NGPULM_SEG(true, false, 2, g2, b2, sm2);
        return NGPULM_SEG(false, false, 2, g2, b2, sm2);
      }
    }
  }
#endif
#undef NGPULM_SEG
#undef NGPULM_SEG_VC
  if (table && pk && m.tiny_chain_bytes > 0) {  // tiny LM: the model in every CTA's shared memory
    const size_t mb = tiny_copy_bytes(m.tiny_chain_bytes, m.tiny_arcq_bytes);
    int R = (B + 147) / 148;
    R = R < 1 ? 1 : (R > kDecodeMaxRows ? kDecodeMaxRows : R);
    int depth = kRingMax;
    while (depth > 2 && mb + dcta_smem(m.V, m.order, R, depth) > 227 * 1024) --depth;
    while (R > 1 && mb + dcta_smem(m.V, m.order, R, depth) > 227 * 1024) --R;
    const size_t sm = mb + dcta_smem(m.V, m.order, R, depth);
    if (sm <= 227 * 1024)
      return launch(ctc_decode_kernel<true, true, false, true>, dim3((B + R - 1) / R), dim3(64 * R), sm, st, m,
                    logits, row_stride, frame_stride, B, T, lengths, states, prev, lambda, blank, depth, frames_out,
                    emit_out, emit_len);
  }
  int R = (B + 147) / 148;
  R = R < 1 ? 1 : (R > kDecodeMaxRows ? kDecodeMaxRows : R);
  int depth = kRingMax;
  while (depth > 2 && dcta_smem(m.V, m.order, R, depth) > 227 * 1024) --depth;
  while (R > 1 && dcta_smem(m.V, m.order, R, depth) > 227 * 1024) --R;
  const size_t sm = dcta_smem(m.V, m.order, R, depth);
  const dim3 g((B + R - 1) / R), b(64 * R);
#define NGPULM_DECODE_LAUNCH(TB, P)                                                                                  \
  return launch(ctc_decode_kernel<TB, P>, g, b, sm, st, m, logits, row_stride, frame_stride, B, T, lengths, states, \
                prev, lambda, blank, depth, frames_out, emit_out, emit_len)
  if (table) { if (pk) NGPULM_DECODE_LAUNCH(true, true); NGPULM_DECODE_LAUNCH(true, false); }
  if (pk) NGPULM_DECODE_LAUNCH(false, true);
  NGPULM_DECODE_LAUNCH(false, false);
#undef NGPULM_DECODE_LAUNCH
}

}  // namespace ngpulm
