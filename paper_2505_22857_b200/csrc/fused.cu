// The fused greedy shallow-fusion step for sm_100a: CTA
// and warp-per-row kernels (CTC, RNN-T, AED), the transducer warp pair and
// label-looping step, the fused top-k, and their launchers.
#include "kcommon.cuh"

namespace ngpulm {
namespace {

template <int kMode, bool kTable>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
    fused_kernel(DevModel m, const float* __restrict__ logits, int64_t row_stride, int32_t* __restrict__ states,
                 int32_t* __restrict__ prev, const uint8_t* __restrict__ active, float lambda, int32_t sp,
                 AuxRow aux, int32_t* __restrict__ tokens_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int32_t V = m.V, ncols = V + 1, b = blockIdx.x;
  const int t = threadIdx.x;
  const Slice s = carve(smem, V, m.order);
  const bool tma = (V & 3) == 0;
  const bool nolm = states == nullptr;  // plain greedy decoding (no LM)
  pdl_trigger();
  prologue(m, s, tma);
  pdl_wait();
  if (active && !__ldg(&active[b])) {
    if (t == 0) tokens_out[b] = -1;
    __syncthreads();  // mbarrier init visible
    if (tma) mbar_wait(s.bar, 0);
    return;
  }
  const float* row = logits + (size_t)b * row_stride;
  const int32_t pc = (kMode == NGPULM_CTC) ? prev[b] : -2;
  float bv = -INFINITY;
  int32_t bc = INT_MAX;
  if (kMode == NGPULM_RNNT) {
    // stage 1: standard greedy prediction over all V+1 columns,
    // its loads issued before the row's levels are needed
    for (int32_t col = t; col < ncols; col += kThreads) {
      const float a = __ldg(&row[col]);
      if (better(a, col, bv, bc)) { bv = a; bc = col; }
    }
  }
  const Row r = nolm ? Row{} : row_levels<kTable>(m, states + b, s);
  if (r.bad) {
    if (t == 0) { tokens_out[b] = -1; atomicMin(m.bad_row, (unsigned long long)b); }
    if (tma) mbar_wait(s.bar, 0);
    return;
  }
  if (kMode == NGPULM_RNNT) {
    cta_argmax(bv, bc, s);
    if (bc == sp) {  // blank is retained: no LM work, state unchanged
      if (t == 0) tokens_out[b] = sp;
      if (tma) mbar_wait(s.bar, 0);
      return;
    }
    bv = -INFINITY;
    bc = INT_MAX;
  }
  if (nolm) {
    if (tma) mbar_wait(s.bar, 0);  // the root copy of the prologue is over
  } else {
    build_row(m, s, r, tma);
  }
  for (int32_t col = t; col < ncols; col += kThreads) {
    const float a = __ldg(&row[col]);
    float val;
    if (col == sp) {
      if (kMode == NGPULM_RNNT) continue;                             // stage 2: non-blank only
      val = (kMode == NGPULM_AED) ? __fmaf_rn(lambda, r.fin, a) : a;  // eos <-> final / blank raw
    } else if (kMode == NGPULM_CTC && col == pc) {
      val = a;                                                        // repeated token: not rescored
    } else {
      const int32_t tok = col < sp ? col : col - 1;
      val = __fmaf_rn(lambda, nolm ? 0.f : s.row_s[tok], a);  // asr + lambda * lm, one rounding
      if (aux.p) val = __fmaf_rn(-aux.lam, __ldg(aux.p + (size_t)b * aux.stride + tok), val);  // - lambda_ilm * ilm (R21)
    }
    if (better(val, col, bv, bc)) { bv = val; bc = col; }
  }
  cta_argmax(bv, bc, s);
  if (t == 0) {
    if (bc < 0 || bc >= ncols) {
      tokens_out[b] = -1;  // all-NaN row (unspecified)
    } else {
      tokens_out[b] = bc;
      if (bc == sp) {
        if (kMode == NGPULM_CTC) prev[b] = -1;
      } else if (!(kMode == NGPULM_CTC && bc == pc)) {  // a repeated CTC token: no LM advance
        if (!nolm) states[b] = s.row_n[bc < sp ? bc : bc - 1];
        if (kMode == NGPULM_CTC) prev[b] = bc;
      }
    }
  }
}

// kTiny: a tiny LM (keyword-biasing size) resident in the CTA's shared memory
// (tiny_copy_issue before the wait): records and arc quads are shared loads.
// kEarly (NGPULM_STEP_LOGITS_READY): the logits are copied before the wait.
// kReady (NGPULM_STEP_INPUTS_READY): no running kernel writes any input, so the
// logits are copied before the wait as well and the state read before it is
// final: no re-read after the wait (a decoder loop whose network kernel is not a
// programmatic-dependent launch: the step starts after it has completed).
template <int kMode, bool kTable, bool kPacked, bool kAux, bool kNoLM = false, bool kTiny = false,
          bool kEarly = false, bool kReady = false>
__global__ void __launch_bounds__(256, 1)
    fused_warp_kernel(DevModel m, const float* __restrict__ logits, int64_t row_stride, int32_t B,
                      int32_t* __restrict__ states, int32_t* __restrict__ prev, const uint8_t* __restrict__ active,
                      float lambda, int32_t sp, AuxRow aux, Loop lp, int32_t* __restrict__ tokens_out) {
  constexpr int kW = 8;
  constexpr bool kTwo = kMode == NGPULM_RNNT || kMode == kLoop;  // two-stage transducer selection
  extern __shared__ __align__(16) unsigned char smem[];
  const int32_t V = m.V, ncols = V + 1;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, R = blockDim.x >> 5;
  const size_t mb = kTiny ? tiny_copy_bytes(m.tiny_chain_bytes, m.tiny_arcq_bytes) : 0;
  unsigned char* base = smem + mb + (size_t)w * fslice_bytes(V, m.order);
  WSlice s = wcarve(base, V, m.order, 0);
  if (kTiny) {
    s.chain_s = reinterpret_cast<const int4*>(smem);
    s.st_q = reinterpret_cast<int4*>(smem + align16((size_t)m.tiny_chain_bytes));
  }
  uint64_t* lbar = s.abar;
  float* lbuf = reinterpret_cast<float*>(base + wslice_bytes(V, m.order, 0));
  const int32_t row = (int32_t)blockIdx.x * R + w;
  // plain greedy decoding without an LM (states == nullptr; the baseline of
  // PAPER.md:279) is its own instantiation: a runtime flag here costs 4x (the
  // speculative build no longer overlaps: 3.4 -> 13.8 us at CTC B=256)
  constexpr bool nolm = kNoLM;
  STAMP(0);
  STAMP(1);
  STAMP(9);
  pdl_trigger();
  if constexpr (kTiny) {
    if (threadIdx.x == 0) tiny_copy_issue(m, smem);
    __syncthreads();  // the copy's barrier initialized for every warp
  }
  if (row >= B) return;
  if (lane == 0 && !nolm) {  // root targets -> the row's next-state slots (immutable model data: before the wait)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(s.bar)) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(lbar)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(s.bar)), "r"((uint32_t)V * 4u)
                 : "memory");
    bulk_g2s(s.row_n, m.arc_to, (uint32_t)V * 4u, s.bar);
  }
  if (lane == 0 && nolm) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(lbar)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncwarp();  // lane 0's barrier inits before any other lane's arrive / wait on them
  float4 rw[8];
  if (!nolm) {
    const float4* w4 = reinterpret_cast<const float4*>(m.arc_w);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (lane + 32 * j < V / 4) rw[j] = __ldg(w4 + lane + 32 * j);
  }
  // The LM row of state st into shared memory (no global writes); ph: the
  // parity of this build's root-target copy.
  auto build = [&](int32_t st, uint32_t ph) -> Row {
    WLevel lv;
    int32_t nslots;
    if (kTiny) mbar_wait(tiny_bar(smem, m), 0);  // the CTA's model copy has landed
    const Row r = warp_row_src<kTable, NoOp, ValState, kTiny>(m, ValState{st}, s, lv, nslots);
    if (r.bad) {
      mbar_wait(s.bar, ph);  // the copy of this phase is over before any re-arm or exit
      return r;
    }
    Window<kW, kPacked> a;
    load_window<kW, kPacked, kTiny>(m, s, lv, r.nlev, 0, nslots, a);
    {  // root scores: acc_root + root weight, while the gathers fly
      float4* s4 = reinterpret_cast<float4*>(s.row_s);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (lane + 32 * j < V / 4) {
          float4 y = rw[j];
          y.x = __fadd_rn(r.acc_root, y.x);
          y.y = __fadd_rn(r.acc_root, y.y);
          y.z = __fadd_rn(r.acc_root, y.z);
          y.w = __fadd_rn(r.acc_root, y.w);
          s4[lane + 32 * j] = y;
        }
    }
    mbar_wait(s.bar, ph);
    __syncwarp();
    for (int32_t k0 = 0; k0 < nslots;) {
      write_window<kW, kPacked>(s, a, k0, nslots, m.pk_bits);
      k0 += kW;
      if (k0 < nslots) load_window<kW, kPacked, kTiny>(m, s, lv, r.nlev, k0, nslots, a);
    }
    return r;
  };
  auto load_state = [&]() {
    int32_t v = 0;
    if (lane == 0) asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(states + row) : "memory");
    return __shfl_sync(kFull, v, 0);
  };
  const float* lrow = logits + (size_t)row * row_stride;
  if (kEarly || kReady) {  // the caller guarantees no running kernel writes the logits (NGPULM_STEP_LOGITS_READY)
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));  // read once
    issue_frame_cover(lrow, ncols, lbuf, lbar, pol, logits, logits + (size_t)(B - 1) * row_stride + ncols);
  }
  // Speculative build (as advance_warp_kernel): the LM row from the state read
  // before griddepcontrol.wait, re-checked after it. Inputs (prev, active, ILM
  // rows, and the logits unless kEarly) are read after the wait only.
  int32_t st = 0;
  Row r{};
  if ((NGPULM_FUSED_SPECULATE || kReady) && !nolm) {
    st = load_state();
    r = build(st, 0);
  }
  pdl_wait();
  STAMP(2);
  float ilm[kAux ? kMaxColsPerLane : 1];
  if (kAux) {  // the row's ILM scores, column layout (lane i: columns i, i+32, ...), loads in flight early
    const float* arow = aux.p + (size_t)row * aux.stride;
#pragma unroll
    for (int j = 0; j < kMaxColsPerLane; ++j) {
      const int32_t col = lane + 32 * j;
      ilm[j] = 0.f;
      if (col < ncols && col != sp) ilm[j] = __ldg(arow + (col - (col > sp)));
    }
  }
  // used only after the state and record loads are issued
  const bool on = kMode == kLoop ? __ldg(&lp.frame[row]) < __ldg(&lp.len[row]) : (!active || __ldg(&active[row]));
  const int32_t pc = (kMode == NGPULM_CTC) ? __ldg(&prev[row]) : -2;
  if (on && !(kEarly || kReady)) {  // the logits (an input: after the wait), copied while the state is checked
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));  // read once
    issue_frame_cover(lrow, ncols, lbuf, lbar, pol, logits, logits + (size_t)(B - 1) * row_stride + ncols);
  }
  const float* lb = lbuf + (reinterpret_cast<uintptr_t>(lrow) & 15) / 4;  // column c at lb[c]
  int32_t dsel = -1;  // TDT duration (loop mode with durations), else -1
  if (kMode == kLoop && lp.D > 0 && on) dsel = tdt_duration(lp, row);
  if (!nolm && !kReady) {
    const int32_t st1 = load_state();
    if (!NGPULM_FUSED_SPECULATE || st1 != st) {
      // the root targets again (the first build overwrote them)
      if (NGPULM_FUSED_SPECULATE) rearm_root_targets(s, m.arc_to, (uint32_t)V * 4u);
      st = st1;
      r = build(st, NGPULM_FUSED_SPECULATE ? 1u : 0u);
    }
  }
  STAMP(11);
  if (!on || r.bad) {  // inactive rows are untouched
    if (lane == 0) {
      tokens_out[row] = -1;
      if (on) atomicMin(m.bad_row, (unsigned long long)row);
      if (kMode == kLoop && on) lp.frame[row] = lp.len[row];  // an invalid state ends the row's loop
    }
    if (on || kEarly || kReady) { mbar_wait(lbar, 0); cp_async_settle(); }  // no exit with a copy in flight
    return;
  }
  mbar_wait(lbar, 0);
  cp_async_settle();
  __syncwarp();
  STAMP(12);
  // fused values and the row's argmax (R13, R14, R19):
  // lane i takes columns i, i+32, ... (at most 33 at V <= 1024); two-pass warp
  // argmax (warp_argmax_cols). Transducers: stage 1 = the raw argmax over all
  // columns; blank is kept, else stage 2 = the fused argmax
  // over the non-blank columns.
  int32_t bc;
  {
    float xs[kMaxColsPerLane];
#pragma unroll
    for (int j = 0; j < kMaxColsPerLane; ++j) {
      const int32_t col = lane + 32 * j;
      xs[j] = __int_as_float(0x7fc00000);  // past the last column: NaN, never taken
      if (col < ncols) xs[j] = lb[col];
    }
    int32_t rc = 0;
    if (kTwo) rc = warp_argmax_cols(xs);
    if (kTwo && rc == sp) {
      bc = sp;  // stage 1 keeps blank: no LM advance
    } else {
      const float sp_val = (kMode == NGPULM_AED) ? r.fin : 0.f;  // eos <-> final (lambda * final + asr)
      float val[kMaxColsPerLane];
#pragma unroll
      for (int j = 0; j < kMaxColsPerLane; ++j) {
        const int32_t col = lane + 32 * j;
        const float x = xs[j];
        const float lmv = nolm ? 0.f : col < ncols && col != sp ? s.row_s[col - (col > sp)] : sp_val;
        float v = __fmaf_rn(lambda, lmv, x);  // asr + lambda * lm, one rounding
        if (kAux && col != sp) v = __fmaf_rn(-aux.lam, ilm[j], v);  // - lambda_ilm * ilm (R21)
        if (kMode == NGPULM_CTC && (col == sp || col == pc)) v = x;  // blank raw, repeated token not rescored
        if (kTwo && col == sp) v = __int_as_float(0x7fc00000);        // stage 2: non-blank only
        val[j] = v;
      }
      bc = warp_argmax_cols(val);
    }
  }
  STAMP(7);
  if (kMode == kLoop) {
    if (lane == 0) {
      const bool lab = bc >= 0 && bc < ncols && bc != sp;
      loop_epilogue(lp, row, bc, sp, ncols, states, lab && !nolm ? s.row_n[bc < sp ? bc : bc - 1] : 0, dsel,
                    tokens_out);
    }
    return;
  }
  if (lane == 0) {
    if (bc < 0 || bc >= ncols) {
      tokens_out[row] = -1;  // all-NaN row (unspecified)
    } else {
      tokens_out[row] = bc;
      if (bc == sp) {
        if (kMode == NGPULM_CTC) prev[row] = -1;
      } else if (!(kMode == NGPULM_CTC && bc == pc)) {  // a repeated CTC token: no LM advance
        if (!nolm) states[row] = s.row_n[bc < sp ? bc : bc - 1];
        if (kMode == NGPULM_CTC) prev[row] = bc;
      }
    }
  }
  STAMP(8);
  if (w == 0) STAMPS_OUT(row);
}

// ---------------------------------------------------------------- fused greedy step, two warps per row
// The same step with the row's work split over a warp pair: warp A builds
// the LM row (state, chain record, gathers, level writes) exactly as
// fused_warp_kernel; warp B, which does not need the state, copies the
// logits as soon as the wait allows and computes the transducer's stage 1
// (the raw argmax) while A builds. After a pair barrier each warp evaluates
// half of the columns (lane columns j < 17 / j >= 17) and the two halves'
// winners are merged through shared memory (R14 order). Used for the
// transducer modes while there are at most 4 rows per SM (CTC and AED have
// no stage 1 to overlap: for them the pair's barriers cost more than the
// halved argmax saves).
constexpr int kPairSplit = 17;

template <int kMode, bool kTable, bool kPacked, bool kAux, bool kNoLM = false>
__global__ void __launch_bounds__(256, 1)
    fused_pair_kernel(DevModel m, const float* __restrict__ logits, int64_t row_stride, int32_t B,
                      int32_t* __restrict__ states, int32_t* __restrict__ prev, const uint8_t* __restrict__ active,
                      float lambda, int32_t sp, AuxRow aux, Loop lp, int32_t* __restrict__ tokens_out) {
  constexpr int kW = 8;
  constexpr bool kTwo = kMode == NGPULM_RNNT || kMode == kLoop;
  extern __shared__ __align__(16) unsigned char smem[];
  const int32_t V = m.V, ncols = V + 1;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, pair = w >> 1, role = w & 1, R = blockDim.x >> 6;
  unsigned char* base = smem + (size_t)pair * (fslice_bytes(V, m.order) + 64);
  const WSlice s = wcarve(base, V, m.order, 0);
  uint64_t* lbar = s.abar;
  float* lbuf = reinterpret_cast<float*>(base + wslice_bytes(V, m.order, 0));
  volatile int32_t* xch = reinterpret_cast<int32_t*>(base + fslice_bytes(V, m.order));  // exchange words
  const int32_t row = (int32_t)blockIdx.x * R + pair;
  const uint32_t bid = 1 + pair;  // named barrier of the pair (0 is __syncthreads)
  auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(bid) : "memory"); };
  constexpr bool nolm = kNoLM;  // plain greedy decoding (no LM)
  pdl_trigger();
  if (row >= B) return;
  if (lane == 0) {  // A: root targets -> next-state slots; B: the logits barrier (model data / no inputs: before the wait)
    const uint64_t* bb = role == 0 ? s.bar : lbar;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bb)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (role == 0 && !nolm) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(s.bar)),
                   "r"((uint32_t)V * 4u)
                   : "memory");
      bulk_g2s(s.row_n, m.arc_to, (uint32_t)V * 4u, s.bar);
    }
  }
  __syncwarp();  // lane 0's barrier init before any other lane's arrive / wait on it
  float4 rw[8];
  if (role == 0 && !nolm) {
    const float4* w4 = reinterpret_cast<const float4*>(m.arc_w);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (lane + 32 * j < V / 4) rw[j] = __ldg(w4 + lane + 32 * j);
  }
  pdl_wait();
  const float* lrow = logits + (size_t)row * row_stride;
  const float* lb = lbuf + (reinterpret_cast<uintptr_t>(lrow) & 15) / 4;  // column c at lb[c]
  const bool on = kMode == kLoop ? __ldg(&lp.frame[row]) < __ldg(&lp.len[row]) : (!active || __ldg(&active[row]));
  const int32_t pc = (kMode == NGPULM_CTC) ? __ldg(&prev[row]) : -2;
  float ilm[kAux ? kMaxColsPerLane : 1];
  if (kAux) {  // this warp's half of the row's ILM scores
    const float* arow = aux.p + (size_t)row * aux.stride;
#pragma unroll
    for (int j = 0; j < kMaxColsPerLane; ++j) {
      const int32_t col = lane + 32 * j;
      ilm[j] = 0.f;
      if ((j < kPairSplit) == (role == 0) && col < ncols && col != sp) ilm[j] = __ldg(arow + (col - (col > sp)));
    }
  }
  float xs[kMaxColsPerLane];
  float fin = 0.f;
  if (role == 1) {
    if (on) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      issue_frame_cover(lrow, ncols, lbuf, lbar, pol, logits, logits + (size_t)(B - 1) * row_stride + ncols);
      mbar_wait(lbar, 0);
      cp_async_settle();
#pragma unroll
      for (int j = 0; j < kMaxColsPerLane; ++j) {
        const int32_t col = lane + 32 * j;
        xs[j] = __int_as_float(0x7fc00000);
        if ((kTwo || j >= kPairSplit) && col < ncols) xs[j] = lb[col];
      }
      if (kTwo) {
        const int32_t rc = warp_argmax_cols(xs);  // stage 1: standard greedy prediction
        if (lane == 0) xch[2] = rc;
      }
      if (kMode == kLoop && lp.D > 0) {  // TDT: the duration, beside the row build
        const int32_t d = tdt_duration(lp, row);
        if (lane == 0) xch[9] = d;
      }
    }
    pair_sync();  // (1) the row is built (or the row is done)
    if (xch[3]) return;
    fin = __int_as_float(xch[4]);
  } else {
    WLevel lv;
    int32_t nslots = 0;
    Row r{};
    if (!nolm) r = warp_row<kTable>(m, states + row, s, lv, nslots);
    if (!on || r.bad) {
      if (lane == 0) {
        tokens_out[row] = -1;
        if (on) atomicMin(m.bad_row, (unsigned long long)row);
        if (kMode == kLoop && on) lp.frame[row] = lp.len[row];
        xch[3] = 1;
      }
      if (!nolm) mbar_wait(s.bar, 0);
      pair_sync();
      return;
    }
    if (!nolm) {
    Window<kW, kPacked> a;
    load_window<kW, kPacked>(m, s, lv, r.nlev, 0, nslots, a);
    {
      float4* s4 = reinterpret_cast<float4*>(s.row_s);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (lane + 32 * j < V / 4) {
          float4 y = rw[j];
          y.x = __fadd_rn(r.acc_root, y.x);
          y.y = __fadd_rn(r.acc_root, y.y);
          y.z = __fadd_rn(r.acc_root, y.z);
          y.w = __fadd_rn(r.acc_root, y.w);
          s4[lane + 32 * j] = y;
        }
    }
    mbar_wait(s.bar, 0);
    __syncwarp();
    for (int32_t k0 = 0; k0 < nslots;) {
      write_window<kW, kPacked>(s, a, k0, nslots, m.pk_bits);
      k0 += kW;
      if (k0 < nslots) load_window<kW, kPacked>(m, s, lv, r.nlev, k0, nslots, a);
    }
    }
    fin = r.fin;
    if (lane == 0) {
      xch[3] = 0;
      xch[4] = __float_as_int(r.fin);
    }
    pair_sync();  // (1)
    mbar_wait(lbar, 0);  // the logits (B saw them land; observe the phase here too)
#pragma unroll
    for (int j = 0; j < kPairSplit; ++j) {
      const int32_t col = lane + 32 * j;
      xs[j] = __int_as_float(0x7fc00000);
      if (col < ncols) xs[j] = lb[col];
    }
  }
  const int32_t rc = kTwo ? xch[2] : 0;
  int32_t bc;
  if (kTwo && rc == sp) {
    bc = sp;  // stage 1 keeps blank
    if (role == 1) return;
  } else {
    const float sp_val = (kMode == NGPULM_AED) ? fin : 0.f;
    float val[kMaxColsPerLane];
#pragma unroll
    for (int j = 0; j < kMaxColsPerLane; ++j) {
      const int32_t col = lane + 32 * j;
      const float x = xs[j];
      float v = __int_as_float(0x7fc00000);
      if ((j < kPairSplit) == (role == 0)) {
        const float lmv = nolm ? 0.f : col < ncols && col != sp ? s.row_s[col - (col > sp)] : sp_val;
        v = __fmaf_rn(lambda, lmv, x);
        if (kAux && col != sp) v = __fmaf_rn(-aux.lam, ilm[j], v);
        if (kMode == NGPULM_CTC && (col == sp || col == pc)) v = x;
        if (kTwo && col == sp) v = __int_as_float(0x7fc00000);
      }
      val[j] = v;
    }
    float M;
    const int32_t c = role == 0 ? warp_argmax_range<0, kPairSplit>(val, M)
                                : warp_argmax_range<kPairSplit, kMaxColsPerLane>(val, M);
    if (lane == 0) {
      xch[5 + 2 * role] = __float_as_int(M);
      xch[6 + 2 * role] = c;
    }
    pair_sync();  // (2) both halves' winners
    if (role == 1) return;
    const float M1 = __int_as_float(xch[7]);
    const int32_t c1 = xch[8];
    bc = (M1 > M || (M1 == M && c1 < c)) ? c1 : c;  // (B's columns are all higher; equal values: lower column)
  }
  if (kMode == kLoop) {
    if (lane == 0) {
      const bool lab = bc >= 0 && bc < ncols && bc != sp;
      loop_epilogue(lp, row, bc, sp, ncols, states, lab && !nolm ? s.row_n[bc < sp ? bc : bc - 1] : 0,
                    lp.D > 0 ? xch[9] : -1, tokens_out);
    }
    return;
  }
  if (lane == 0) {
    if (bc < 0 || bc >= ncols) {
      tokens_out[row] = -1;
    } else {
      tokens_out[row] = bc;
      if (bc == sp) {
        if (kMode == NGPULM_CTC) prev[row] = -1;
      } else if (!(kMode == NGPULM_CTC && bc == pc)) {
        if (!nolm) states[row] = s.row_n[bc < sp ? bc : bc - 1];
        if (kMode == NGPULM_CTC) prev[row] = bc;
      }
    }
  }
}

// ---------------------------------------------------------------- fused step from precomputed LM rows
// Overlap mode: in a decode loop the LM query of step t needs
// only the states left by step t-1, not step t's logits, so the caller issues
// ngpulm_advance(states) on a second stream while its network computes the
// logits, and this kernel then makes the mode's decision from the two rows
// (R13, R14, R19): one warp per row, lane i takes
// columns i, i+32, ... of the logits and the LM row (coalesced loads, all in
// flight together), the two-pass warp argmax, and one gather of the winning
// token's next state. A row whose LM row is marked invalid (next = -1, written
// by the advance for an out-of-range state) gets token -1 and is untouched.
template <int kMode>
__global__ void __launch_bounds__(256)
    fused_rows_kernel(const float* __restrict__ logits, int64_t row_stride, const float* __restrict__ lm_s,
                      const int32_t* __restrict__ lm_n, const float* __restrict__ lm_f, int64_t lm_stride, int32_t B,
                      int32_t V, int32_t* __restrict__ states, int32_t* __restrict__ prev,
                      const uint8_t* __restrict__ active, float lambda, int32_t sp, int32_t* __restrict__ tokens_out) {
  constexpr bool kTwo = kMode == NGPULM_RNNT;
  const int lane = threadIdx.x & 31;
  const int32_t row = (int32_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), ncols = V + 1;
  pdl_trigger();
  pdl_wait();  // logits, LM rows, states and prev all come from preceding kernels
  if (row >= B) return;
  if (active && !__ldg(&active[row])) {
    if (lane == 0) tokens_out[row] = -1;
    return;
  }
  const float* lrow = logits + (size_t)row * row_stride;
  const float* srow = lm_s + (size_t)row * lm_stride;
  const int32_t* nrow = lm_n + (size_t)row * lm_stride;
  const int32_t valid = __ldg(nrow);  // -1: the advance saw an invalid state
  const int32_t pc = (kMode == NGPULM_CTC) ? __ldg(&prev[row]) : -2;
  const float sp_val = (kMode == NGPULM_AED) ? __ldg(&lm_f[row]) : 0.f;  // eos <-> final
  float xs[kMaxColsPerLane], lm[kMaxColsPerLane];
#pragma unroll
  for (int j = 0; j < kMaxColsPerLane; ++j) {
    const int32_t col = lane + 32 * j;
    xs[j] = __int_as_float(0x7fc00000);  // past the last column: NaN, never taken
    lm[j] = sp_val;
    if (col < ncols) {
      xs[j] = __ldg(lrow + col);
      if (col != sp) lm[j] = __ldg(srow + (col - (col > sp)));
    }
  }
  if (valid < 0) {
    if (lane == 0) tokens_out[row] = -1;
    return;
  }
  int32_t bc;
  const int32_t rc = kTwo ? warp_argmax_cols(xs) : 0;  // stage 1
  if (kTwo && rc == sp) {
    bc = sp;
  } else {
    float val[kMaxColsPerLane];
#pragma unroll
    for (int j = 0; j < kMaxColsPerLane; ++j) {
      const int32_t col = lane + 32 * j;
      float v = __fmaf_rn(lambda, lm[j], xs[j]);                    // asr + lambda * lm, one rounding
      if (kMode == NGPULM_CTC && (col == sp || col == pc)) v = xs[j];  // blank raw, repeated token not rescored
      if (kTwo && col == sp) v = __int_as_float(0x7fc00000);           // stage 2: non-blank only
      val[j] = v;
    }
    bc = warp_argmax_cols(val);
  }
  if (lane == 0) {
    if (bc < 0 || bc >= ncols) {
      tokens_out[row] = -1;
    } else {
      tokens_out[row] = bc;
      if (bc == sp) {
        if (kMode == NGPULM_CTC) prev[row] = -1;
      } else if (!(kMode == NGPULM_CTC && bc == pc)) {
        states[row] = __ldg(nrow + (bc < sp ? bc : bc - 1));
        if (kMode == NGPULM_CTC) prev[row] = bc;
      }
    }
  }
}

// ---------------------------------------------------------------- fused top-k
// The k best expansions of each row for AED beam search with NGPU-LM fusion
// ("greedy and beam search"): fused values over all V+1
// columns by the AED rule (token columns fmaf(lambda, lm, asr) [- lambda_ilm
// * ilm], eos column fmaf(lambda, final(state), asr[eos])), sorted by value
// descending, lowest column first on ties, NaN never selected. Row build and
// logits staging as in fused_warp_kernel; k rounds of a two-pass warp
// argmax over the values held in registers.
template <bool kTable, bool kPacked>
__global__ void __launch_bounds__(256, 1)
    topk_warp_kernel(DevModel m, const float* __restrict__ logits, int64_t row_stride, int32_t B,
                     const int32_t* __restrict__ states, float lambda, int32_t sp, AuxRow aux, int32_t k,
                     float* __restrict__ out_scores, int32_t* __restrict__ out_cols, int32_t* __restrict__ out_next) {
  constexpr int kW = 8;
  extern __shared__ __align__(16) unsigned char smem[];
  const int32_t V = m.V, ncols = V + 1;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, R = blockDim.x >> 5;
  unsigned char* base = smem + (size_t)w * fslice_bytes(V, m.order);
  const WSlice s = wcarve(base, V, m.order, 0);
  uint64_t* lbar = s.abar;
  float* lbuf = reinterpret_cast<float*>(base + wslice_bytes(V, m.order, 0));
  const int32_t row = (int32_t)blockIdx.x * R + w;
  pdl_trigger();
  if (row >= B) return;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(s.bar)) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(lbar)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(s.bar)), "r"((uint32_t)V * 4u)
                 : "memory");
    bulk_g2s(s.row_n, m.arc_to, (uint32_t)V * 4u, s.bar);
  }
  __syncwarp();  // lane 0's barrier inits before any other lane's arrive / wait on them
  float4 rw[8];
  {
    const float4* w4 = reinterpret_cast<const float4*>(m.arc_w);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (lane + 32 * j < V / 4) rw[j] = __ldg(w4 + lane + 32 * j);
  }
  pdl_wait();
  const float* lrow = logits + (size_t)row * row_stride;
  float ilm[kMaxColsPerLane];
#pragma unroll
  for (int j = 0; j < kMaxColsPerLane; ++j) {
    const int32_t col = lane + 32 * j;
    ilm[j] = 0.f;
    if (aux.p && col < ncols && col != sp) ilm[j] = __ldg(aux.p + (size_t)row * aux.stride + (col - (col > sp)));
  }
  WLevel lv;
  int32_t nslots;
  bool started = false;
  auto begin_logits = [&]() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    issue_frame_cover(lrow, ncols, lbuf, lbar, pol, logits, logits + (size_t)(B - 1) * row_stride + ncols);
    started = true;
  };
  const Row r = warp_row<kTable>(m, states + row, s, lv, nslots, begin_logits);
  const float* lb = lbuf + (reinterpret_cast<uintptr_t>(lrow) & 15) / 4;  // column c at lb[c]
  float* osc = out_scores + (size_t)row * k;
  int32_t* ocol = out_cols + (size_t)row * k;
  int32_t* onx = out_next ? out_next + (size_t)row * k : nullptr;
  if (r.bad) {
    if (lane == 0) atomicMin(m.bad_row, (unsigned long long)row);
    for (int32_t i = lane; i < k; i += 32) {
      osc[i] = __int_as_float(0x7fc00000);
      ocol[i] = -1;
      if (onx) onx[i] = -1;
    }
    mbar_wait(s.bar, 0);
    if (started) { mbar_wait(lbar, 0); cp_async_settle(); }
    return;
  }
  Window<kW, kPacked> a;
  load_window<kW, kPacked>(m, s, lv, r.nlev, 0, nslots, a);
  {
    float4* s4 = reinterpret_cast<float4*>(s.row_s);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (lane + 32 * j < V / 4) {
        float4 y = rw[j];
        y.x = __fadd_rn(r.acc_root, y.x);
        y.y = __fadd_rn(r.acc_root, y.y);
        y.z = __fadd_rn(r.acc_root, y.z);
        y.w = __fadd_rn(r.acc_root, y.w);
        s4[lane + 32 * j] = y;
      }
  }
  mbar_wait(s.bar, 0);
  __syncwarp();
  for (int32_t k0 = 0; k0 < nslots;) {
    write_window<kW, kPacked>(s, a, k0, nslots, m.pk_bits);
    k0 += kW;
    if (k0 < nslots) load_window<kW, kPacked>(m, s, lv, r.nlev, k0, nslots, a);
  }
  mbar_wait(lbar, 0);
  cp_async_settle();
  __syncwarp();
  float val[kMaxColsPerLane];
#pragma unroll
  for (int j = 0; j < kMaxColsPerLane; ++j) {
    const int32_t col = lane + 32 * j;
    float x = __int_as_float(0x7fc00000);
    float v = x;
    if (col < ncols) {
      x = lb[col];
      if (col == sp) {
        v = __fmaf_rn(lambda, r.fin, x);  // eos <-> final weight
      } else {
        v = __fmaf_rn(lambda, s.row_s[col - (col > sp)], x);
        if (aux.p) v = __fmaf_rn(-aux.lam, ilm[j], v);
      }
    }
    val[j] = v;
  }
  for (int32_t i = 0; i < k; ++i) {
    const int32_t bc = warp_argmax_cols(val);
    if (bc == INT_MAX) {  // fewer than k selectable (non-NaN) columns
      if (lane == 0) { osc[i] = -INFINITY; ocol[i] = -1; if (onx) onx[i] = -1; }
      continue;
    }
    float mine = 0.f;
#pragma unroll
    for (int j = 0; j < kMaxColsPerLane; ++j)
      if (lane + 32 * j == bc) {
        mine = val[j];
        val[j] = __int_as_float(0x7fc00000);  // taken
      }
    const float M = __shfl_sync(kFull, mine, bc & 31);
    if (lane == 0) {
      osc[i] = M;
      ocol[i] = bc;
      if (onx) onx[i] = bc == sp ? r.state : s.row_n[bc - (bc > sp)];
    }
  }
}

}  // namespace

template <int kMode>
int launch_fused_mode(const DevModel& m, const float* logits, int64_t row_stride, int32_t B, int32_t* states,
                      int32_t* prev, const uint8_t* active, float lambda, int32_t blank, AuxRow aux,
                      int32_t* tokens_out, cudaStream_t st, uint32_t flags) {
  // (permissions: other paths ignore them; inputs ready implies logits ready)
  const bool early = (flags & (NGPULM_STEP_LOGITS_READY | NGPULM_STEP_INPUTS_READY)) && !aux.p;
  if (m.V % 4 == 0 && m.V <= 1024 && m.adv_kind != NGPULM_ADVANCE_CTA) {
    const bool pk = m.arc_q != nullptr && m.adv_kind == NGPULM_ADVANCE_AUTO, table = m.chain != nullptr;
    if (states == nullptr) {  // plain greedy (no LM): one warp per row, no row build
      int R = (B + 147) / 148;
      R = R < 1 ? 1 : (R > NGPULM_FUSED_MAX_ROWS ? NGPULM_FUSED_MAX_ROWS : R);
      if (early)
        return launch(fused_warp_kernel<kMode, true, true, false, true, false, true>, dim3((B + R - 1) / R),
                      dim3(32 * R), (size_t)R * fslice_bytes(m.V, m.order), st, m, logits, row_stride, B, states,
                      prev, active, lambda, blank, aux, Loop{}, tokens_out);
      return launch(fused_warp_kernel<kMode, true, true, false, true>, dim3((B + R - 1) / R), dim3(32 * R),
                    (size_t)R * fslice_bytes(m.V, m.order), st, m, logits, row_stride, B, states, prev, active,
                    lambda, blank, aux, Loop{}, tokens_out);
    }
    if (table && pk && m.tiny_chain_bytes > 0) {  // tiny LM: the model in every CTA's shared memory
      const size_t mb = tiny_copy_bytes(m.tiny_chain_bytes, m.tiny_arcq_bytes);
      int R = (B + 147) / 148;
      R = R < 1 ? 1 : (R > NGPULM_FUSED_MAX_ROWS ? NGPULM_FUSED_MAX_ROWS : R);
      while (R > 1 && mb + (size_t)R * fslice_bytes(m.V, m.order) > 227 * 1024) --R;
      const size_t tsm = mb + (size_t)R * fslice_bytes(m.V, m.order);
      if (tsm <= 227 * 1024) {
        const dim3 tg((B + R - 1) / R), tb(32 * R);
        if (early)
          return launch(fused_warp_kernel<kMode, true, true, false, false, true, true>, tg, tb, tsm, st, m, logits,
                        row_stride, B, states, prev, active, lambda, blank, aux, Loop{}, tokens_out);
        return aux.p ? launch(fused_warp_kernel<kMode, true, true, true, false, true>, tg, tb, tsm, st, m, logits,
                              row_stride, B, states, prev, active, lambda, blank, aux, Loop{}, tokens_out)
                     : launch(fused_warp_kernel<kMode, true, true, false, false, true>, tg, tb, tsm, st, m, logits,
                              row_stride, B, states, prev, active, lambda, blank, aux, Loop{}, tokens_out);
      }
    }
    if ((flags & NGPULM_STEP_INPUTS_READY) && !aux.p && table && pk) {  // every mode: one warp per row
      int R = (B + 147) / 148;
      R = R < 1 ? 1 : (R > NGPULM_FUSED_MAX_ROWS ? NGPULM_FUSED_MAX_ROWS : R);
      return launch(fused_warp_kernel<kMode, true, true, false, false, false, false, true>, dim3((B + R - 1) / R),
                    dim3(32 * R), (size_t)R * fslice_bytes(m.V, m.order), st, m, logits, row_stride, B, states, prev,
                    active, lambda, blank, aux, Loop{}, tokens_out);
    }
    if (kMode != NGPULM_RNNT || B > NGPULM_PAIR_MAX_B) if (early && table && pk) {
      int R = (B + 147) / 148;
      R = R < 1 ? 1 : (R > NGPULM_FUSED_MAX_ROWS ? NGPULM_FUSED_MAX_ROWS : R);
      return launch(fused_warp_kernel<kMode, true, true, false, false, false, true>, dim3((B + R - 1) / R),
                    dim3(32 * R), (size_t)R * fslice_bytes(m.V, m.order), st, m, logits, row_stride, B, states, prev,
                    active, lambda, blank, aux, Loop{}, tokens_out);
    }
    if constexpr (kMode == NGPULM_RNNT) if (B <= NGPULM_PAIR_MAX_B) {  // two warps per row (stage 1 beside the row build)
      int R = (B + 147) / 148;
      R = R < 1 ? 1 : (R > 4 ? 4 : R);
      const size_t psm = (size_t)R * (fslice_bytes(m.V, m.order) + 64);
      const dim3 pg((B + R - 1) / R), pb(64 * R);
#define NGPULM_PAIR_LAUNCH(T, P)                                                                                  \
  return aux.p ? launch(fused_pair_kernel<kMode, T, P, true>, pg, pb, psm, st, m, logits, row_stride, B, states,   \
                        prev, active, lambda, blank, aux, Loop{}, tokens_out)                                      \
               : launch(fused_pair_kernel<kMode, T, P, false>, pg, pb, psm, st, m, logits, row_stride, B, states,  \
                        prev, active, lambda, blank, aux, Loop{}, tokens_out)
      if (table) { if (pk) NGPULM_PAIR_LAUNCH(true, true); NGPULM_PAIR_LAUNCH(true, false); }
      if (pk) NGPULM_PAIR_LAUNCH(false, true);
      NGPULM_PAIR_LAUNCH(false, false);
#undef NGPULM_PAIR_LAUNCH
    }
    int R = (B + 147) / 148;
    R = R < 1 ? 1 : (R > NGPULM_FUSED_MAX_ROWS ? NGPULM_FUSED_MAX_ROWS : R);
    const size_t wsm = (size_t)R * fslice_bytes(m.V, m.order);
    const dim3 wg((B + R - 1) / R), wb(32 * R);
#define NGPULM_FUSED_LAUNCH(T, P)                                                                                 \
  return aux.p ? launch(fused_warp_kernel<kMode, T, P, true>, wg, wb, wsm, st, m, logits, row_stride, B, states,    \
                        prev, active, lambda, blank, aux, Loop{}, tokens_out)                                       \
               : launch(fused_warp_kernel<kMode, T, P, false>, wg, wb, wsm, st, m, logits, row_stride, B, states,   \
                        prev, active, lambda, blank, aux, Loop{}, tokens_out)
    if (table) { if (pk) NGPULM_FUSED_LAUNCH(true, true); NGPULM_FUSED_LAUNCH(true, false); }
    if (pk) NGPULM_FUSED_LAUNCH(false, true);
    NGPULM_FUSED_LAUNCH(false, false);
#undef NGPULM_FUSED_LAUNCH
  }
  const size_t sm = row_smem(m.V, m.order);
  const dim3 gd(B), bd(kThreads);
  if (m.chain != nullptr)
    return launch(fused_kernel<kMode, true>, gd, bd, sm, st, m, logits, row_stride, states, prev, active, lambda,
                  blank, aux, tokens_out);
  return launch(fused_kernel<kMode, false>, gd, bd, sm, st, m, logits, row_stride, states, prev, active, lambda,
                blank, aux, tokens_out);
}

int launch_fused(const DevModel& m, int32_t mode, const float* logits, int64_t row_stride, int32_t B,
                 int32_t* states, int32_t* prev, const uint8_t* active, float lambda, int32_t blank,
                 const float* aux, int64_t aux_stride, float lambda_ilm, int32_t* tokens_out, void* stream,
                 uint32_t flags) {
  cudaStream_t st = (cudaStream_t)stream;
  const AuxRow ax{aux, aux_stride, lambda_ilm};
  switch (mode) {
    case NGPULM_CTC:
      return launch_fused_mode<NGPULM_CTC>(m, logits, row_stride, B, states, prev, active, lambda, blank, ax,
                                           tokens_out, st, flags);
    case NGPULM_RNNT:
      return launch_fused_mode<NGPULM_RNNT>(m, logits, row_stride, B, states, prev, active, lambda, blank, ax,
                                            tokens_out, st, flags);
    default:
      return launch_fused_mode<NGPULM_AED>(m, logits, row_stride, B, states, prev, active, lambda, blank, ax,
                                           tokens_out, st, flags);
  }
}

int launch_fused_rows(int32_t mode, const float* logits, int64_t row_stride, const float* lm_s, const int32_t* lm_n,
                      const float* lm_f, int64_t lm_stride, int32_t B, int32_t V, int32_t* states, int32_t* prev,
                      const uint8_t* active, float lambda, int32_t blank, int32_t* tokens_out, void* stream) {
  if (V > 1024) return (int)cudaErrorNotSupported;
  const dim3 g((B + 7) / 8), b(256);
  cudaStream_t st = (cudaStream_t)stream;
  switch (mode) {
    case NGPULM_CTC:
      return launch(fused_rows_kernel<NGPULM_CTC>, g, b, 0, st, logits, row_stride, lm_s, lm_n, lm_f, lm_stride, B, V,
                    states, prev, active, lambda, blank, tokens_out);
    case NGPULM_RNNT:
      return launch(fused_rows_kernel<NGPULM_RNNT>, g, b, 0, st, logits, row_stride, lm_s, lm_n, lm_f, lm_stride, B,
                    V, states, prev, active, lambda, blank, tokens_out);
    default:
      return launch(fused_rows_kernel<NGPULM_AED>, g, b, 0, st, logits, row_stride, lm_s, lm_n, lm_f, lm_stride, B, V,
                    states, prev, active, lambda, blank, tokens_out);
  }
}

int launch_transducer_loop(const DevModel& m, const float* logits, int64_t row_stride, int32_t B, int32_t* states,
                           int32_t* frame, int32_t* sym, const int32_t* lengths, int32_t max_sym, float lambda,
                           int32_t blank, const float* aux, int64_t aux_stride, float lambda_ilm,
                           int32_t* tokens_out, int32_t* emit, int32_t* emit_len, int32_t* last, int32_t max_len,
                           const float* dur, int64_t dur_stride, const int32_t* durations, int32_t D,
                           uint32_t flags, void* stream) {
  if (m.V % 4 != 0 || m.V > 1024) return (int)cudaErrorNotSupported;
  const bool ready = (flags & NGPULM_STEP_INPUTS_READY) != 0;
  int R = (B + 147) / 148;
  R = R < 1 ? 1 : (R > 8 ? 8 : R);
  const size_t wsm = (size_t)R * fslice_bytes(m.V, m.order);
  const dim3 wg((B + R - 1) / R), wb(32 * R);
  const bool pk = m.arc_q != nullptr && m.adv_kind == NGPULM_ADVANCE_AUTO, table = m.chain != nullptr;
  const AuxRow ax{aux, aux_stride, lambda_ilm};
  Loop lp{frame, sym, lengths, emit, emit_len, last, max_sym, max_len, dur, dur_stride, D, {}};
  for (int32_t j = 0; j < D && j < kMaxDur; ++j) lp.durs[j] = durations[j];
  cudaStream_t st = (cudaStream_t)stream;
  if (states == nullptr) {  // plain greedy label looping (no LM)
    if (ready && !aux)  // (inputs ready: the logits copied at the kernel's start)
      return launch(fused_warp_kernel<kLoop, true, true, false, true, false, true>, wg, wb, wsm, st, m, logits,
                    row_stride, B, states, (int32_t*)nullptr, (const uint8_t*)nullptr, lambda, blank, ax, lp,
                    tokens_out);
    return launch(fused_warp_kernel<kLoop, true, true, false, true>, wg, wb, wsm, st, m, logits, row_stride, B, states,
                  (int32_t*)nullptr, (const uint8_t*)nullptr, lambda, blank, ax, lp, tokens_out);
  }
  if (table && pk && m.tiny_chain_bytes > 0) {  // tiny LM: the model in every CTA's shared memory
    const size_t mb = tiny_copy_bytes(m.tiny_chain_bytes, m.tiny_arcq_bytes);
    int Rt = R;
    while (Rt > 1 && mb + (size_t)Rt * fslice_bytes(m.V, m.order) > 227 * 1024) --Rt;
    const size_t tsm = mb + (size_t)Rt * fslice_bytes(m.V, m.order);
    if (tsm <= 227 * 1024) {
      const dim3 tg((B + Rt - 1) / Rt), tb(32 * Rt);
      return aux ? launch(fused_warp_kernel<kLoop, true, true, true, false, true>, tg, tb, tsm, st, m, logits,
                          row_stride, B, states, (int32_t*)nullptr, (const uint8_t*)nullptr, lambda, blank, ax, lp,
                          tokens_out)
                 : launch(fused_warp_kernel<kLoop, true, true, false, false, true>, tg, tb, tsm, st, m, logits,
                          row_stride, B, states, (int32_t*)nullptr, (const uint8_t*)nullptr, lambda, blank, ax, lp,
                          tokens_out);
    }
  }
  // inputs ready (NGPULM_STEP_INPUTS_READY) beyond the warp-pair range: one warp per row without the state
  // re-read. Up to 4 rows per SM the pair kernel stays: it reads its inputs after the wait only (no
  // speculation to re-check), and in the label loop (B = 512, mostly-blank rows) its stage 1 beside the
  // row build measured faster than one warp per row with the flag (1.53 vs 1.55 ms)
  if (ready && !aux && table && pk && B > NGPULM_PAIR_MAX_B)
    return launch(fused_warp_kernel<kLoop, true, true, false, false, false, false, true>, wg, wb, wsm, st, m, logits,
                  row_stride, B, states, (int32_t*)nullptr, (const uint8_t*)nullptr, lambda, blank, ax, lp,
                  tokens_out);
  if (B <= NGPULM_PAIR_MAX_B) {  // two warps per row
    int Rp = (B + 147) / 148;
    Rp = Rp < 1 ? 1 : (Rp > 4 ? 4 : Rp);
    const size_t psm = (size_t)Rp * (fslice_bytes(m.V, m.order) + 64);
    const dim3 pg((B + Rp - 1) / Rp), pb(64 * Rp);
#define NGPULM_PAIR_LOOP(T, P)                                                                                     \
  return aux ? launch(fused_pair_kernel<kLoop, T, P, true>, pg, pb, psm, st, m, logits, row_stride, B, states,      \
                      (int32_t*)nullptr, (const uint8_t*)nullptr, lambda, blank, ax, lp, tokens_out)                \
             : launch(fused_pair_kernel<kLoop, T, P, false>, pg, pb, psm, st, m, logits, row_stride, B, states,     \
                      (int32_t*)nullptr, (const uint8_t*)nullptr, lambda, blank, ax, lp, tokens_out)
    if (table) { if (pk) NGPULM_PAIR_LOOP(true, true); NGPULM_PAIR_LOOP(true, false); }
    if (pk) NGPULM_PAIR_LOOP(false, true);
    NGPULM_PAIR_LOOP(false, false);
#undef NGPULM_PAIR_LOOP
  }
#define NGPULM_LOOP_LAUNCH(T, P)                                                                                     \
  return aux ? launch(fused_warp_kernel<kLoop, T, P, true>, wg, wb, wsm, st, m, logits, row_stride, B, states,       \
                      (int32_t*)nullptr, (const uint8_t*)nullptr, lambda, blank, ax, lp, tokens_out)                 \
             : launch(fused_warp_kernel<kLoop, T, P, false>, wg, wb, wsm, st, m, logits, row_stride, B, states,      \
                      (int32_t*)nullptr, (const uint8_t*)nullptr, lambda, blank, ax, lp, tokens_out)
  if (table) { if (pk) NGPULM_LOOP_LAUNCH(true, true); NGPULM_LOOP_LAUNCH(true, false); }
  if (pk) NGPULM_LOOP_LAUNCH(false, true);
  NGPULM_LOOP_LAUNCH(false, false);
#undef NGPULM_LOOP_LAUNCH
}

int launch_topk(const DevModel& m, const float* logits, int64_t row_stride, int32_t B, const int32_t* states,
                const float* aux, int64_t aux_stride, float lambda, float lambda_ilm, int32_t eos, int32_t k,
                float* out_scores, int32_t* out_cols, int32_t* out_next, void* stream) {
  if (m.V % 4 != 0 || m.V > 1024) return (int)cudaErrorNotSupported;
  int R = (B + 147) / 148;
  R = R < 1 ? 1 : (R > 8 ? 8 : R);
  const size_t wsm = (size_t)R * fslice_bytes(m.V, m.order);
  const dim3 wg((B + R - 1) / R), wb(32 * R);
  const bool pk = m.arc_q != nullptr && m.adv_kind == NGPULM_ADVANCE_AUTO, table = m.chain != nullptr;
  const AuxRow ax{aux, aux_stride, lambda_ilm};
  cudaStream_t st = (cudaStream_t)stream;
#define NGPULM_TOPK_LAUNCH(T, P)                                                                                   \
  return launch(topk_warp_kernel<T, P>, wg, wb, wsm, st, m, logits, row_stride, B, states, lambda, eos, ax, k, \
                out_scores, out_cols, out_next)
  if (table) { if (pk) NGPULM_TOPK_LAUNCH(true, true); NGPULM_TOPK_LAUNCH(true, false); }
  if (pk) NGPULM_TOPK_LAUNCH(false, true);
  NGPULM_TOPK_LAUNCH(false, false);
#undef NGPULM_TOPK_LAUNCH
}

}  // namespace ngpulm
