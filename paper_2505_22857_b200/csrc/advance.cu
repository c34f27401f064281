// NGPU-LM batched full-vocabulary query (Algorithm 1) for sm_100a:
// the advance kernels (warp per row with the speculative pre-wait build, tiny
// LMs in shared memory, CTA per row / vocabulary tile), the final-weight
// gather, and their launchers. Design: kcommon.cuh, DESIGN.md §7.
#include "kcommon.cuh"

namespace ngpulm {
namespace {

// ---------------------------------------------------------------- advance
// Vocabulary tiling: when a row does not fit in shared
// memory, CTA (b, y) answers tokens [y * tile, y * tile + tv) of row b —
// Algorithm 1 restricted to the tile is exact (each token's value depends only
// on the arcs for that token); every CTA reads the row's full arc list and
// keeps its tile's tokens.
template <bool kVec4, bool kTable>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
    advance_kernel(DevModel m, const int32_t* __restrict__ states, float* __restrict__ scores,
                   int32_t* __restrict__ next, float* __restrict__ final_out, int32_t tile) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int32_t b = blockIdx.x, t0 = (int32_t)blockIdx.y * tile, V = min(tile, m.V - t0);
  const int t = threadIdx.x;
  const Slice s = carve(smem, V, m.order);
  STAMP(0);
  STAMP(1);
  STAMP(9);
  pdl_trigger();
#ifdef NGPULM_PHASE_TIMING
  const bool use_tma = kVec4 && !(g_skip & 1);
#else
  const bool use_tma = kVec4;
#endif
  prologue(m, s, use_tma, t0, V);
  pdl_wait();
  STAMP(2);
  const Row r = row_levels<kTable>(m, states + b, s);
  STAMP(3);
  if (t == 0 && t0 == 0) {
    if (r.bad) atomicMin(m.bad_row, (unsigned long long)b);
    if (final_out) final_out[b] = r.bad ? __int_as_float(0x7fc00000) : r.fin;
  }
  float* srow = scores + (size_t)b * m.V + t0;
  int32_t* nrow = next + (size_t)b * m.V + t0;
  if (r.bad) {
    for (int32_t v = t; v < V; v += kThreads) { srow[v] = __int_as_float(0x7fc00000); nrow[v] = -1; }
    if (use_tma) mbar_wait(s.bar, 0);  // no exit with the bulk copy in flight
    return;
  }
  build_row(m, s, r, use_tma, t0, V);

  if (kVec4) {
    // step 4: the finished row leaves by TMA bulk stores (SASS: UBLKCP shared -> global)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy writes -> async proxy
    __syncthreads();
    if (t == 0) {
      const uint32_t bytes = (uint32_t)V * 4u;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(srow),
                   "r"(smem_u32(s.row_s)), "r"(bytes)
                   : "memory");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(nrow),
                   "r"(smem_u32(s.row_n)), "r"(bytes)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      STAMP(7);
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem stays valid until read
    }
  } else {
    for (int32_t v = t; v < V; v += kThreads) {
      __stcs(srow + v, s.row_s[v]);
      __stcs(nrow + v, s.row_n[v]);
    }
  }
  STAMP(8);
  STAMPS_OUT(b);
}

// kRegRoot (V <= 1024): every lane keeps its 32 root weights in registers,
// loaded before the wait, so the root fill is register -> shared stores that
// overlap the arc gathers (shared-memory loads issued after the gathers would
// return behind them); otherwise the CTA bulk-copies the root weights once.
// kIndep (NGPULM_ADVANCE_INDEPENDENT): no running kernel writes this call's
// states or touches its outputs, so the row is built and stored before
// griddepcontrol.wait, which moves to the end (the grid still completes after
// its predecessor: stream completion order is kept) — consecutive calls'
// stores overlap instead of each waiting for the previous call to drain.
template <bool kTable, int kW, bool kPacked, bool kRegRoot, bool kIndep = false>
__global__ void __launch_bounds__(32, NGPULM_ADV_MINB(kW, kPacked))
    advance_warp_kernel(DevModel m, const int32_t* __restrict__ states, int32_t B, float* __restrict__ scores,
                        int32_t* __restrict__ next, float* __restrict__ final_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int32_t V = m.V;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, R = blockDim.x >> 5;
  const size_t rb = kRegRoot ? 0 : align16((size_t)V * 4);  // (kRegRoot: the root weights live in registers)
  const float* root_w = reinterpret_cast<const float*>(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + rb);
  const WSlice s = wcarve(smem + rb + 16 + (size_t)w * wslice_bytes(V, m.order, 0), V, m.order, 0);
  const int32_t row = (int32_t)blockIdx.x * R + w;
  const uint32_t bytes = (uint32_t)V * 4u;
  STAMP(0);
  STAMP(9);
  pdl_trigger();
  // step 0, on immutable model data, so before the wait: the root targets
  // straight into the row's next-state slots (the root has an
  // arc for every token, [0, V)), the root weights into registers (or once
  // per CTA into shared memory).
  if (lane == 0 && row < B) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(s.bar)) : "memory");
    if (w == 0 && !kRegRoot) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(s.bar)), "r"(bytes)
                 : "memory");
    bulk_g2s(s.row_n, m.arc_to, bytes, s.bar);
    if (w == 0 && !kRegRoot) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
      bulk_g2s(const_cast<float*>(root_w), m.arc_w, bytes, bar);
    }
  }
  __syncwarp();  // lane 0's barrier init before the other lanes wait on it
  float4 rw[kRegRoot ? 8 : 1];
  if (kRegRoot && row < B) {
    const float4* w4 = reinterpret_cast<const float4*>(m.arc_w);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (lane + 32 * j < V / 4) rw[j] = __ldg(w4 + lane + 32 * j);
  }
  if (!kRegRoot) __syncthreads();  // the CTA barrier's init visible to every warp
  if (row >= B) return;  // warp 0 always has a row and waits for the CTA's bulk copy
  float* srow = scores + (size_t)row * V;
  int32_t* nrow = next + (size_t)row * V;
  // Steps 1-3 for state st into shared memory (nothing global is written).
  // ph: parity of this build's root-target copy (0: first build, 1: rebuild).
  // The copy's phase is always waited for, so it is over before any re-arm.
  auto build = [&](int32_t st, uint32_t ph) -> Row {
    WLevel lv;
    int32_t nslots;
    const Row r = warp_row_src<kTable>(m, ValState{st}, s, lv, nslots);
    if (r.bad) {
      mbar_wait(s.bar, ph);
      return r;
    }
    STAMP(3);
    Window<kW, kPacked> a;
    if (kRegRoot) {
      load_window<kW, kPacked>(m, s, lv, r.nlev, 0, nslots, a);
      // root scores: acc_root + root weight, while the gathers fly
      float4* s4 = reinterpret_cast<float4*>(s.row_s);
      const float ar = r.acc_root;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (lane + 32 * j < V / 4) {
          float4 y = rw[j];
          y.x = __fadd_rn(ar, y.x);
          y.y = __fadd_rn(ar, y.y);
          y.z = __fadd_rn(ar, y.z);
          y.w = __fadd_rn(ar, y.w);
          s4[lane + 32 * j] = y;
        }
    } else {
      mbar_wait(bar, 0);  // the CTA's root weights have landed (long ago, normally)
      // the root fill goes first: its shared-memory loads would otherwise return
      // behind the arc gathers
      root_fill(s, root_w, r.acc_root, V);
      load_window<kW, kPacked>(m, s, lv, r.nlev, 0, nslots, a);
    }
    STAMP(4);
    mbar_wait(s.bar, ph);  // root targets in row_n
    __syncwarp();
    for (int32_t k0 = 0; k0 < nslots;) {
      write_window<kW, kPacked>(s, a, k0, nslots, m.pk_bits);
      k0 += kW;
      if (k0 < nslots) load_window<kW, kPacked>(m, s, lv, r.nlev, k0, nslots, a);
    }
    return r;
  };
  // Speculative build, store first: the row only needs the
  // model (immutable) and the row's state, so it is built from the state read
  // BEFORE griddepcontrol.wait, overlapping the previous kernel. After the
  // wait (outputs may be written from then on) the finished row leaves at
  // once, and the state is read again while the stores drain: only if the
  // previous kernel changed it is the row rebuilt and stored again, after the
  // first stores have completed (so the rebuilt row is the one that stays).
  // Both state reads are coherent (ld.relaxed.gpu: no stale cache line).
  auto load_state = [&]() {
    int32_t v = 0;
    if (lane == 0) asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(states + row) : "memory");
    return __shfl_sync(kFull, v, 0);
  };
  int32_t st = load_state();
  Row r = build(st, 0);
  if (!r.bad) proxy_fence_warp();  // the row's generic writes -> the bulk stores
  if constexpr (kIndep) {
    if (lane == 0) {
      if (!r.bad) store_row_bulk(s, srow, nrow, bytes);
      if (r.bad) atomicMin(m.bad_row, (unsigned long long)row);
      if (final_out) final_out[row] = r.bad ? __int_as_float(0x7fc00000) : r.fin;
    }
    if (r.bad) {
      for (int32_t v = lane; v < V; v += 32) { srow[v] = __int_as_float(0x7fc00000); nrow[v] = -1; }
    }
    if (!r.bad && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    if (w == 0 && !kRegRoot) mbar_wait(bar, 0);
    // the grid completes only after its predecessor (stream order of completion)
    // as long as one CTA waits for it; the others leave at once, freeing their slot
    if (blockIdx.x == 0) pdl_wait();
    return;
  }
  pdl_wait();
  STAMP(2);
  bool stored = false;
  if (!r.bad && lane == 0) {
    store_row_bulk(s, srow, nrow, bytes);
    STAMP(7);
  }
  stored = !r.bad;
  const int32_t st1 = load_state();
  if (st1 != st) {  // the previous kernel changed the state: rebuild after the wait
    if (stored) {
      // the first stores must be complete (global writes done, shared reads
      // over) before the row is rewritten and stored again
      if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      __syncwarp();
    }
    rearm_root_targets(s, m.arc_to, bytes);
    st = st1;
    r = build(st, 1);
    if (!r.bad) {
      proxy_fence_warp();
      if (lane == 0) store_row_bulk(s, srow, nrow, bytes);
    }
    stored = !r.bad;
  }
  if (lane == 0) {
    if (r.bad) atomicMin(m.bad_row, (unsigned long long)row);
    if (final_out) final_out[row] = r.bad ? __int_as_float(0x7fc00000) : r.fin;
  }
  if (r.bad) {
    for (int32_t v = lane; v < V; v += 32) { srow[v] = __int_as_float(0x7fc00000); nrow[v] = -1; }
  }
  if (stored && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem valid until read
  if (w == 0 && !kRegRoot) mbar_wait(bar, 0);  // no exit with the CTA's bulk copy in flight
  STAMP(8);
  if (w == 0) STAMPS_OUT(row);
}

// ---------------------------------------------------------------- advance, tiny LM resident in shared memory
// Tiny LMs (the paper's 200-keyword biasing LM,
// PAPER.md:295): the whole chain table and the packed arc quads are
// bulk-copied into every CTA's shared memory before griddepcontrol.wait (model
// data is immutable, so the copy overlaps the previous kernel), and a row's
// record and arc quads are then read from shared memory — the two dependent
// L2 round trips after the state load become ~30-cycle shared loads. Row
// construction otherwise as advance_warp_kernel (root level from registers,
// level-ordered writes, bulk stores).
__host__ __device__ constexpr size_t tiny_model_bytes(int64_t chain_bytes, int64_t arcq_bytes, int32_t V) {
  return align16((size_t)chain_bytes) + align16((size_t)arcq_bytes) + align16((size_t)V * 4) + 16;
}

template <int kW>
__global__ void __launch_bounds__(256, 1)
    advance_tiny_kernel(DevModel m, const int32_t* __restrict__ states, int32_t B, float* __restrict__ scores,
                        int32_t* __restrict__ next, float* __restrict__ final_out, int32_t chain_bytes,
                        int32_t arcq_bytes) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int32_t V = m.V;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, R = blockDim.x >> 5;
  const int4* chain_s = reinterpret_cast<const int4*>(smem);
  int4* arcq_s = reinterpret_cast<int4*>(smem + align16(chain_bytes));
  int32_t* root_to = reinterpret_cast<int32_t*>(smem + align16(chain_bytes) + align16(arcq_bytes));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + align16(chain_bytes) + align16(arcq_bytes) + align16(V * 4));
  const size_t mb = tiny_model_bytes(chain_bytes, arcq_bytes, V);
  WSlice s = wcarve(smem + mb + (size_t)w * wslice_bytes(V, m.order, 0), V, m.order, 0);
  s.st_q = arcq_s;  // the quads are read from the CTA's copy (absolute quad index)
  const int32_t row = (int32_t)blockIdx.x * R + w;
  const uint32_t bytes = (uint32_t)V * 4u;
  pdl_trigger();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"((uint32_t)(chain_bytes + arcq_bytes) + bytes)
                 : "memory");
    bulk_g2s(const_cast<int4*>(chain_s), m.chain, (uint32_t)chain_bytes, bar);
    bulk_g2s(arcq_s, m.arc_q, (uint32_t)arcq_bytes, bar);
    bulk_g2s(root_to, m.arc_to, bytes, bar);
  }
  float4 rw[8];
  if (row < B) {
    const float4* w4 = reinterpret_cast<const float4*>(m.arc_w);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (lane + 32 * j < V / 4) rw[j] = __ldg(w4 + lane + 32 * j);
  }
  __syncthreads();  // the barrier's init visible to every warp
  if (row < B) {
    mbar_wait(bar, 0);
    const int4* src = reinterpret_cast<const int4*>(root_to);
    int4* dst = reinterpret_cast<int4*>(s.row_n);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (lane + 32 * j < V / 4) dst[lane + 32 * j] = src[lane + 32 * j];
  }
  if (row >= B) return;  // warp 0 of every CTA has a row (and waited for the CTA's copy)
  float* srow = scores + (size_t)row * V;
  int32_t* nrow = next + (size_t)row * V;
  // the row for state st from the shared copies (speculatively before the wait, as advance_warp_kernel)
  auto build = [&](int32_t st, bool& bad, float& fin) {
    bad = st < 0 || st >= m.S;
    int4 x = make_int4(0, 0, 0, 0);
    if (!bad && lane < m.chain_slots) x = chain_s[(size_t)st * m.chain_slots + lane];
    const int32_t nlev = __shfl_sync(kFull, x.x, 0);
    const float acc_root = __int_as_float(__shfl_sync(kFull, x.y, 0));
    fin = __int_as_float(__shfl_sync(kFull, x.z, 0));
    if (bad) return;
    WLevel lv;
    lv.beg = 0; lv.qbase = 0; lv.info = 0; lv.eslot = INT_MAX; lv.acc = 0.f;
    if (lane >= 1 && lane <= nlev) {
      lv.beg = x.x;
      lv.acc = __int_as_float(x.z);
      lv.info = x.w;
      lv.eslot = (lv.info >> 16) + (((lv.info & 0xffff) + 31) >> 5);
    }
    lv.qbase = lv.beg >> 2;
    const int32_t nslots = nlev > 0 ? __shfl_sync(kFull, lv.eslot, 1) : 0;
    Window<kW, true> a;
    load_window<kW, true, true>(m, s, lv, nlev, 0, nslots, a);
    {  // root scores: acc_root + root weight
      float4* s4 = reinterpret_cast<float4*>(s.row_s);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (lane + 32 * j < V / 4) {
          float4 y = rw[j];
          y.x = __fadd_rn(acc_root, y.x);
          y.y = __fadd_rn(acc_root, y.y);
          y.z = __fadd_rn(acc_root, y.z);
          y.w = __fadd_rn(acc_root, y.w);
          s4[lane + 32 * j] = y;
        }
    }
    __syncwarp();
    for (int32_t k0 = 0; k0 < nslots;) {
      write_window<kW, true>(s, a, k0, nslots, m.pk_bits);
      k0 += kW;
      if (k0 < nslots) load_window<kW, true, true>(m, s, lv, nlev, k0, nslots, a);
    }
  };
  auto load_state = [&]() {
    int32_t v = 0;
    if (lane == 0) asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(states + row) : "memory");
    return __shfl_sync(kFull, v, 0);
  };
  // speculative build and store-first, as advance_warp_kernel
  bool bad = false;
  float fin = 0.f;
  int32_t st = load_state();
  build(st, bad, fin);
  if (!bad) proxy_fence_warp();
  pdl_wait();
  if (!bad && lane == 0) store_row_bulk(s, srow, nrow, bytes);
  bool stored = !bad;
  const int32_t st1 = load_state();
  if (st1 != st) {
    if (stored) {
      if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      __syncwarp();
    }
    // the root targets again (the first build overwrote them), generic copies
    const int4* src = reinterpret_cast<const int4*>(root_to);
    int4* dst = reinterpret_cast<int4*>(s.row_n);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (lane + 32 * j < V / 4) dst[lane + 32 * j] = src[lane + 32 * j];
    __syncwarp();
    st = st1;
    build(st, bad, fin);
    if (!bad) {
      proxy_fence_warp();
      if (lane == 0) store_row_bulk(s, srow, nrow, bytes);
    }
    stored = !bad;
  }
  if (lane == 0) {
    if (bad) atomicMin(m.bad_row, (unsigned long long)row);
    if (final_out) final_out[row] = bad ? __int_as_float(0x7fc00000) : fin;
  }
  if (bad) {
    for (int32_t v = lane; v < V; v += 32) { srow[v] = __int_as_float(0x7fc00000); nrow[v] = -1; }
  }
  if (stored && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// ---------------------------------------------------------------- final
__global__ void final_kernel(DevModel m, const int32_t* __restrict__ states, int32_t B,
                             float* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
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

}  // namespace

// The largest row (multiple of 4 tokens) the CTA kernels hold in shared memory.
int max_row_in_smem(int32_t order) {
  int v = 32768;
  while (v > 0 && row_smem(v, order) > 227 * 1024) v -= 4;
  return v;
}
// advance / final: any V (rows are tiled); fused step, top-k, decode: one row in shared memory.
int max_vocab_supported() { return 1 << 24; }
int max_fused_vocab() { return max_row_in_smem(NGPULM_MAX_ORDER); }
// Tile of the CTA advance kernel: the whole row if it fits, else the largest
// multiple of 4 that fits (unaligned V: the scalar path, any tile).
int32_t vocab_tile(int32_t V, int32_t order) {
  const int32_t cap = max_row_in_smem(order);
  return V <= cap ? V : cap;
}

int launch_advance(const DevModel& m, const int32_t* states, int32_t B, float* scores, int32_t* next,
                   float* final_out, void* stream, uint32_t flags) {
  const bool indep = flags & NGPULM_ADVANCE_INDEPENDENT;  // (a permission: paths without it ignore it)
  const bool vec = (m.V % 4 == 0) && ((uintptr_t)scores % 16 == 0) && ((uintptr_t)next % 16 == 0);
  const bool table = m.chain != nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  if (vec && table && m.tiny_chain_bytes > 0 && m.adv_kind == NGPULM_ADVANCE_AUTO && B <= NGPULM_TINY_MAX_B) {
    // tiny LM: model resident in every CTA's shared memory
    const size_t mb = tiny_model_bytes(m.tiny_chain_bytes, m.tiny_arcq_bytes, m.V);
    int R = (B + 147) / 148;
    R = R < 1 ? 1 : (R > NGPULM_TINY_ROWS ? NGPULM_TINY_ROWS : R);
    while (R > 1 && mb + (size_t)R * wslice_bytes(m.V, m.order, 0) > 227 * 1024) --R;
    const size_t tsm = mb + (size_t)R * wslice_bytes(m.V, m.order, 0);
    if (tsm <= 227 * 1024) {
      const dim3 tg((B + R - 1) / R), tb(32 * R);
      if (B > 8 * 148)
        return launch(advance_tiny_kernel<8>, tg, tb, tsm, st, m, states, B, scores, next, final_out,
                      m.tiny_chain_bytes, m.tiny_arcq_bytes);
      return launch(advance_tiny_kernel<16>, tg, tb, tsm, st, m, states, B, scores, next, final_out,
                    m.tiny_chain_bytes, m.tiny_arcq_bytes);
    }
  }
  if (vec && m.adv_kind != NGPULM_ADVANCE_CTA) {
    // up to 8 rows per SM: 16-slot windows (almost every row in one window);
    // more rows per SM: 8-slot windows (registers for occupancy)
    const bool wide = B <= NGPULM_WIDE_MAX_B, pk = m.arc_q != nullptr && m.adv_kind == NGPULM_ADVANCE_AUTO;
    const bool small_v = m.V <= 1024;
    // one row (warp) per CTA: a CTA leaves as soon as its row is stored and the
    // next call's CTA starts its speculative build in its place (B=1024: 7 rows
    // per CTA 3.29 us, 1 row 2.83 us; B=4096: 10.1 -> 9.4 us)
    const int R = NGPULM_ADV_ROWS;
    if (wcta_smem(m.V, m.order, R, 0) <= 227 * 1024) {
      // (V <= 1024: root weights in registers, no shared copy)
      const size_t wsm = wcta_smem(m.V, m.order, R, 0) - (small_v ? align16((size_t)m.V * 4) : 0);
      // the grid is padded to a multiple of the SM count (the extra CTAs exit at
      // once), so every SM holds the same number of rows of a call and
      // consecutive calls' CTAs line up on the same SMs: measured B=128 1.92 ->
      // 1.69 us, B=147 1.93 -> 1.34 (one CTA per SM)
      int32_t nrows = B;
      if (B >= NGPULM_PAD_MIN_B) {
#if NGPULM_PAD_MODE == 0
        if (B < NGPULM_PAD_GRID) nrows = NGPULM_PAD_GRID;
#elif NGPULM_PAD_MODE == 1
        nrows = (B + NGPULM_PAD_GRID - 1) / NGPULM_PAD_GRID * NGPULM_PAD_GRID;
#else
        const int32_t per = (B + NGPULM_PAD_GRID - 1) / NGPULM_PAD_GRID;  // rows per SM, rounded to a power of 2
        int32_t p2 = 1;
        while (p2 < per) p2 *= 2;
        nrows = p2 * NGPULM_PAD_GRID;
#endif
      }
      const dim3 wg((nrows + R - 1) / R), wb(32 * R);
#define NGPULM_WARP_LAUNCH(T, W, P)                                                                                 \
  return small_v ? launch(advance_warp_kernel<T, W, P, true>, wg, wb, wsm, st, m, states, B, scores, next, final_out) \
                 : launch(advance_warp_kernel<T, W, P, false>, wg, wb, wsm, st, m, states, B, scores, next, final_out)
      if (indep && table && small_v) {
        if (pk)
          return wide ? launch(advance_warp_kernel<true, 16, true, true, true>, wg, wb, wsm, st, m, states, B,
                               scores, next, final_out)
                      : launch(advance_warp_kernel<true, 8, true, true, true>, wg, wb, wsm, st, m, states, B,
                               scores, next, final_out);
        return wide ? launch(advance_warp_kernel<true, 16, false, true, true>, wg, wb, wsm, st, m, states, B, scores,
                             next, final_out)
                    : launch(advance_warp_kernel<true, 8, false, true, true>, wg, wb, wsm, st, m, states, B, scores,
                             next, final_out);
      }
      if (table) {
        if (wide) { if (pk) NGPULM_WARP_LAUNCH(true, 16, true); NGPULM_WARP_LAUNCH(true, 16, false); }
        if (pk) NGPULM_WARP_LAUNCH(true, 8, true);
        NGPULM_WARP_LAUNCH(true, 8, false);
      }
      if (wide) { if (pk) NGPULM_WARP_LAUNCH(false, 16, true); NGPULM_WARP_LAUNCH(false, 16, false); }
      if (pk) NGPULM_WARP_LAUNCH(false, 8, true);
      NGPULM_WARP_LAUNCH(false, 8, false);
#undef NGPULM_WARP_LAUNCH
    }
  }
  const int32_t tile = vocab_tile(m.V, m.order);
  const size_t sm = row_smem(tile, m.order);
  const dim3 gd(B, (m.V + tile - 1) / tile), bd(kThreads);
  if (vec && table)
    return launch(advance_kernel<true, true>, gd, bd, sm, st, m, states, scores, next, final_out, tile);
  if (vec) return launch(advance_kernel<true, false>, gd, bd, sm, st, m, states, scores, next, final_out, tile);
  if (table) return launch(advance_kernel<false, true>, gd, bd, sm, st, m, states, scores, next, final_out, tile);
  return launch(advance_kernel<false, false>, gd, bd, sm, st, m, states, scores, next, final_out, tile);
}

int launch_final(const DevModel& m, const int32_t* states, int32_t B, float* out, void* stream) {
  return launch(final_kernel, dim3((B + 255) / 256), dim3(256), 0, (cudaStream_t)stream, m, states, B, out);
}

}  // namespace ngpulm
