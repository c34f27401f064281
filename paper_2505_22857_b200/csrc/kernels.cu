// NGPU-LM hot path for sm_100a: batched full-vocabulary query (Algorithm 1,
// PAPER.md:54-89) and the fused greedy shallow-fusion step.
//
// Design: one CTA of 256 threads per batch row; the row
// lives in shared memory as (score, next state) per token, 8 KB at V = 1024,
// so 8 CTAs fit per SM and B = 1024 rows run as one wave. Bulk data moves by
// TMA (cp.async.bulk), so the SM's load/store queue only carries the
// latency-critical gathers (state, chain record, arcs), which complete in
// issue order behind whatever else that queue holds.
//  0. prologue, independent of earlier kernels (model data is immutable): one
//     thread bulk-copies the root level (an arc for every token,
//     [0, V)) into the row: weights into the score slots, targets into the
//     next-state slots. Then griddepcontrol.wait (programmatic dependent
//     launch), so launch and prologue overlap the previous kernel.
//  1. warp 0 reads the row's state and its back-off levels (Algorithm 1 lines
//     72, 81-82) — from the load-time chain table (one 16-byte record slot per
//     level and lane, acc_boff pre-accumulated left to right in float, R10)
//     or, in walk mode, lane 0 walks boff_to_states level by level exactly as
//     Algorithm 1 does. One barrier publishes them.
//  2. every thread gathers up to 4 arcs of the row into registers, all loads
//     in flight together (a level's arcs are contiguous: arcs are sorted by
//     (from_state, token)), while the root slots get acc_root
//     added (root score = acc_root + root weight).
//  3. the gathered arcs are written into the row level by level from the
//     lowest order up, one barrier per level, so a higher-order arc
//     overwrites a lower-order one — Algorithm 1's "first level found wins"
//     (lines 77-79) with plain shared-memory stores, no atomics.
//  4. advance: the finished row leaves by two TMA bulk stores (scores, next);
//     fused step: the columns' fused values feed a shuffle argmax, so the LM
//     row never touches HBM.
// Rows with more than 1024 non-root arcs repeat steps 2-3 per 1024-arc chunk.
// No tensor cores: gather/scatter + store bandwidth only.
#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <cstdint>
#include <type_traits>

#include "ngpulm_internal.h"

namespace ngpulm {
namespace {

#ifndef NGPULM_THREADS
#define NGPULM_THREADS 256
#endif
#ifndef NGPULM_UNROLL
#define NGPULM_UNROLL 4
#endif
constexpr int kThreads = NGPULM_THREADS;   // threads per row (CTA)
constexpr int kMinBlocks = 2048 / kThreads;  // CTAs per SM: 64 warps, 32 registers per thread
constexpr int kWarps = kThreads / 32;
constexpr int kUnroll = NGPULM_UNROLL;     // arcs gathered per thread per chunk
constexpr int kChunk = kThreads * kUnroll;
constexpr uint32_t kFull = 0xffffffffu;

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) / 16 * 16; }
__host__ __device__ constexpr int32_t level_cap(int32_t order) { return order > 1 ? order : 1; }
__host__ __device__ constexpr size_t levels_bytes(int32_t order) {  // beg[Lc] pre[Lc+1] acc[Lc]
  return align16(((size_t)3 * level_cap(order) + 1) * 4);
}
// row_s[V] | row_n[V] | st_tok/st_s/st_n[kChunk] | scratch, barrier, row scalars | levels
__host__ __device__ constexpr size_t row_smem(int32_t V, int32_t order) {
  return 2 * align16((size_t)V * 4) + (size_t)kChunk * 12 + 128 + levels_bytes(order);
}

struct Row {  // per-row scalars
  int32_t state, nlev, total, bad;
  float acc_root, fin;
};

struct Slice {     // the row in shared memory
  float* row_s;    // [V] score per token (root weight until step 2)
  int32_t* row_n;  // [V] next state per token
  float* red_v;    // argmax scratch [kWarps]
  int32_t* red_c;
  uint64_t* bar;   // mbarrier of the root bulk copy
  Row* row;        // row scalars (written by warp 0)
  int32_t* st_tok; // [kChunk] staged arcs of the current round: token
  float* st_s;     //          acc_boff + arc weight
  int32_t* st_n;   //          target
  int32_t* beg;    // levels: [Lc] first arc of level i
  int32_t* pre;    // [Lc+1] prefix count of arcs (pre[nlev] = total)
  float* acc;      // [Lc] acc_boff when level i is visited
};

__device__ __forceinline__ Slice carve(unsigned char* p, int32_t V, int32_t order) {
  const int32_t Lc = level_cap(order);
  Slice s;
  s.row_s = reinterpret_cast<float*>(p);
  p += align16((size_t)V * 4);
  s.row_n = reinterpret_cast<int32_t*>(p);
  p += align16((size_t)V * 4);
  s.st_tok = reinterpret_cast<int32_t*>(p);
  s.st_s = reinterpret_cast<float*>(p + kChunk * 4);
  s.st_n = reinterpret_cast<int32_t*>(p + kChunk * 8);
  p += (size_t)kChunk * 12;
  s.red_v = reinterpret_cast<float*>(p);
  s.red_c = reinterpret_cast<int32_t*>(p + 32);
  s.bar = reinterpret_cast<uint64_t*>(p + 64);
  s.row = reinterpret_cast<Row*>(p + 72);
  p += 128;
  int32_t* l = reinterpret_cast<int32_t*>(p);
  s.beg = l;
  s.pre = l + Lc;
  s.acc = reinterpret_cast<float*>(l + 2 * Lc + 1);
  return s;
}

#ifdef NGPULM_PHASE_TIMING
// Debug build only (tools/phase_timing.py): per-row stamps of thread 0, kept
// in shared memory during the row (so the stamps add no global traffic) and
// written out at the end: 0 entry (globaltimer ns), 1 entry, 2 after
// griddepcontrol.wait, 3 levels published, 4 arcs staged, 5 root fix-up
// barrier, 6 levels written, 7 stores issued (clock64), 8 end (ns), 9 SM id.
__device__ unsigned long long g_phase[16384 * 16];
__device__ int g_skip;  // bit 0: no TMA prologue (CTA kernel); warp kernel: bit 1 no stores, bit 2 no arcs, bit 3 no fill
__device__ __forceinline__ unsigned long long* stamp_buf() {
  __shared__ unsigned long long buf[16];
  return buf;
}
#define STAMP(i)                                                                        \
  do {                                                                                  \
    if (threadIdx.x == 0) {                                                             \
      unsigned long long t;                                                             \
      if ((i) == 0 || (i) == 8) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));   \
      else if ((i) == 9) asm volatile("mov.u32 %0, %%smid;" : "=r"(*(unsigned*)&t));   \
      else t = clock64();                                                               \
      stamp_buf()[i] = t;                                                               \
    }                                                                                   \
  } while (0)
#define STAMPS_OUT(row)                                                                 \
  do {                                                                                  \
    if (threadIdx.x == 0 && (row) < 16384)                                              \
      for (int _i = 0; _i < 16; ++_i) g_phase[(row) * 16 + _i] = stamp_buf()[_i];       \
  } while (0)
#else
#define STAMP(i) \
  do {           \
  } while (0)
#define STAMPS_OUT(row) \
  do {                  \
  } while (0)
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t b = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(b), "r"(phase)
        : "memory");
  } while (!done);
}

// Step 0 (one thread of warp 1, so warp 0's state load is not queued behind
// it): root level -> row slots by TMA bulk copy (SASS: UBLKCP). The barrier
// init is made visible to the async proxy with a CTA-scope proxy fence.
constexpr int kTmaThread = 32;
// lo / tv: the vocabulary tile [lo, lo + tv) this CTA answers (the whole row
// when the row fits in shared memory).
__device__ __forceinline__ void prologue(const DevModel& m, const Slice& s, bool tma, int32_t lo = 0,
                                         int32_t tv = -1) {
  if (threadIdx.x != kTmaThread) return;
  const uint32_t b = smem_u32(s.bar), bytes = (uint32_t)(tv < 0 ? m.V : tv) * 4u;
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (!tma) return;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(2u * bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(s.row_s)),
               "l"(m.arc_w + lo), "r"(bytes), "r"(b)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(s.row_n)),
               "l"(m.arc_to + lo), "r"(bytes), "r"(b)
               : "memory");
}

// Where a row's state comes from: a device array (advance, fused step) or a
// register (the persistent decode, which holds the state across frames).
struct PtrState {
  const int32_t* p;
  __device__ __forceinline__ int32_t operator()() const { return __ldg(p); }
};
struct ValState {
  int32_t v;
  __device__ __forceinline__ int32_t operator()() const { return v; }
};

// Step 1, warp 0: the row's levels into shared memory + the Row scalars.
template <bool kTable, typename SF = PtrState>
__device__ __forceinline__ Row load_levels(const DevModel& m, SF state_src, int32_t* beg, int32_t* pre_,
                                           float* accs) {
  const int lane = threadIdx.x & 31;
  Row r;
  // Kernel parameters sit in the constant bank; a constant-cache miss costs an
  // L2 round trip. Read the ones this step needs into registers now, before
  // the state arrives (volatile asm pins them here), so their misses overlap
  // the state load instead of following it.
  const int4* table = reinterpret_cast<const int4*>(m.chain) + lane;
  int32_t slots = m.chain_slots, S = m.S;
  asm volatile("" : "+l"(table), "+r"(slots), "+r"(S));
  const int32_t st = __shfl_sync(kFull, lane == 0 ? state_src() : 0, 0);
  STAMP(10);
  r.state = st;
  r.bad = st < 0 || st >= S;
  r.nlev = 0; r.total = 0; r.acc_root = 0.f; r.fin = 0.f;
  if (r.bad) return r;
  if (kTable) {
    // record = [header {nlev, acc_root, final, total}] + nlev x {begin, prefix, acc, 0}
    int4 x = make_int4(0, 0, 0, 0);
    if (lane < slots) x = __ldg(table + (size_t)st * slots);
    r.nlev = __shfl_sync(kFull, x.x, 0);
    r.acc_root = __int_as_float(__shfl_sync(kFull, x.y, 0));
    r.fin = __int_as_float(__shfl_sync(kFull, x.z, 0));
    r.total = __shfl_sync(kFull, x.w, 0);
    if (lane >= 1 && lane <= r.nlev) { beg[lane - 1] = x.x; pre_[lane - 1] = x.y; accs[lane - 1] = __int_as_float(x.z); }
    if (lane == 0) pre_[r.nlev] = r.total;
  } else {
    // Algorithm 1 lines 67-82, serial by nature (pointer chase), lane 0
    int32_t n = 0, pre = 0, bad = 0;
    float acc = 0.f, fin = 0.f;
    if (lane == 0) {
      const int4* rec = reinterpret_cast<const int4*>(m.srec);
      int32_t x = st;
      for (; n < level_cap(m.order) && x != 0; ++n) {
        const int4 q = __ldg(rec + x);  // {arc_begin, arc_end, boff_to, boff_w}
        beg[n] = q.x;
        pre_[n] = pre;
        accs[n] = acc;
        pre += q.y - q.x;
        acc = __fadd_rn(acc, __int_as_float(q.w));  // acc_boff += boff_weights[state]
        x = q.z;                                     // state = boff_to_states[state]
      }
      pre_[n] = pre;
      bad = x != 0;
      fin = bad ? 0.f : __ldg(&m.final_w[st]);
    }
    r.nlev = __shfl_sync(kFull, n, 0);
    r.total = __shfl_sync(kFull, pre, 0);
    r.acc_root = __shfl_sync(kFull, acc, 0);
    r.fin = __shfl_sync(kFull, fin, 0);
    r.bad = __shfl_sync(kFull, bad, 0);
  }
  return r;
}

// Warp 0 loads, everyone reads the result after one barrier.
template <bool kTable>
__device__ __forceinline__ Row row_levels(const DevModel& m, const int32_t* state_ptr, const Slice& s) {
  if (threadIdx.x < 32) {
    const Row rr = load_levels<kTable>(m, PtrState{state_ptr}, s.beg, s.pre, s.acc);
    STAMP(11);
    if (threadIdx.x == 0) *s.row = rr;
  }
  __syncthreads();
  return *s.row;
}

__device__ __forceinline__ int level_of(const Slice& s, int32_t j) {
  int L = 0;
  while (j >= s.pre[L + 1]) ++L;
  return L;
}

// Step 2 for one round of arcs [lo, hi) (hi - lo <= kChunk): every thread
// loads its (up to kUnroll) arcs — all loads in flight together — and stages
// them in shared memory at slot j - lo as (token, acc_boff + weight, target).
__device__ __forceinline__ void stage_arcs(const DevModel& m, const Slice& s, int32_t lo, int32_t hi) {
  int32_t tk[kUnroll], to[kUnroll], Ls[kUnroll];
  float w[kUnroll];
  int L = 0;
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    const int32_t j = lo + u * kThreads + (int32_t)threadIdx.x;
    Ls[u] = -1;
    if (j < hi) {
      while (j >= s.pre[L + 1]) ++L;
      const int32_t arc = s.beg[L] + (j - s.pre[L]);
      Ls[u] = L;
      tk[u] = __ldg(&m.arc_tok[arc]);
      w[u] = __ldg(&m.arc_w[arc]);
      to[u] = __ldg(&m.arc_to[arc]);
    }
  }
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    if (Ls[u] < 0) continue;
    const int32_t slot = u * kThreads + (int32_t)threadIdx.x;
    s.st_tok[slot] = tk[u];
    s.st_s[slot] = __fadd_rn(s.acc[Ls[u]], w[u]);  // acc_boff + arc_weights (Alg. 1 line 74)
    s.st_n[slot] = to[u];
  }
}

// Step 3 for one round: levels from the highest index (lowest order) down,
// one barrier each, threads strided over the level's staged slots.
// (tile: tokens [t0, t0 + tv) of the row; others are skipped)
__device__ __forceinline__ void write_levels(const Slice& s, int32_t lo, int32_t hi, int Llo, int Lhi, int32_t t0,
                                             uint32_t tv) {
  for (int L = Lhi; L >= Llo; --L) {
    const int32_t j1 = min(hi, s.pre[L + 1]) - lo;
    for (int32_t j = max(lo, s.pre[L]) - lo + (int32_t)threadIdx.x; j < j1; j += kThreads) {
      const uint32_t i = (uint32_t)(s.st_tok[j] - t0);
      if (i < tv) {
        s.row_s[i] = s.st_s[j];
        s.row_n[i] = s.st_n[j];
      }
    }
    __syncthreads();
  }
}

// Steps 2-3: root slots get acc_root; non-root arcs overwrite, lowest order
// first. Rounds of kChunk arcs run from the last (lowest-order) arcs to the
// first; the first round's loads are issued before the root fix-up so their
// latencies overlap.
__device__ __forceinline__ void build_row(const DevModel& m, const Slice& s, const Row& r, bool tma, int32_t t0 = 0,
                                          int32_t tv = -1) {
  const int32_t V = tv < 0 ? m.V : tv, T = r.total;
  const float acc_root = r.acc_root;
  int32_t lo = T > kChunk ? T - kChunk : 0;
  if (T > 0) stage_arcs(m, s, lo, T);
  STAMP(4);
  if (tma) mbar_wait(s.bar, 0);
  if ((V & 3) == 0 && tma) {
    float4* s4 = reinterpret_cast<float4*>(s.row_s);
    for (int32_t q = threadIdx.x; q < V / 4; q += kThreads) {
      float4 x = s4[q];
      x.x = __fadd_rn(acc_root, x.x);  // root level: acc_root + root weight
      x.y = __fadd_rn(acc_root, x.y);
      x.z = __fadd_rn(acc_root, x.z);
      x.w = __fadd_rn(acc_root, x.w);
      s4[q] = x;
    }
  } else {
    for (int32_t v = threadIdx.x; v < V; v += kThreads) {
      s.row_s[v] = __fadd_rn(acc_root, __ldg(&m.arc_w[t0 + v]));
      s.row_n[v] = __ldg(&m.arc_to[t0 + v]);
    }
  }
  __syncthreads();
  STAMP(5);
  for (int32_t hi = T; hi > 0;) {
    const int Llo = lo == 0 ? 0 : level_of(s, lo), Lhi = hi == T ? r.nlev - 1 : level_of(s, hi - 1);
    write_levels(s, lo, hi, Llo, Lhi, t0, (uint32_t)V);
    hi = lo;
    if (hi == 0) break;
    lo = hi > kChunk ? hi - kChunk : 0;
    stage_arcs(m, s, lo, hi);
    __syncthreads();
  }
  STAMP(6);
}

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

// ---------------------------------------------------------------- advance, one warp per row
// A CTA of R warps answers R rows, one per warp; the CTA shares one copy of
// the root level (bulk-copied once per CTA, before griddepcontrol.wait).
// Lane l+1 of a warp holds level l of its row (the chain-table record is
// already laid out that way). Every level is cut into "slots" of 32 16-byte
// quads (lane i of a slot loads quad i: up to four consecutive arcs of that
// level; every model array is padded in the blob, so a quad never leaves it).
// Slots are numbered from the last level (lowest order) to the first, so
// writing them in slot order, with a __syncwarp where the level changes, lets
// the highest order found win — Algorithm 1 lines 77-79 — with plain
// shared-memory stores. kSlots slots are in flight at once (all their loads
// issued together); rows with more slots take more windows. Masked-off arc
// lanes store into a trash word behind the row, so the write loop has no
// branches. No CTA-wide barrier after the prologue: rows never wait for each
// other.
#ifndef NGPULM_STORE_HINT
#define NGPULM_STORE_HINT 1
#endif
#ifndef NGPULM_PAIR_MAX_B
#define NGPULM_PAIR_MAX_B (4 * 148)  // transducer steps: two warps per row up to 4 rows per SM (measured:
                                     // RNN-T B=512 4.36 -> 4.00 us; CTC/AED lose, they keep one warp)
#endif
#ifndef NGPULM_SPECULATE
#define NGPULM_SPECULATE 1
#endif
// launch bounds of the warp advance kernel: with one row per CTA (32
// threads), the minimum CTAs per SM sets the register budget
// (one warp per CTA; 8-slot windows and the staged path: 16 CTAs per SM =
// 128 registers, measured B=4096 9.46 -> 8.16 us, B=128 1.90 -> 1.66 us;
// the 16-slot path keeps its 245 registers: capped it spills, B=1024 2.82 -> 4.29)
#define NGPULM_ADV_MINB(kW, kPacked, kStage) ((kStage) ? 16 : (kW) == 8 ? ((kPacked) ? 16 : 10) : 8)
#ifndef NGPULM_TINY_MAX_B
#define NGPULM_TINY_MAX_B 148  // tiny LM in shared memory up to one row per SM (B=128: 1.34 vs 1.66 us);
#endif                         // beyond, the one-row-per-CTA global kernel wins (B=1024: 2.53 vs 3.08)
#ifndef NGPULM_TINY_ROWS
#define NGPULM_TINY_ROWS 8
#endif
#ifndef NGPULM_FUSED_MAX_ROWS
#define NGPULM_FUSED_MAX_ROWS 8
#endif
#ifndef NGPULM_CTA_ROOT
#define NGPULM_CTA_ROOT 0  // (with 7 rows per CTA: 3.74 -> 3.64 us at B = 1024; with one row per CTA: 2.83 vs 3.00)
#endif
#ifndef NGPULM_WIDE_MAX_B
#define NGPULM_WIDE_MAX_B (8 * 148)  // up to 8 rows per SM: 16-slot windows (measured)
#endif

__host__ __device__ constexpr size_t wrow_bytes(int32_t V) { return align16((size_t)V * 4 + 4); }  // + trash word
// staged arcs: kStageQuads packed arc quads (32 bytes each)
constexpr int kStageQuads = 512;
#ifndef NGPULM_STAGE_MAX_B
#define NGPULM_STAGE_MAX_B 148  // batches of 2 .. one row per SM stage their arcs by bulk copy (measured)
#endif
__host__ __device__ constexpr size_t wslice_bytes(int32_t V, int32_t order, int stage_q) {
  return 2 * wrow_bytes(V) + levels_bytes(order) + 16 + (size_t)stage_q * 32;
}
// root_w[V] | mbarrier | R x (row_s[V+1] | row_n[V+1] | levels | 2 mbarriers | staged arcs)
__host__ __device__ constexpr size_t wcta_smem(int32_t V, int32_t order, int R, int stage_q) {
  return align16((size_t)V * 4) + 16 + (size_t)R * wslice_bytes(V, order, stage_q);
}

struct WSlice {
  float* row_s;  // [V] + trash
  int32_t* row_n;
  int32_t* beg;  // levels (walk mode: written by lane 0)
  int32_t* pre;
  float* acc;
  uint64_t* bar;   // the root targets' bulk copy into row_n
  uint64_t* abar;  // the arcs' bulk copies into the staging area
  int4* st_q;      // [stage_q][2] staged packed arc quads
};

__device__ __forceinline__ WSlice wcarve(unsigned char* p, int32_t V, int32_t order, int stage_q) {
  const int32_t Lc = level_cap(order);
  WSlice s;
  s.row_s = reinterpret_cast<float*>(p);
  p += wrow_bytes(V);
  s.row_n = reinterpret_cast<int32_t*>(p);
  p += wrow_bytes(V);
  int32_t* l = reinterpret_cast<int32_t*>(p);
  s.beg = l;
  s.pre = l + Lc;
  s.acc = reinterpret_cast<float*>(l + 2 * Lc + 1);
  s.bar = reinterpret_cast<uint64_t*>(p + levels_bytes(order));
  s.abar = s.bar + 1;
  s.st_q = reinterpret_cast<int4*>(p + levels_bytes(order) + 16);
  return s;
}

struct WLevel {  // lane l+1: level l of the row
  int32_t beg;       // first arc (16-byte aligned in the device layout)
  int32_t qbase;     // first quad of the level where the gathers read it (global arrays or staging)
  int32_t info;      // (first slot << 16) | quads
  int32_t eslot;     // one past the level's last slot (INT_MAX on lanes without a level)
  float acc;         // acc_boff at the level
};

// The row's state, header and levels (Algorithm 1 lines 67-82).
struct NoOp {
  __device__ void operator()() const {}
};

// after_issue() runs once the chain-record load is in flight (table mode) or
// before the walk: independent loads issued there overlap its latency.
template <bool kTable, typename F = NoOp, typename SF = PtrState>
__device__ __forceinline__ Row warp_row_src(const DevModel& m, SF state_src, const WSlice& s, WLevel& lv,
                                            int32_t& nslots, F after_issue = F()) {
  const int lane = threadIdx.x & 31;
  Row r;
  lv.beg = 0; lv.qbase = 0; lv.info = 0; lv.eslot = INT_MAX; lv.acc = 0.f;
  nslots = 0;
  if (kTable) {
    const int4* table = reinterpret_cast<const int4*>(m.chain) + lane;
    int32_t slots = m.chain_slots, S = m.S;
    asm volatile("" : "+l"(table), "+r"(slots), "+r"(S));  // parameters read before the state arrives
    const int32_t st = __shfl_sync(kFull, lane == 0 ? state_src() : 0, 0);
    STAMP(10);
    r.state = st;
    r.bad = st < 0 || st >= S;
    r.nlev = 0; r.total = 0; r.acc_root = 0.f; r.fin = 0.f;
    if (r.bad) return r;
    int4 x = make_int4(0, 0, 0, 0);
    if (lane < slots) x = __ldg(table + (size_t)st * slots);
    after_issue();
    r.nlev = __shfl_sync(kFull, x.x, 0);
    r.acc_root = __int_as_float(__shfl_sync(kFull, x.y, 0));
    r.fin = __int_as_float(__shfl_sync(kFull, x.z, 0));
    r.total = __shfl_sync(kFull, x.w, 0);
    if (lane >= 1 && lane <= r.nlev) {
      lv.beg = x.x;
      lv.acc = __int_as_float(x.z);
      lv.info = x.w;
    }
  } else {
    after_issue();
    r = load_levels<false>(m, state_src, s.beg, s.pre, s.acc);
    if (r.bad) return r;
    __syncwarp();
    int32_t nq = 0;
    if (lane >= 1 && lane <= r.nlev) {
      lv.beg = s.beg[lane - 1];
      lv.acc = s.acc[lane - 1];
      nq = (s.pre[lane] - s.pre[lane - 1] + 3) >> 2;
    }
    int32_t inc = (nq + 31) >> 5;  // slots of levels >= this one, then exclusive
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_down_sync(kFull, inc, o);
      if (lane + o < 32) inc += y;
    }
    lv.info = ((inc - ((nq + 31) >> 5)) << 16) | nq;
  }
  if (lane >= 1 && lane <= r.nlev) lv.eslot = (lv.info >> 16) + (((lv.info & 0xffff) + 31) >> 5);
  lv.qbase = lv.beg >> 2;
  nslots = r.nlev > 0 ? __shfl_sync(kFull, lv.eslot, 1) : 0;
  return r;
}

template <bool kTable, typename F = NoOp>
__device__ __forceinline__ Row warp_row(const DevModel& m, const int32_t* state_ptr, const WSlice& s, WLevel& lv,
                                        int32_t& nslots, F after_issue = F()) {
  return warp_row_src<kTable>(m, PtrState{state_ptr}, s, lv, nslots, after_issue);
}

// One window of kW slots, in registers, processed in groups of 8 slots; a
// group wholly past the row's last slot is skipped (uniform branch). Arcs are
// either packed ((target << pk_bits) | token next to the weight: two 16-byte
// loads per quad) or three arrays (three loads per quad).
template <int kW, bool kPacked>
struct Window {
  float4 w[kW];
  int4 tok[kW];  // packed: (target << pk_bits) | token
  int4 to[kPacked ? 1 : kW];
  float acc[kW];  // acc_boff of the slot's level
};

// Within a group everything is branch-free, so the group's shuffles and loads
// are scheduled together. A level starts on a quad boundary and the rest of
// its last quad repeats its last arc, so whole quads are written; an idle lane
// (past its level's quads) loads the level's first quad again, and a slot
// past the row's last one repeats the last slot (of the highest order, which
// is written last anyway): rewriting an arc of the same level stores the
// value already there.
// kSmem: the quads come from the row's staging area (bulk-copied there),
// else from the global arrays.
template <int kW, bool kPacked, bool kSmem = false>
__device__ __forceinline__ void load_window(const DevModel& m, const WSlice& s, const WLevel& lv, int32_t nlev,
                                            int32_t k0, int32_t nslots, Window<kW, kPacked>& a) {
  const int lane = threadIdx.x & 31;
  const int4* tok4 = reinterpret_cast<const int4*>(m.arc_tok);
  const float4* w4 = reinterpret_cast<const float4*>(m.arc_w);
  const int4* to4 = reinterpret_cast<const int4*>(m.arc_to);
#pragma unroll
  for (int g = 0; g < kW; g += 8) {
    if (g > 0 && k0 + g >= nslots) break;
    int32_t qv[8];
#pragma unroll
    for (int u = g; u < g + 8; ++u) {
      const int32_t k = min(k0 + u, nslots - 1);  // a slot past the last one repeats the last one
      // levels entirely before slot k (in slot order) are the levels after its own
      const int32_t L = nlev - 1 - __popc(__ballot_sync(kFull, lv.eslot <= k));
      const int src = L + 1;
      const int32_t info = __shfl_sync(kFull, lv.info, src), qb = __shfl_sync(kFull, lv.qbase, src);
      a.acc[u] = __shfl_sync(kFull, lv.acc, src);
      const int32_t i = (k - (info >> 16)) * 32 + lane;
      qv[u - g] = qb + (i < (info & 0xffff) ? i : 0);
    }
#pragma unroll
    for (int u = g; u < g + 8; ++u) {
      if (u > g && k0 + u >= nslots) break;  // (uniform) no load for slots past the row's last one
      if (kSmem) {  // two 16-byte shared loads of the staged quad
        a.tok[u] = s.st_q[2 * qv[u - g]];
        const int4 x = s.st_q[2 * qv[u - g] + 1];
        a.w[u] = make_float4(__int_as_float(x.x), __int_as_float(x.y), __int_as_float(x.z), __int_as_float(x.w));
      } else if (kPacked) {  // one 32-byte load: 4 packed arcs + 4 weights
        const uint4* p = reinterpret_cast<const uint4*>(m.arc_q) + 2 * (size_t)qv[u - g];
        int4 t;
        float4 x;
        asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(t.x), "=r"(t.y), "=r"(t.z), "=r"(t.w), "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
                     : "l"(p));
        a.tok[u] = t;
        a.w[u] = x;
      } else {
        a.tok[u] = __ldg(tok4 + qv[u - g]);
        a.w[u] = __ldg(w4 + qv[u - g]);
        a.to[u] = __ldg(to4 + qv[u - g]);
      }
    }
  }
}

template <int kW, bool kPacked>
__device__ __forceinline__ void write_window(const WSlice& s, const Window<kW, kPacked>& a, int32_t k0,
                                             int32_t nslots, int32_t pk_bits) {
  const uint32_t tmask = (1u << pk_bits) - 1u;
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
        s.row_s[tk] = __fadd_rn(a.acc[u], ww[j]);  // acc_boff + arc_weights (Alg. 1 line 74)
        s.row_n[tk] = nx;
      }
    }
  }
  __syncwarp();
}

// Root level into the row's scores: acc_root + root weight;
// all loads of a batch issued before its stores. (The root targets reach the
// next-state slots by a bulk copy.)
__device__ __forceinline__ void root_fill(const WSlice& s, const float* root_w, float ar, int32_t V) {
  const int lane = threadIdx.x & 31;
  const float4* w4 = reinterpret_cast<const float4*>(root_w);
  float4* s4 = reinterpret_cast<float4*>(s.row_s);
  const int32_t nq4 = V / 4;
  for (int32_t q0 = lane; q0 < nq4; q0 += 256) {
    float4 y[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (q0 + 32 * j < nq4) y[j] = w4[q0 + 32 * j];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (q0 + 32 * j < nq4) {
        y[j].x = __fadd_rn(ar, y[j].x);
        y[j].y = __fadd_rn(ar, y[j].y);
        y[j].z = __fadd_rn(ar, y[j].z);
        y[j].w = __fadd_rn(ar, y[j].w);
        s4[q0 + 32 * j] = y[j];
      }
  }
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// kRegRoot (V <= 1024): every lane keeps its 32 root weights in registers,
// loaded before the wait, so the root fill is register -> shared stores that
// overlap the arc gathers (shared-memory loads issued after the gathers would
// return behind them).
// kStage (packed arcs, register root): the row's arcs are bulk-copied level by
// level into the warp's staging area (when they fit), so the gathers do not
// queue in the SM's load pipeline; the write loop then reads shared memory.
template <bool kTable, int kW, bool kPacked, bool kRegRoot, bool kStage>
__global__ void __launch_bounds__(32, NGPULM_ADV_MINB(kW, kPacked, kStage))
    advance_warp_kernel(DevModel m, const int32_t* __restrict__ states, int32_t B, float* __restrict__ scores,
                        int32_t* __restrict__ next, float* __restrict__ final_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int32_t V = m.V;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, R = blockDim.x >> 5;
  const size_t rb = align16((size_t)V * 4);
  const float* root_w = reinterpret_cast<const float*>(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + rb);
  constexpr int kSQ = kStage ? kStageQuads : 0;
  static_assert(!kStage || (kPacked && kRegRoot), "staging holds packed arcs");
  const WSlice s = wcarve(smem + rb + 16 + (size_t)w * wslice_bytes(V, m.order, kSQ), V, m.order, kSQ);
  const int32_t row = (int32_t)blockIdx.x * R + w;
  const uint32_t bytes = (uint32_t)V * 4u;
  STAMP(0);
  STAMP(1);
  STAMP(9);
  pdl_trigger();
  // step 0, on immutable model data, so before the wait: the root weights
  // once per CTA, and the root targets straight into every row's next-state
  // slots (the root has an arc for every token, [0, V)).
  // kCtaRoot (register root): the root targets reach the CTA once (one bulk
  // copy into the otherwise unused root-weight buffer) and every row copies
  // them shared -> shared, so the 4 KB root level is read from L2 once per CTA
  // instead of once per row (1024 rows reading the same 32 lines at once
  // queue on their L2 slices).
  constexpr bool kCtaRoot = kRegRoot && kW == 16 && !kStage && NGPULM_CTA_ROOT;
  if (lane == 0 && row < B) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(s.bar)) : "memory");
    if (kStage) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(s.abar)) : "memory");
    if (w == 0 && (!kRegRoot || kCtaRoot))
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (!kCtaRoot) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(s.bar)), "r"(bytes)
                   : "memory");
      bulk_g2s(s.row_n, m.arc_to, bytes, s.bar);
    } else {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(s.bar)) : "memory");  // unused phase
    }
    if (w == 0 && (!kRegRoot || kCtaRoot)) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
      bulk_g2s(const_cast<float*>(root_w), kCtaRoot ? static_cast<const void*>(m.arc_to) : m.arc_w, bytes, bar);
    }
  }
  float4 rw[kRegRoot ? 8 : 1];
  if (kRegRoot && row < B) {
    const float4* w4 = reinterpret_cast<const float4*>(m.arc_w);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (lane + 32 * j < V / 4) rw[j] = __ldg(w4 + lane + 32 * j);
  }
  if (!kRegRoot || kCtaRoot) __syncthreads();  // the CTA barrier's init visible to every warp
  if (kCtaRoot && row < B) {  // model data only: before the wait
    mbar_wait(bar, 0);
    const int4* src = reinterpret_cast<const int4*>(root_w);
    int4* dst = reinterpret_cast<int4*>(s.row_n);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (lane + 32 * j < V / 4) dst[lane + 32 * j] = src[lane + 32 * j];
  }
  if (row >= B) return;  // warp 0 always has a row and waits for the CTA's bulk copy
#ifdef NGPULM_PHASE_TIMING
  const int skip = g_skip;
#else
  constexpr int skip = 0;
#endif
  float* srow = scores + (size_t)row * V;
  int32_t* nrow = next + (size_t)row * V;
  // Steps 1-3 for state st into shared memory (nothing global is written).
  // ph: parity of this build's mbarrier phases (0: first build, 1: rebuild).
  auto build = [&](int32_t st, uint32_t ph) -> Row {
    WLevel lv;
    int32_t nslots;
    const Row r = warp_row_src<kTable>(m, ValState{st}, s, lv, nslots);
    STAMP(11);
    if (r.bad) return r;
    STAMP(3);
    Window<kW, kPacked> a;
    bool staged = false;
    if (kStage) {
      // staging offsets: levels in slot order (the last level first), packed tight
      const int32_t nq = lv.info & 0xffff;
      int32_t inc = nq;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_down_sync(kFull, inc, o);
        if (lane + o < 32) inc += y;
      }
      const int32_t total = __shfl_sync(kFull, inc, 0);
      staged = total <= kSQ && !(skip & 4);
      if (staged) {
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(s.abar)),
                       "r"((uint32_t)total * 32u)
                       : "memory");
        __syncwarp();
        const int32_t off = inc - nq;
        if (nq > 0)  // lanes 1..nlev: one bulk copy per level
          bulk_g2s(s.st_q + 2 * off, reinterpret_cast<const uint4*>(m.arc_q) + 2 * (lv.beg >> 2),
                   (uint32_t)nq * 32u, s.abar);
        lv.qbase = off;
      }
    }
    if (kRegRoot) {
      if (skip & 4) nslots = 0;
      if (!staged && !(skip & 4)) load_window<kW, kPacked>(m, s, lv, r.nlev, 0, nslots, a);
      STAMP(12);
      if (!(skip & 8)) {  // root scores: acc_root + root weight, while the gathers fly
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
      }
    } else {
      mbar_wait(bar, 0);  // the CTA's root weights have landed (long ago, normally)
      // the root fill goes first: its shared-memory loads would otherwise return
      // behind the arc gathers
      if (!(skip & 8)) root_fill(s, root_w, r.acc_root, V);
      STAMP(12);
      if (skip & 4) nslots = 0;
      if (!(skip & 4)) load_window<kW, kPacked>(m, s, lv, r.nlev, 0, nslots, a);
    }
    STAMP(4);
    if (!kCtaRoot) mbar_wait(s.bar, ph);  // root targets in row_n (kCtaRoot: copied synchronously)
    __syncwarp();
    STAMP(5);
    if (staged) {
      mbar_wait(s.abar, ph);  // the row's arcs are in the staging area
      for (int32_t k0 = 0; k0 < nslots; k0 += kW) {
        load_window<kW, kPacked, true>(m, s, lv, r.nlev, k0, nslots, a);
        write_window<kW, kPacked>(s, a, k0, nslots, m.pk_bits);
      }
    } else {
      for (int32_t k0 = 0; k0 < nslots;) {
        write_window<kW, kPacked>(s, a, k0, nslots, m.pk_bits);
        k0 += kW;
        if (k0 < nslots) load_window<kW, kPacked>(m, s, lv, r.nlev, k0, nslots, a);
      }
    }
    return r;
  };
  // Speculative build: the row only needs the model (immutable)
  // and the row's state, so it is built from the state read BEFORE
  // griddepcontrol.wait — overlapping the previous kernel — and the state is
  // read again after the wait; only if it changed (the previous kernel wrote
  // it) is the row rebuilt. Outputs are written after the wait only. Both
  // reads are coherent (ld.relaxed.gpu: no stale non-coherent cache line).
  auto load_state = [&]() {
    int32_t v = 0;
    if (lane == 0) asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(states + row) : "memory");
    return __shfl_sync(kFull, v, 0);
  };
  bool waited = !NGPULM_SPECULATE;
  if (waited) pdl_wait();
  int32_t st = load_state();
  uint32_t ph = 0;
  Row r;
  for (;;) {  // one build site: at most two passes
    r = build(st, ph);
    if (r.bad && !kCtaRoot) mbar_wait(s.bar, ph);  // the phase is over before any re-arm
    if (waited) break;
    pdl_wait();
    waited = true;
    STAMP(2);
    const int32_t st1 = load_state();
    if (st1 == st) break;
    st = st1;  // the previous kernel changed the state: rebuild after the wait
    ph = 1;
    if (kCtaRoot) {  // the root targets again (the first build overwrote them)
      const int4* src = reinterpret_cast<const int4*>(root_w);
      int4* dst = reinterpret_cast<int4*>(s.row_n);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (lane + 32 * j < V / 4) dst[lane + 32 * j] = src[lane + 32 * j];
    } else if (lane == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(s.bar)), "r"(bytes)
                   : "memory");
      bulk_g2s(s.row_n, m.arc_to, bytes, s.bar);
    }
    __syncwarp();
  }
  if (lane == 0) {
    if (r.bad) atomicMin(m.bad_row, (unsigned long long)row);
    if (final_out) final_out[row] = r.bad ? __int_as_float(0x7fc00000) : r.fin;
  }
  if (r.bad) {
    for (int32_t v = lane; v < V; v += 32) { srow[v] = __int_as_float(0x7fc00000); nrow[v] = -1; }
    if (w == 0 && !kRegRoot) mbar_wait(bar, 0);
    return;
  }
  STAMP(6);
  // step 4: the row leaves by two bulk stores issued by lane 0
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0 && !(skip & 2)) {
#if NGPULM_STORE_HINT
    // outputs are streamed: first to leave L2, so the trie stays resident
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(srow),
                 "r"(smem_u32(s.row_s)), "r"(bytes), "l"(pol)
                 : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(nrow),
                 "r"(smem_u32(s.row_n)), "r"(bytes), "l"(pol)
                 : "memory");
#else
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(srow), "r"(smem_u32(s.row_s)),
                 "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(nrow), "r"(smem_u32(s.row_n)),
                 "r"(bytes)
                 : "memory");
#endif
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    STAMP(7);
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
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
  bool waited = !NGPULM_SPECULATE, bad = false;
  float fin = 0.f;
  if (waited) pdl_wait();
  int32_t st = load_state();
  for (;;) {
    build(st, bad, fin);
    if (waited) break;
    pdl_wait();
    waited = true;
    const int32_t st1 = load_state();
    if (st1 == st) break;
    st = st1;  // rebuild: the root targets again (the first build overwrote them)
    const int4* src = reinterpret_cast<const int4*>(root_to);
    int4* dst = reinterpret_cast<int4*>(s.row_n);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (lane + 32 * j < V / 4) dst[lane + 32 * j] = src[lane + 32 * j];
    __syncwarp();
  }
  if (lane == 0) {
    if (bad) atomicMin(m.bad_row, (unsigned long long)row);
    if (final_out) final_out[row] = bad ? __int_as_float(0x7fc00000) : fin;
  }
  if (bad) {
    for (int32_t v = lane; v < V; v += 32) { srow[v] = __int_as_float(0x7fc00000); nrow[v] = -1; }
    return;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(srow),
                 "r"(smem_u32(s.row_s)), "r"(bytes), "l"(pol)
                 : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(nrow),
                 "r"(smem_u32(s.row_n)), "r"(bytes), "l"(pol)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
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

// ---------------------------------------------------------------- fused greedy step
// Optional internal-LM subtraction (HAT "-ILM+LM"):
// the LM-rescored columns get fmaf(-lam, ilm[token], fmaf(lambda, lm, asr))
// (R21). ilm row b: p + b * stride, indexed by LM token (V entries).
struct AuxRow {
  const float* p;  // nullptr: no ILM term
  int64_t stride;
  float lam;
};

// (value, column) order: larger value first, then lower column (R14).
__device__ __forceinline__ bool better(float v2, int32_t c2, float v, int32_t c) {
  return v2 > v || (v2 == v && c2 < c);
}

// argmax over the CTA: warp shuffles, then the warp winners via smem.
__device__ __forceinline__ void cta_argmax(float& v, int32_t& c, const Slice& s) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float v2 = __shfl_xor_sync(kFull, v, o);
    const int32_t c2 = __shfl_xor_sync(kFull, c, o);
    if (better(v2, c2, v, c)) { v = v2; c = c2; }
  }
  if ((threadIdx.x & 31) == 0) { s.red_v[threadIdx.x >> 5] = v; s.red_c[threadIdx.x >> 5] = c; }
  __syncthreads();
  v = s.red_v[0];
  c = s.red_c[0];
#pragma unroll
  for (int i = 1; i < kWarps; ++i)
    if (better(s.red_v[i], s.red_c[i], v, c)) { v = s.red_v[i]; c = s.red_c[i]; }
  __syncthreads();  // scratch reusable
}

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
  const Row r = row_levels<kTable>(m, states + b, s);
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
  build_row(m, s, r, tma);
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
      val = __fmaf_rn(lambda, s.row_s[tok], a);  // asr + lambda * lm, one rounding
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
        states[b] = s.row_n[bc < sp ? bc : bc - 1];
        if (kMode == NGPULM_CTC) prev[b] = bc;
      }
    }
  }
}

// ---------------------------------------------------------------- fused greedy step, one warp per row
// The LM row is built in shared memory exactly as advance_warp_kernel builds
// it (root targets by bulk copy, root scores from registers, quad gathers in
// 8-slot windows, level-ordered writes) and never leaves the SM. The row's
// logits (V+1 columns) are bulk-copied into shared memory as soon as the wait
// allows — off the load pipeline, so they do not delay the state, record and
// arc loads queued behind them — except the <= 3 columns on each side of the
// copy's 16-byte-aligned interior, which two lanes load directly. The fused
// values are reduced with warp shuffles.
constexpr int kMaxColsPerLane = 33;  // (1024 + 1 + 31) / 32

// per warp: row_s | row_n | levels | 2 mbarriers | logits (V+1 floats + 16-byte slack)
__host__ __device__ constexpr size_t fslice_bytes(int32_t V, int32_t order) {
  return wslice_bytes(V, order, 0) + align16((size_t)(V + 1) * 4 + 16);
}

// Issue frame row `lrow` (ncols floats) into `buf` (column c lands at
// buf[h + c], h = (lrow & 15) / 4, so the interior copies 16-byte aligned).
__device__ __forceinline__ void issue_frame(const float* lrow, int32_t ncols, float* buf, uint64_t* bar,
                                            uint64_t pol) {
  const int lane = threadIdx.x & 31;
  const uintptr_t src = reinterpret_cast<uintptr_t>(lrow);
  const uintptr_t lo = (src + 15) & ~(uintptr_t)15, hi = (src + (uintptr_t)ncols * 4) & ~(uintptr_t)15;
  const int32_t h = (int32_t)((src & 15) / 4);
  const bool bulk = hi > lo;
  const int32_t head = bulk ? (int32_t)((lo - src) / 4) : ncols, tail = bulk ? (int32_t)((hi - src) / 4) : ncols;
  int32_t c = -1;
  if (lane < head && lane < ncols) c = lane;
  else if (lane >= 8 && lane - 8 < ncols - tail) c = tail + lane - 8;
  if (c >= 0) {  // edge column: 4-byte async copy; the mbarrier's pending count covers it until it lands
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(buf + h + c)), "l"(lrow + c) : "memory");
    asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
  }
  __syncwarp();
  if (lane == 0) {
    const uint32_t bytes = bulk ? (uint32_t)(hi - lo) : 0u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    if (bulk)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
              smem_u32(buf + h + head)),
          "l"(lo), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
          : "memory");
  }
}

// Total order of floats as unsigned keys (larger float -> larger key).
__device__ __forceinline__ uint32_t fkey(float v) {
  const uint32_t u = __float_as_uint(v);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Argmax over a row held in registers, lane i holding columns i + 32 j (R14):
// the largest value (NaN never taken), then the lowest column holding it, by
// two warp reductions. Returns INT_MAX when every value is NaN.
__device__ __forceinline__ int32_t warp_argmax_cols(const float (&v)[kMaxColsPerLane]) {
  const int lane = threadIdx.x & 31;
  float mx[kMaxColsPerLane];
#pragma unroll
  for (int j = 0; j < kMaxColsPerLane; ++j) mx[j] = v[j];
#pragma unroll
  for (int d = 1; d < kMaxColsPerLane; d *= 2)
#pragma unroll
    for (int j = 0; j + d < kMaxColsPerLane; j += 2 * d) mx[j] = fmaxf(mx[j], mx[j + d]);
  const float lmax = mx[0] == mx[0] ? mx[0] : -INFINITY;
  const uint32_t kmax = __reduce_max_sync(kFull, fkey(lmax));
  const float M = __uint_as_float((kmax & 0x80000000u) ? (kmax ^ 0x80000000u) : ~kmax);
  int32_t cm = INT_MAX;
#pragma unroll
  for (int j = kMaxColsPerLane - 1; j >= 0; --j)
    if (v[j] == M) cm = lane + 32 * j;
  return (int32_t)__reduce_min_sync(kFull, (uint32_t)cm);
}

// The same over the lane columns j in [J0, J1) only; also returns the maximum
// (-inf with column INT_MAX when every value there is NaN).
template <int J0, int J1>
__device__ __forceinline__ int32_t warp_argmax_range(const float (&v)[kMaxColsPerLane], float& M) {
  const int lane = threadIdx.x & 31;
  constexpr int N = J1 - J0;
  float mx[N];
#pragma unroll
  for (int j = 0; j < N; ++j) mx[j] = v[J0 + j];
#pragma unroll
  for (int d = 1; d < N; d *= 2)
#pragma unroll
    for (int j = 0; j + d < N; j += 2 * d) mx[j] = fmaxf(mx[j], mx[j + d]);
  const float lmax = mx[0] == mx[0] ? mx[0] : -INFINITY;
  const uint32_t kmax = __reduce_max_sync(kFull, fkey(lmax));
  M = __uint_as_float((kmax & 0x80000000u) ? (kmax ^ 0x80000000u) : ~kmax);
  int32_t cm = INT_MAX;
#pragma unroll
  for (int j = J1 - 1; j >= J0; --j)
    if (v[j] == M) cm = lane + 32 * j;
  return (int32_t)__reduce_min_sync(kFull, (uint32_t)cm);
}

// Transducer label-looping bookkeeping (
// SPEC.md:317-325): with kMode == kLoop the fused step makes the RNN-T
// two-stage decision for the rows whose frame index is inside their length,
// then moves each row's loop state: blank -> next frame; a label -> emitted,
// LM advance, one more symbol on this frame, and after max_sym symbols the
// frame advances anyway.
constexpr int kLoop = 3;
struct Loop {
  int32_t* frame;        // [B] current frame of the row
  int32_t* sym;          // [B] symbols emitted on the current frame
  const int32_t* len;    // [B] frames of the row
  int32_t* emit;         // [B, max_len] emitted columns
  int32_t* emit_len;     // [B] emissions so far (may exceed max_len: truncated)
  int32_t* last;         // [B] last emitted LM token (-1 none), or nullptr
  int32_t max_sym, max_len;
};

template <int kMode, bool kTable, bool kPacked, bool kAux>
__global__ void __launch_bounds__(256, 1)
    fused_warp_kernel(DevModel m, const float* __restrict__ logits, int64_t row_stride, int32_t B,
                      int32_t* __restrict__ states, int32_t* __restrict__ prev, const uint8_t* __restrict__ active,
                      float lambda, int32_t sp, AuxRow aux, Loop lp, int32_t* __restrict__ tokens_out) {
  constexpr int kW = 8;
  constexpr bool kTwo = kMode == NGPULM_RNNT || kMode == kLoop;  // two-stage transducer selection
  extern __shared__ __align__(16) unsigned char smem[];
  const int32_t V = m.V, ncols = V + 1;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, R = blockDim.x >> 5;
  unsigned char* base = smem + (size_t)w * fslice_bytes(V, m.order);
  const WSlice s = wcarve(base, V, m.order, 0);
  uint64_t* lbar = s.abar;
  float* lbuf = reinterpret_cast<float*>(base + wslice_bytes(V, m.order, 0));
  const int32_t row = (int32_t)blockIdx.x * R + w;
  STAMP(0);
  STAMP(1);
  STAMP(9);
  pdl_trigger();
  if (row >= B) return;
  if (lane == 0) {  // root targets -> the row's next-state slots (immutable model data: before the wait)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(s.bar)) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(lbar)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(s.bar)), "r"((uint32_t)V * 4u)
                 : "memory");
    bulk_g2s(s.row_n, m.arc_to, (uint32_t)V * 4u, s.bar);
  }
  float4 rw[8];
  {
    const float4* w4 = reinterpret_cast<const float4*>(m.arc_w);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (lane + 32 * j < V / 4) rw[j] = __ldg(w4 + lane + 32 * j);
  }
  pdl_wait();
  STAMP(2);
  const float* lrow = logits + (size_t)row * row_stride;
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
  WLevel lv;
  int32_t nslots;
  bool started = false;
  auto begin_logits = [&]() {  // the logits' copy, issued once the chain record is in flight
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));  // read once
    issue_frame(lrow, ncols, lbuf, lbar, pol);
    started = true;
  };
  const Row r = warp_row<kTable>(m, states + row, s, lv, nslots, begin_logits);
  const float* lb = lbuf + (reinterpret_cast<uintptr_t>(lrow) & 15) / 4;  // column c at lb[c]
  STAMP(11);
  if (!on || r.bad) {  // inactive rows are untouched (their state is not even checked)
    if (lane == 0) {
      tokens_out[row] = -1;
      if (on) atomicMin(m.bad_row, (unsigned long long)row);
      if (kMode == kLoop && on) lp.frame[row] = lp.len[row];  // an invalid state ends the row's loop
    }
    mbar_wait(s.bar, 0);  // no exit with a bulk copy in flight
    if (started) mbar_wait(lbar, 0);
    return;
  }
  // (RNN-T: the LM row is built before stage 1 is known — it waits for the
  // logits — and is simply not used when blank wins)
  Window<kW, kPacked> a;
  load_window<kW, kPacked>(m, s, lv, r.nlev, 0, nslots, a);
  STAMP(3);
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
  STAMP(4);
  mbar_wait(s.bar, 0);
  __syncwarp();
  STAMP(5);
  for (int32_t k0 = 0; k0 < nslots;) {
    write_window<kW, kPacked>(s, a, k0, nslots, m.pk_bits);
    k0 += kW;
    if (k0 < nslots) load_window<kW, kPacked>(m, s, lv, r.nlev, k0, nslots, a);
  }
  STAMP(6);
  mbar_wait(lbar, 0);
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
        const float lmv = col < ncols && col != sp ? s.row_s[col - (col > sp)] : sp_val;
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
      const bool ok = bc >= 0 && bc < ncols;
      tokens_out[row] = ok ? bc : -1;
      int32_t fr = lp.frame[row], sy = lp.sym[row];
      if (!ok || bc == sp) {  // blank (or an all-NaN row): next frame
        ++fr;
        sy = 0;
      } else {  // a label: emit it, advance the LM, stay on the frame (up to max_sym symbols)
        const int32_t tok = bc < sp ? bc : bc - 1;
        const int32_t e = lp.emit_len[row];
        if (e < lp.max_len) lp.emit[(size_t)row * lp.max_len + e] = bc;
        lp.emit_len[row] = e + 1;
        if (lp.last) lp.last[row] = tok;
        states[row] = s.row_n[tok];
        if (++sy >= lp.max_sym) {
          ++fr;
          sy = 0;
        }
      }
      lp.frame[row] = fr;
      lp.sym[row] = sy;
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
        states[row] = s.row_n[bc < sp ? bc : bc - 1];
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

template <int kMode, bool kTable, bool kPacked, bool kAux>
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
  pdl_trigger();
  if (row >= B) return;
  if (lane == 0) {  // A: root targets -> next-state slots; B: the logits barrier (model data / no inputs: before the wait)
    const uint64_t* bb = role == 0 ? s.bar : lbar;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bb)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (role == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(s.bar)),
                   "r"((uint32_t)V * 4u)
                   : "memory");
      bulk_g2s(s.row_n, m.arc_to, (uint32_t)V * 4u, s.bar);
    }
  }
  float4 rw[8];
  if (role == 0) {
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
      issue_frame(lrow, ncols, lbuf, lbar, pol);
      mbar_wait(lbar, 0);
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
    }
    pair_sync();  // (1) the row is built (or the row is done)
    if (xch[3]) return;
    fin = __int_as_float(xch[4]);
  } else {
    WLevel lv;
    int32_t nslots;
    const Row r = warp_row<kTable>(m, states + row, s, lv, nslots);
    if (!on || r.bad) {
      if (lane == 0) {
        tokens_out[row] = -1;
        if (on) atomicMin(m.bad_row, (unsigned long long)row);
        if (kMode == kLoop && on) lp.frame[row] = lp.len[row];
        xch[3] = 1;
      }
      mbar_wait(s.bar, 0);
      pair_sync();
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
        const float lmv = col < ncols && col != sp ? s.row_s[col - (col > sp)] : sp_val;
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
      const bool ok = bc >= 0 && bc < ncols;
      tokens_out[row] = ok ? bc : -1;
      int32_t fr = lp.frame[row], sy = lp.sym[row];
      if (!ok || bc == sp) {
        ++fr;
        sy = 0;
      } else {
        const int32_t tok = bc < sp ? bc : bc - 1;
        const int32_t e = lp.emit_len[row];
        if (e < lp.max_len) lp.emit[(size_t)row * lp.max_len + e] = bc;
        lp.emit_len[row] = e + 1;
        if (lp.last) lp.last[row] = tok;
        states[row] = s.row_n[tok];
        if (++sy >= lp.max_sym) {
          ++fr;
          sy = 0;
        }
      }
      lp.frame[row] = fr;
      lp.sym[row] = sy;
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
        states[row] = s.row_n[bc < sp ? bc : bc - 1];
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
    issue_frame(lrow, ncols, lbuf, lbar, pol);
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
    if (started) mbar_wait(lbar, 0);
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

template <bool kTable, bool kPacked>
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
  int32_t st = __ldg(&states[row]);
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
        const int32_t ns = s.row_n[bc < sp ? bc : bc - 1];
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
    states[row] = st;
    prev[row] = pc;
    if (emit_len) emit_len[row] = nemit;
  }
}

// ---------------------------------------------------------------- launch
template <typename... KArgs, typename... Args>
int launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return (int)cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace

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
                   float* final_out, void* stream) {
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
    // up to 8 rows per SM: 16-slot windows (almost every row in one window),
    // packed arcs bulk-copied into a staging area; more rows per SM: 8-slot
    // windows of direct gathers (registers and shared memory for occupancy)
    const bool wide = B <= NGPULM_WIDE_MAX_B, pk = m.arc_q != nullptr && m.adv_kind == NGPULM_ADVANCE_AUTO;
    const bool small_v = m.V <= 1024, stage = B >= 2 && B <= NGPULM_STAGE_MAX_B && pk && small_v && table;
    const int sq = stage ? kStageQuads : 0;
    // one row (warp) per CTA: a CTA leaves as soon as its row is stored and the
    // next call's CTA starts its speculative build in its place (B=1024: 7 rows
    // per CTA 3.29 us, 1 row 2.83 us; B=4096: 10.1 -> 9.4 us)
    const int R = 1;
    if (wcta_smem(m.V, m.order, R, sq) <= 227 * 1024) {
      const size_t wsm = wcta_smem(m.V, m.order, R, sq);
      const dim3 wg((B + R - 1) / R), wb(32 * R);
      if (stage)
        return launch(advance_warp_kernel<true, 16, true, true, true>, wg, wb, wsm, st, m, states, B, scores, next,
                      final_out);
#define NGPULM_WARP_LAUNCH(T, W, P)                                                                               \
  return small_v ? launch(advance_warp_kernel<T, W, P, true, false>, wg, wb, wsm, st, m, states, B, scores, next, \
                          final_out)                                                                                \
                 : launch(advance_warp_kernel<T, W, P, false, false>, wg, wb, wsm, st, m, states, B, scores, next,  \
                          final_out)
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

template <int kMode>
int launch_fused_mode(const DevModel& m, const float* logits, int64_t row_stride, int32_t B, int32_t* states,
                      int32_t* prev, const uint8_t* active, float lambda, int32_t blank, AuxRow aux,
                      int32_t* tokens_out, cudaStream_t st) {
  if (m.V % 4 == 0 && m.V <= 1024 && m.adv_kind != NGPULM_ADVANCE_CTA) {
    const bool pk = m.arc_q != nullptr && m.adv_kind == NGPULM_ADVANCE_AUTO, table = m.chain != nullptr;
    if (kMode == NGPULM_RNNT && B <= NGPULM_PAIR_MAX_B) {  // two warps per row (stage 1 beside the row build)
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
#define NGPULM_DECODE_LAUNCH(TB, P)                                                                                  \
  return launch(ctc_decode_kernel<TB, P>, g, b, sm, st, m, logits, row_stride, frame_stride, B, T, lengths, states, \
                prev, lambda, blank, depth, frames_out, emit_out, emit_len)
  if (table) { if (pk) NGPULM_DECODE_LAUNCH(true, true); NGPULM_DECODE_LAUNCH(true, false); }
  if (pk) NGPULM_DECODE_LAUNCH(false, true);
  NGPULM_DECODE_LAUNCH(false, false);
#undef NGPULM_DECODE_LAUNCH
}

int launch_fused(const DevModel& m, int32_t mode, const float* logits, int64_t row_stride, int32_t B,
                 int32_t* states, int32_t* prev, const uint8_t* active, float lambda, int32_t blank,
                 const float* aux, int64_t aux_stride, float lambda_ilm, int32_t* tokens_out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const AuxRow ax{aux, aux_stride, lambda_ilm};
  switch (mode) {
    case NGPULM_CTC:
      return launch_fused_mode<NGPULM_CTC>(m, logits, row_stride, B, states, prev, active, lambda, blank, ax,
                                           tokens_out, st);
    case NGPULM_RNNT:
      return launch_fused_mode<NGPULM_RNNT>(m, logits, row_stride, B, states, prev, active, lambda, blank, ax,
                                            tokens_out, st);
    default:
      return launch_fused_mode<NGPULM_AED>(m, logits, row_stride, B, states, prev, active, lambda, blank, ax,
                                           tokens_out, st);
  }
}

int launch_transducer_loop(const DevModel& m, const float* logits, int64_t row_stride, int32_t B, int32_t* states,
                           int32_t* frame, int32_t* sym, const int32_t* lengths, int32_t max_sym, float lambda,
                           int32_t blank, const float* aux, int64_t aux_stride, float lambda_ilm,
                           int32_t* tokens_out, int32_t* emit, int32_t* emit_len, int32_t* last, int32_t max_len,
                           void* stream) {
  if (m.V % 4 != 0 || m.V > 1024) return (int)cudaErrorNotSupported;
  int R = (B + 147) / 148;
  R = R < 1 ? 1 : (R > 8 ? 8 : R);
  const size_t wsm = (size_t)R * fslice_bytes(m.V, m.order);
  const dim3 wg((B + R - 1) / R), wb(32 * R);
  const bool pk = m.arc_q != nullptr && m.adv_kind == NGPULM_ADVANCE_AUTO, table = m.chain != nullptr;
  const AuxRow ax{aux, aux_stride, lambda_ilm};
  const Loop lp{frame, sym, lengths, emit, emit_len, last, max_sym, max_len};
  cudaStream_t st = (cudaStream_t)stream;
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
