// Shared device code of the NGPU-LM kernels (advance.cu, fused.cu, decode.cu):
// row layout in shared memory, the chain-record and arc-window helpers, the
// logits staging and the warp argmax, the launch helper.
#pragma once
// NGPU-LM hot path for sm_100a: batched full-vocabulary query (Algorithm 1,
// PAPER.md:54-89) and the fused greedy shallow-fusion step.
//
// A row (the LM scores and next states of one state over the vocabulary)
// lives in shared memory as (score, next state) per token, 8 KB at V = 1024,
// and is built in four steps:
//  0. prologue on immutable model data, before griddepcontrol.wait
//     (programmatic dependent launch): the root level (an arc
//     for every token) — targets by TMA bulk copy into the next-state slots,
//     weights into registers;
//  1. the row's back-off levels (Algorithm 1 lines 72, 81-82) from the
//     load-time chain table (one 16-byte record slot per level and lane,
//     acc_boff accumulated left to right in float, R10), or Algorithm 1's
//     literal walk;
//  2. the levels' arcs, cut into slots of 32 16-byte quads, gathered into
//     registers a window of slots at a time, while the root scores
//     acc_root + root weight are stored;
//  3. slots written in level order, lowest order first, so a higher-order arc
//     overwrites a lower-order one — Algorithm 1's "first level found wins"
//     (lines 77-79) with plain shared-memory stores, no atomics.
// advance.cu stores the row by TMA bulk copies (one warp per row and per CTA,
// steps 1-3 speculatively before the PDL wait); fused.cu and decode.cu feed
// it to the fused argmax and it never touches HBM. The CTA-per-row kernels
// (one 256-thread CTA per row or vocabulary tile) serve unaligned outputs and
// rows beyond shared memory. No tensor cores: gathers, shared-memory scatter
// and store bandwidth only (DESIGN.md §7 Roofline).
#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <cstdint>
#include <map>
#include <mutex>
#include <type_traits>
#include <utility>

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
#ifndef NGPULM_FUSED_SPECULATE
#define NGPULM_FUSED_SPECULATE 1
#endif
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
// (8-slot windows: 16 CTAs per SM = 128 registers, measured B=4096 9.46 ->
// 8.16 us, B=128 1.90 -> 1.66 us; the 16-slot path keeps its 245 registers:
// capped it spills, B=1024 2.82 -> 4.29)
#ifndef NGPULM_ADV_MINB_WIDE
#define NGPULM_ADV_MINB_WIDE 8
#endif
#ifndef NGPULM_ADV_MINB_PACKED8
#define NGPULM_ADV_MINB_PACKED8 16
#endif
#ifndef NGPULM_ADV_MINB_UNPACKED8
#define NGPULM_ADV_MINB_UNPACKED8 10
#endif
#define NGPULM_ADV_MINB(kW, kPacked) \
  ((kW) == 8 ? ((kPacked) ? NGPULM_ADV_MINB_PACKED8 : NGPULM_ADV_MINB_UNPACKED8) : NGPULM_ADV_MINB_WIDE)
#ifndef NGPULM_TINY_MAX_B
#define NGPULM_TINY_MAX_B 148  // tiny LM in shared memory up to one row per SM (B=128: 1.34 vs 1.66 us);
#endif                         // beyond, the one-row-per-CTA global kernel wins (B=1024: 2.53 vs 3.08)
#ifndef NGPULM_TINY_ROWS
#define NGPULM_TINY_ROWS 8
#endif
#ifndef NGPULM_ADV_ROWS
#define NGPULM_ADV_ROWS 1  // rows (warps) per CTA of the warp advance kernel
#endif
#ifndef NGPULM_FUSED_MAX_ROWS
#define NGPULM_FUSED_MAX_ROWS 8
#endif
#ifndef NGPULM_WIDE_MAX_B
#define NGPULM_WIDE_MAX_B (4 * 148)  // up to 4 rows per SM: 16-slot windows, 8 CTAs per SM; beyond, 8-slot
                                     // windows at 16 CTAs per SM (B=1024: 2.64 -> 2.53 us, B=128: 1.43 vs 1.55)
#endif

__host__ __device__ constexpr size_t wrow_bytes(int32_t V) { return align16((size_t)V * 4 + 4); }  // + trash word
#ifndef NGPULM_PAD_GRID
#define NGPULM_PAD_GRID 148
#endif
#ifndef NGPULM_PAD_MODE
#define NGPULM_PAD_MODE 1
#endif
#ifndef NGPULM_PAD_MIN_B
#define NGPULM_PAD_MIN_B 65
#endif
__host__ __device__ constexpr size_t wslice_bytes(int32_t V, int32_t order, int stage_q) {
  return 2 * wrow_bytes(V) + levels_bytes(order) + 16 + (size_t)stage_q * 32;
}
// root_w[V] | mbarrier | R x (row_s[V+1] | row_n[V+1] | levels | 2 mbarriers | stage_q arc quads)
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
  uint64_t* abar;  // second mbarrier (the fused kernels' logits copy)
  int4* st_q;      // packed arc quads read from shared memory (tiny-LM kernels: the CTA's model copy)
  const int4* chain_s;  // tiny-LM kernels: the CTA's copy of the chain table
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
  s.chain_s = nullptr;
  return s;
}

// Tiny LMs (keyword-biasing size): the chain
// table and the packed arc quads copied into a CTA's shared memory (before
// griddepcontrol.wait: model data is immutable), so a row's record and arc
// quads are shared loads. Layout: chain | arc quads | mbarrier.
__host__ __device__ constexpr size_t tiny_copy_bytes(int64_t chain_bytes, int64_t arcq_bytes) {
  return align16((size_t)chain_bytes) + align16((size_t)arcq_bytes) + 16;
}
__device__ __forceinline__ uint64_t* tiny_bar(unsigned char* base, const DevModel& m) {
  return reinterpret_cast<uint64_t*>(base + align16((size_t)m.tiny_chain_bytes) + align16((size_t)m.tiny_arcq_bytes));
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
// kSmemModel: the chain record comes from the CTA's tiny-LM copy (s.chain_s).
template <bool kTable, typename F = NoOp, typename SF = PtrState, bool kSmemModel = false>
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
    if (lane < slots) x = kSmemModel ? s.chain_s[(size_t)st * slots + lane] : __ldg(table + (size_t)st * slots);
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

// The tiny-LM copy into `base` (tiny_copy_bytes), issued by one thread; the
// caller makes the barrier init visible to the CTA (__syncthreads) and every
// row waits on tiny_bar (phase 0) before its first record read.
__device__ __forceinline__ void tiny_copy_issue(const DevModel& m, unsigned char* base) {
  uint64_t* bar = tiny_bar(base, m);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"((uint32_t)(m.tiny_chain_bytes + m.tiny_arcq_bytes))
               : "memory");
  bulk_g2s(base, m.chain, (uint32_t)m.tiny_chain_bytes, bar);
  bulk_g2s(base + align16((size_t)m.tiny_chain_bytes), m.arc_q, (uint32_t)m.tiny_arcq_bytes, bar);
}

// A ring slot's consumers are done with it: every lane's generic reads of the
// slot are ordered before the async-proxy (TMA / cp.async) writes that refill
// it (proxy fence + warp sync), then lane 0 arrives on the slot's "empty"
// mbarrier (release).
__device__ __forceinline__ void release_slot(uint64_t* empty) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if ((threadIdx.x & 31) == 0)
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty)) : "memory");
}
// After waiting on an mbarrier that tracks this thread's cp.async (edge
// columns of issue_frame): the thread's own completion wait (a no-op by then;
// the mbarrier phase already implies it) so every cp.async has a matching wait.
__device__ __forceinline__ void cp_async_settle() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Generic-proxy shared-memory writes -> later async-proxy accesses (a bulk
// store reading the row, or a bulk copy overwriting it): every writing lane
// fences, then the warp synchronizes before one lane issues the bulk op.
__device__ __forceinline__ void proxy_fence_warp() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
}

// Re-arm the row's root-target copy (advance / fused step rebuild after the
// PDL wait): the previous build overwrote row_n with generic stores, so the
// warp fences before the bulk copy is issued (write-after-write across proxies).
__device__ __forceinline__ void rearm_root_targets(const WSlice& s, const int32_t* root_to, uint32_t bytes) {
  proxy_fence_warp();
  if ((threadIdx.x & 31) == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(s.bar)), "r"(bytes)
                 : "memory");
    bulk_g2s(s.row_n, root_to, bytes, s.bar);
  }
  __syncwarp();
}

// The row leaves by two bulk stores (scores, next) issued by lane 0, with an
// L2 evict-first policy: outputs are streamed, the trie should stay in L2.
// The caller has fenced (proxy_fence_warp) after the row's last generic write.
__device__ __forceinline__ void store_row_bulk(const WSlice& s, float* srow, int32_t* nrow, uint32_t bytes) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(srow),
               "r"(smem_u32(s.row_s)), "r"(bytes), "l"(pol)
               : "memory");
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(nrow),
               "r"(smem_u32(s.row_n)), "r"(bytes), "l"(pol)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
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
  return wslice_bytes(V, order, 0) + align16((size_t)(V + 1) * 4 + 32);  // (+ a 16-byte-aligned cover's slack)
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

// issue_frame when the frame's 16-byte-aligned cover [floor16(lrow),
// ceil16(lrow + ncols)) lies inside [lo, hi) (the bytes the caller's logits
// view spans): ONE bulk copy of the cover by lane 0 (the few columns of the
// neighbouring frames it also brings are never read); column c lands at
// buf[h + c] as with issue_frame. Otherwise (the first / last frame of the
// view, unaligned) issue_frame's interior + edge copies. Warp-uniform call.
__device__ __forceinline__ void issue_frame_cover(const float* lrow, int32_t ncols, float* buf, uint64_t* bar,
                                                  uint64_t pol, const float* lo, const float* hi) {
  const uintptr_t src = reinterpret_cast<uintptr_t>(lrow);
  const uintptr_t c0 = src & ~(uintptr_t)15, c1 = (src + (uintptr_t)ncols * 4 + 15) & ~(uintptr_t)15;
  if (c0 >= reinterpret_cast<uintptr_t>(lo) && c1 <= reinterpret_cast<uintptr_t>(hi)) {
    if ((threadIdx.x & 31) == 0) {
      const uint32_t bytes = (uint32_t)(c1 - c0);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
              smem_u32(buf)),
          "l"(c0), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
          : "memory");
    }
    return;
  }
  issue_frame(lrow, ncols, buf, bar, pol);
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
// Token-and-Duration Transducer (TDT; R25), D > 0:
// the row also carries D duration logits; the duration is their raw argmax
// (lowest index on ties, untouched by the LM): a blank advances the frame by
// max(d, 1), a label by d (d = 0: same frame, up to max_sym labels).
constexpr int kLoop = 3;
constexpr int kMaxDur = NGPULM_MAX_DURATIONS;  // (include/ngpulm.h)
struct Loop {
  int32_t* frame;        // [B] current frame of the row
  int32_t* sym;          // [B] symbols emitted on the current frame
  const int32_t* len;    // [B] frames of the row
  int32_t* emit;         // [B, max_len] emitted columns
  int32_t* emit_len;     // [B] emissions so far (may exceed max_len: truncated)
  int32_t* last;         // [B] last emitted LM token (-1 none), or nullptr
  int32_t max_sym, max_len;
  const float* dur;      // TDT: row b's duration logits at dur + b * dur_stride (D entries), or nullptr
  int64_t dur_stride;
  int32_t D;             // number of durations (0: RNN-T)
  int32_t durs[kMaxDur]; // frames advanced by duration index j
};

// TDT duration of a row: the whole warp takes the raw argmax of the D duration
// logits (NaN never taken, lowest index on ties; an all-NaN row takes index 0)
// and returns durs[index] to every lane.
__device__ __forceinline__ int32_t tdt_duration(const Loop& lp, int32_t row) {
  const int lane = threadIdx.x & 31;
  float x = -INFINITY;
  if (lane < lp.D) {
    x = __ldg(lp.dur + (size_t)row * lp.dur_stride + lane);
    if (x != x) x = -INFINITY;
  }
  const uint32_t kmax = __reduce_max_sync(kFull, fkey(lane < lp.D ? x : -INFINITY));
  const float M = __uint_as_float((kmax & 0x80000000u) ? (kmax ^ 0x80000000u) : ~kmax);
  uint32_t idx = __reduce_min_sync(kFull, (lane < lp.D && x == M) ? (uint32_t)lane : 0xffffffffu);
  if (idx >= (uint32_t)lp.D) idx = 0;
  int32_t dv = 0;
#pragma unroll
  for (int j = 0; j < kMaxDur; ++j)
    if (lane == j) dv = lp.durs[j];
  return __shfl_sync(kFull, dv, (int)idx);
}

// The loop bookkeeping of one row after its decision bc (lane 0; d = the TDT
// duration or -1 for RNN-T). states == nullptr: no LM state (plain greedy).
__device__ __forceinline__ void loop_epilogue(const Loop& lp, int32_t row, int32_t bc, int32_t sp, int32_t ncols,
                                              int32_t* states, int32_t next_state, int32_t d,
                                              int32_t* tokens_out) {
  const bool ok = bc >= 0 && bc < ncols;
  tokens_out[row] = ok ? bc : -1;
  int32_t fr = lp.frame[row], sy = lp.sym[row];
  if (!ok || bc == sp) {  // blank (or an all-NaN row): next frame (TDT: max(d, 1) frames)
    fr += d > 1 ? d : 1;
    sy = 0;
  } else {  // a label: emit it, advance the LM, stay on the frame (up to max_sym symbols)
    const int32_t tok = bc < sp ? bc : bc - 1;
    const int32_t e = lp.emit_len[row];
    if (e < lp.max_len) lp.emit[(size_t)row * lp.max_len + e] = bc;
    lp.emit_len[row] = e + 1;
    if (lp.last) lp.last[row] = tok;
    if (states) states[row] = next_state;
    if (d > 0) {  // TDT: the label's duration moves the frame
      fr += d;
      sy = 0;
    } else if (++sy >= lp.max_sym) {
      ++fr;
      sy = 0;
    }
  }
  lp.frame[row] = fr;
  lp.sym[row] = sy;
}

// ---------------------------------------------------------------- launch
// The dynamic shared-memory limit of a kernel is raised once per (device,
// kernel) to the largest size seen, not on every launch (cudaFuncSetAttribute
// is a driver call).
inline int ensure_smem(const void* kern, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[{dev, kern}];
  if (smem <= have) return 0;
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  have = smem;
  return 0;
}

// Kernels whose residency is sized by several CTAs' shared memory per SM ask
// for the largest shared-memory carveout once per (device, kernel).
inline int ensure_max_carveout(const void* kern) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, bool> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  bool& d = done[{dev, kern}];
  if (d) return 0;
  const cudaError_t e =
      cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return (int)e;
  d = true;
  return 0;
}

template <typename... KArgs, typename... Args>
int launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  if (smem > 48 * 1024) {
    const int e = ensure_smem((const void*)kern, smem);
    if (e) return e;
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

// The largest row the CTA kernels hold in shared memory, and the advance tile (advance.cu).
int max_row_in_smem(int32_t order);
int32_t vocab_tile(int32_t V, int32_t order);
}  // namespace ngpulm
