// Internal types of libngpulm (product code; never seen by the oracle).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/ngpulm.h"

namespace ngpulm {

// One 16-byte record per state: the chain walk (Algorithm 1 lines 72, 81, 82)
// reads exactly one aligned sector per back-off level.
struct alignas(16) StateRec {
  int32_t arc_begin;  // start_arcs[state]
  int32_t arc_end;    // end_arcs[state]
  int32_t boff_to;    // boff_to_states[state]
  float boff_w;       // boff_weights[state]
};

// The flat trie on the host (SPEC.md:95-111 FlatLM).
struct HostModel {
  int32_t V = 0, order = 0, num_states = 0, bos_state = 0;
  int64_t num_unk_filled = 0, num_dropped = 0;
  std::vector<int32_t> arc_tok, arc_to;  // [A]
  std::vector<float> arc_w;              // [A]
  std::vector<int32_t> arc_off;          // [S+1]
  std::vector<int32_t> boff_to;          // [S]
  std::vector<float> boff_w, final_w;    // [S]
  // (parent state, token) -> child state: the prefix edges of the context trie
  std::vector<uint64_t> child_keys;
  std::vector<int32_t> child_vals;
  uint64_t child_mask = 0;

  int32_t child(int32_t parent, int32_t tok) const;
};

// Parse + validate + build. Returns NGPULM_OK or an error code with `err` set.
int build_from_arpa(const char* arpa_path, const char* vocab_path, int32_t vocab_size,
                    HostModel& out, std::string& err);

// NGLM binary files (nglm.cpp) and the prefix-edge map
// rebuilt from the flat arrays (build.cpp).
int save_binary(const HostModel& m, const char* path, std::string& err);
int load_binary(const char* path, HostModel& m, std::string& err);
bool rebuild_child_map(HostModel& m, std::string& err);

// Device arc layout: state s's arcs start at
// arc_begin[s], a multiple of 4 (one 16-byte quad); the gap before the next
// state repeats the state's last arc, so a whole quad can be written into a
// row (a repeated arc rewrites the value it already wrote). Returns the
// padded arc count.
size_t device_arc_layout(const HostModel& m, std::vector<int32_t>& arc_begin);

// Bits of the token field in a packed arc ((target << bits) | token), and
// whether every target fits the remaining bits.
int32_t packed_token_bits(int32_t V);
bool packable(const HostModel& m);

// Load-time chain table (DESIGN.md §Kernels "chain table"): per state a fixed
// record of `slots` int4: slot 0 = {nlev, acc_root, final, total_arcs}, slots
// 1..nlev = {arc_begin, arc_prefix, acc_boff, (first_slot << 16) | quads} for
// every level of the back-off chain that has arcs, in Algorithm 1 order
// (quads: 16-byte groups the level's arcs span; slots: 32-quad groups,
// numbered from the last level); padding slots = {0, total_arcs, 0, 0}.
// acc_boff is accumulated exactly as Algorithm 1 does (left to right, float).
// slots = max(1, order).
// Arc begins are the device layout's.
void build_chain_table(const HostModel& m, const std::vector<int32_t>& arc_begin, std::vector<int32_t>& out,
                       int32_t& slots);

// Load-time bound for the bound-pruned CTC decode: per state s,
// ub[s] = max over the levels L of its back-off chain (root included) of
// fadd(acc_boff_L, max arc weight of level L), in float with the kernels'
// rounding (fadd is monotone), so ub[s] >= every score of the row of s
// (Algorithm 1 takes each token's score from one of these levels).
void build_row_bounds(const HostModel& m, std::vector<float>& ub);

// Device-side view passed to kernels by value.
struct DevModel {
  const StateRec* srec;
  const float* final_w;
  const int32_t* arc_tok;
  const float* arc_w;
  const int32_t* arc_to;
  const void* chain;  // chain table (int4 records) or nullptr = walk the chain at query time
  int32_t chain_slots;
  int32_t S, V, order;
  // packed arc quads, or nullptr (targets too large): 32-byte units, one per
  // 4 arcs of the device layout: {u32 (target << pk_bits) | token [4], f32 weight [4]}
  const void* arc_q;
  int32_t pk_bits;
  int32_t adv_kind;             // NGPULM_ADVANCE_*
  unsigned long long* bad_row;  // sticky min bad row (ULLONG_MAX = none)
  // tiny LMs: bytes of the chain table and of the packed arc quads, both
  // staged into shared memory by the advance kernel (0: not a tiny LM)
  int32_t tiny_chain_bytes, tiny_arcq_bytes;
  const float* lm_ub;  // [S] build_row_bounds
};

// Kernel launchers (advance.cu, fused.cu, decode.cu). Return cudaError_t as int.
int launch_advance(const DevModel& m, const int32_t* states, int32_t B, float* scores,
                   int32_t* next, float* final_out, void* stream, uint32_t flags = 0);
int launch_final(const DevModel& m, const int32_t* states, int32_t B, float* out, void* stream);
int launch_fused(const DevModel& m, int32_t mode, const float* logits, int64_t row_stride,
                 int32_t B, int32_t* states, int32_t* prev, const uint8_t* active, float lambda,
                 int32_t blank, const float* aux, int64_t aux_stride, float lambda_ilm,
                 int32_t* tokens_out, void* stream, uint32_t flags = 0);
int launch_fused_rows(int32_t mode, const float* logits, int64_t row_stride, const float* lm_s, const int32_t* lm_n,
                      const float* lm_f, int64_t lm_stride, int32_t B, int32_t V, int32_t* states, int32_t* prev,
                      const uint8_t* active, float lambda, int32_t blank, int32_t* tokens_out, void* stream);
int launch_transducer_loop(const DevModel& m, const float* logits, int64_t row_stride, int32_t B, int32_t* states,
                           int32_t* frame, int32_t* sym, const int32_t* lengths, int32_t max_sym, float lambda,
                           int32_t blank, const float* aux, int64_t aux_stride, float lambda_ilm,
                           int32_t* tokens_out, int32_t* emit, int32_t* emit_len, int32_t* last, int32_t max_len,
                           const float* dur, int64_t dur_stride, const int32_t* durations, int32_t D,
                           uint32_t flags, void* stream);
int launch_topk(const DevModel& m, const float* logits, int64_t row_stride, int32_t B, const int32_t* states,
                const float* aux, int64_t aux_stride, float lambda, float lambda_ilm, int32_t eos, int32_t k,
                float* out_scores, int32_t* out_cols, int32_t* out_next, void* stream);
int launch_ctc_decode(const DevModel& m, const float* logits, int64_t row_stride, int64_t frame_stride, int32_t B,
                      int32_t T, const int32_t* lengths, int32_t* states, int32_t* prev, float lambda, int32_t blank,
                      int32_t* frames_out, int32_t* emit_out, int32_t* emit_len, void* stream);
int max_vocab_supported();
int max_fused_vocab();

}  // namespace ngpulm
