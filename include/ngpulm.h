/* ngpulm.h — C ABI of the B200-native NGPU-LM hot path (libngpulm.so).
 *
 * NGPU-LM (arXiv 2505.22857) stores a back-off n-gram LM as flat tensors and
 * answers batched full-vocabulary queries  state[B] -> (token_weights[B,V],
 * next_states[B,V])  (§2.2) with Algorithm 1
 * (PAPER.md:54-89), and fuses that query into greedy shallow-fusion decoding
 * for CTC, transducer and AED models (§2.3).
 *
 * Conventions for every call below:
 *  - All log-probabilities are natural-log float32 (ARPA log10 values are
 *    converted at load, R1). ARPA's -99 dummy becomes -1e30 (R3).
 *  - Token ids are 0..V-1 (vocabulary line index, or the decimal token itself
 *    when no vocabulary file is given). State ids are 0..S-1, root = 0, ids
 *    ordered by (context length, context token ids) with <s> = V (R6).
 *  - "dev" pointers are CUDA device memory on the model's device; that device
 *    must be the caller's current device. Hot-path calls (advance, final,
 *    fused_greedy_step) are asynchronous on `stream` (NULL = legacy default
 *    stream), never synchronize, never allocate and are CUDA-graph capturable.
 *  - Return codes: NGPULM_OK, or
 *      NGPULM_EDOMAIN  invalid ARPA / vocabulary content (message names the line),
 *      NGPULM_EUSAGE   bad arguments (NULL, negative sizes, bad mode/blank id,
 *                      wrong current device, V beyond the kernels' limit:
 *                      info.max_vocab for advance/final — vocabulary-tiled
 *                      rows — and info.max_fused_vocab for the fused step),
 *      NGPULM_ECUDA    a CUDA runtime error (message carries cudaGetErrorString),
 *      NGPULM_EIO      a file could not be read.
 *    ngpulm_last_error() returns a thread-local message for the last non-OK return.
 *  - Out-of-range state ids are reported asynchronously: the affected row gets
 *    NaN scores / -1 next states (advance), NaN (final) or token -1 and an
 *    unchanged state (fused step), and the first offending row index is kept
 *    in a sticky per-model device word read by ngpulm_check().
 *  - B = 0 is a no-op returning NGPULM_OK.
 *  - A model is immutable after load: concurrent calls on distinct streams are
 *    safe; outputs depend only on inputs.
 */
#ifndef NGPULM_H
#define NGPULM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ngpulm_model ngpulm_model;
typedef struct CUstream_st* ngpulm_stream; /* == cudaStream_t */

enum { NGPULM_OK = 0, NGPULM_EDOMAIN = 1, NGPULM_EUSAGE = 2, NGPULM_ECUDA = 3, NGPULM_EIO = 4 };
enum { NGPULM_CTC = 0, NGPULM_RNNT = 1, NGPULM_AED = 2 };
enum { NGPULM_MAX_ORDER = 32 };
enum { NGPULM_MAX_TOPK = 256 };
enum { NGPULM_MAX_DURATIONS = 32 }; /* TDT duration set size limit (ngpulm_tdt_loop_step) */
enum { NGPULM_CHAIN_TABLE = 0, NGPULM_CHAIN_WALK = 1 };
enum { NGPULM_ADVANCE_AUTO = 0, NGPULM_ADVANCE_WARP = 1, NGPULM_ADVANCE_CTA = 2 };

typedef struct {
  int32_t order;          /* N, highest n-gram order in the ARPA */
  int32_t vocab_size;     /* V */
  int32_t num_states;     /* S */
  int32_t root_state;     /* always 0: the empty context (unigram state) */
  int32_t bos_state;      /* state of "<s>", or root when absent (R4) */
  int32_t device;         /* CUDA device, or -1 for a host-only model */
  int64_t num_arcs;       /* incl. the V root arcs */
  int64_t num_unk_filled; /* M: vocabulary tokens without a unigram (R2) */
  int64_t num_dropped;    /* n-grams with <unk> beyond the unigram, dropped (R5) */
  int64_t device_bytes;   /* bytes of the resident model on the device */
  int32_t max_vocab;      /* largest V advance/final accept (rows beyond shared memory are tiled) */
  int32_t chain_mode;     /* NGPULM_CHAIN_TABLE or NGPULM_CHAIN_WALK */
  int32_t advance_kernel; /* NGPULM_ADVANCE_* as set (AUTO by default) */
  int32_t packed_arcs;    /* 1: the device also holds arcs packed as (target << bits) | token */
  int32_t max_fused_vocab;/* largest V of the fused step (its row must fit in shared memory) */
  int32_t tiny_resident;  /* 1: a tiny LM (<= 96 KiB of chain table + packed arcs): NGPULM_ADVANCE_AUTO
                             answers from a copy in every CTA's shared memory */
} ngpulm_info;

/* Read-only view of the model's host copy of the flat arrays.
 * Valid until ngpulm_free. Arcs are sorted by (from_state, token); state s owns
 * arcs [arc_offsets[s], arc_offsets[s+1]) (PAPER.md:122 start_arcs/end_arcs);
 * the root owns exactly arcs [0, V) with arc_tokens[v] = v. */
typedef struct {
  const int32_t* arc_tokens;     /* [num_arcs] */
  const float* arc_weights;      /* [num_arcs] */
  const int32_t* arc_to_states;  /* [num_arcs] */
  const int32_t* arc_offsets;    /* [num_states + 1] */
  const int32_t* boff_to_states; /* [num_states]; root -> root */
  const float* boff_weights;     /* [num_states]; root -> 0 */
  const float* final_weights;    /* [num_states] */
} ngpulm_host_view;

/* Parse an ARPA file (PAPER.md:94-96 line format), validate it, build the flat
 * trie on the host (sorted arcs, arc ranges, back-off targets and weights,
 * root filled to V arcs with the normalized <unk> weight, precomputed finals)
 * and upload it to `cuda_device` (-1: host only; hot-path calls then return
 * EUSAGE). `vocab_path`: one token per line, id = line index;
 * NULL: tokens are canonical decimal ids in [0, vocab_size). `vocab_size` may
 * be 0 with a vocabulary file. Synchronous. On success *out owns everything. */
int ngpulm_load_arpa(const char* arpa_path, const char* vocab_path, int32_t vocab_size,
                     int32_t cuda_device, ngpulm_model** out);

/* NGLM binary model files (format SPEC.md:209: "NGLM" magic,
 * u32 version = 1, u32 order, u32 vocab_size, u32 num_states, u64 num_arcs,
 * u32 root_state, u32 bos_state, then arc_tokens u32[A], arc_weights f32[A],
 * arc_to_states u32[A], start_arcs u64[S], end_arcs u64[S], boff_weights
 * f32[S], boff_to_states u32[S], final_weights f32[S], and a trailing CRC-32
 * (IEEE) of all preceding bytes; little-endian).
 * ngpulm_save writes the model's host arrays (synchronous; EIO on a write
 * failure). ngpulm_load_binary reads such a file and builds/uploads the model
 * exactly as ngpulm_load_arpa would from the ARPA it came from (arrays
 * bit-identical, hence bit-identical query results), without parsing text.
 * Errors: EIO (cannot read), EDOMAIN with a message naming the failure: "bad
 * magic", "unsupported version", "truncated header"/"truncated payload",
 * "checksum mismatch", or an inconsistent array. info.num_unk_filled is
 * recomputed from the root arcs for order >= 2 (else -1); info.num_dropped
 * is -1 (not stored). The vocabulary strings are not stored: token ids are
 * the file's ids. */
int ngpulm_save(const ngpulm_model* model, const char* path);
int ngpulm_load_binary(const char* path, int32_t cuda_device, ngpulm_model** out);

/* Copy an existing model's arrays to another device without re-parsing
 * (one replica per GPU for multi-GPU sharding). */
int ngpulm_replicate(const ngpulm_model* src, int32_t cuda_device, ngpulm_model** out);

void ngpulm_free(ngpulm_model* model);

/* How the kernels obtain a row's back-off levels (Algorithm 1 lines 72, 81-82):
 *   NGPULM_CHAIN_TABLE (default): from a per-state record built at load time
 *     (arc range and acc_boff of every level of the back-off chain, accumulated
 *     in Algorithm 1's order) — one dependent memory access instead of one per
 *     level; costs 16 * max(1, order) bytes per state of HBM.
 *   NGPULM_CHAIN_WALK: walk boff_to_states / boff_weights at query time, level
 *     by level, exactly as Algorithm 1 is written.
 * Both give bit-identical results. Not to be called concurrently with hot-path
 * calls on the same model (it changes what later launches read). */
int ngpulm_set_chain_mode(ngpulm_model* model, int32_t mode);

/* Which kernel ngpulm_advance runs; all give
 * bit-identical results:
 *   NGPULM_ADVANCE_AUTO (default): one warp per row, reading the arcs packed as
 *     (target << ceil(log2 V)) | token beside the weights when every target
 *     fits (info.packed_arcs), else as NGPULM_ADVANCE_WARP; a tiny LM
 *     (info.tiny_resident) is read from a copy in shared memory;
 *   NGPULM_ADVANCE_WARP: one warp per row over the token/weight/target arrays;
 *   NGPULM_ADVANCE_CTA: one 256-thread CTA per row.
 * The warp kernels need V % 4 == 0 and 16-byte aligned outputs; otherwise
 * (and always for CTA) the CTA kernel runs. Same concurrency rule as
 * ngpulm_set_chain_mode. EUSAGE for an unknown kind. */
int ngpulm_set_advance_kernel(ngpulm_model* model, int32_t kind);
int ngpulm_get_info(const ngpulm_model* model, ngpulm_info* out);
int ngpulm_host_view_get(const ngpulm_model* model, ngpulm_host_view* out);
const char* ngpulm_last_error(void);

/* Host helper: the state of the longest suffix of ("<s>" if with_bos) + tokens[0..n)
 * that is a state — the LM context a decoder holds after those tokens. */
int ngpulm_state_of(const ngpulm_model* model, int32_t with_bos, const int32_t* tokens,
                    int32_t n, int32_t* out_state);

/* Batched full-vocabulary query, Algorithm 1 for each row:
 *   scores[b*V + v] = log P(v | context(states[b]))  (float32; back-off
 *                     weights accumulated left to right, R10)
 *   next[b*V + v]   = state after emitting v (longest suffix of context+v that
 *                     is a state, R7)
 *   final_out[b]    = final weight of states[b], when non-NULL.
 * states: dev [B] int32. scores: dev [B,V] float32, next: dev [B,V] int32,
 * both row-major and caller-owned; final_out: dev [B] float32 or NULL.
 * The outputs must not overlap `states` (the kernel may read states[b] again
 * after other rows' outputs are written). Rows are built from the state read
 * before the kernel's programmatic-dependent-launch wait and re-checked after
 * it, so a preceding kernel on the stream may still be writing
 * `states` when this call starts: the result is always that of the final
 * states. */
int ngpulm_advance(const ngpulm_model* model, const int32_t* states, int32_t B, float* scores,
                   int32_t* next, float* final_out, ngpulm_stream stream);

/* ngpulm_advance with flags:
 *   NGPULM_ADVANCE_INDEPENDENT: the caller guarantees that no kernel which may
 *     still be running when this call's kernel starts writes `states` or reads
 *     or writes `scores`, `next`, `final_out` — e.g. consecutive calls over
 *     independent batches with distinct output buffers (batch rescoring of
 *     many state batches, PAPER.md:111-113's batched query issued back to
 *     back). Each row is then built AND stored before the kernel waits for its
 *     predecessor (programmatic dependent launch), so consecutive calls' 8 V B
 *     output bytes stream out back to back instead of each call waiting for
 *     the previous one to drain; the call still completes after its
 *     predecessor (stream completion order is kept). Results are identical.
 * flags == 0 is ngpulm_advance. EUSAGE for unknown flags. */
enum { NGPULM_ADVANCE_INDEPENDENT = 1 };
int ngpulm_advance_ex(const ngpulm_model* model, const int32_t* states, int32_t B, float* scores,
                      int32_t* next, float* final_out, uint32_t flags, ngpulm_stream stream);

/* final_out[b] = final weight of states[b] (the AED <eos> score).
 * states: dev [B] int32; final_out: dev [B] float32. */
int ngpulm_final(const ngpulm_model* model, const int32_t* states, int32_t B, float* final_out,
                 ngpulm_stream stream);

/* One greedy shallow-fusion step for B rows, with the LM
 * row of each state computed on chip and never written to memory.
 *   logits:  dev float32; row b is logits + b*row_stride, V+1 columns: the V
 *            tokens and the special column `blank_id` (blank for CTC/RNN-T,
 *            <eos> for AED); token v sits in column v (v < blank_id) or v+1 (R19).
 *   states:  dev [B] int32, in/out LM states.
 *   prev:    dev [B] int32, in/out, CTC only (else ignored, may be NULL): column
 *            selected at the previous frame, -1 = none/blank (R17).
 *   active:  dev [B] uint8 or NULL (= all rows); inactive rows are untouched
 *            and get tokens_out = -1.
 *   tokens_out: dev [B] int32: the selected column.
 * Decision rules (fused value = fmaf(lambda, lm, asr), single rounding, R13;
 * argmax ties -> lowest column, R14):
 *   NGPULM_RNNT two-stage: raw argmax over all columns; blank -> keep it (state
 *               unchanged); else argmax of fused values over non-blank columns,
 *               state <- next.
 *   NGPULM_CTC  blank and prev columns raw, all others fused; argmax; blank ->
 *               prev = -1; == prev -> no LM advance; else state <- next,
 *               prev <- column.
 *   NGPULM_AED  token columns fused, the <eos> column fmaf(lambda, final(state),
 *               asr[eos]); eos -> state unchanged; else state <- next.
 * states == NULL (with lambda == 0, else EUSAGE): plain greedy decoding without
 * an LM, the same kernel with no LM row — the baseline of the paper's overhead
 * figure; decisions are those of lambda = 0.
 */
int ngpulm_fused_greedy_step(const ngpulm_model* model, int32_t mode, const float* logits,
                             int64_t row_stride, int32_t B, int32_t* states, int32_t* prev,
                             const uint8_t* active, float lambda, int32_t blank_id,
                             int32_t* tokens_out, ngpulm_stream stream);

/* ngpulm_fused_greedy_step with flags:
 *   NGPULM_STEP_LOGITS_READY: the caller guarantees that no kernel which may
 *     still be running when this call's kernel starts writes `logits` — e.g.
 *     a CTC loop over an encoder output produced before the loop (the kernel
 *     then copies its logits rows before its programmatic-dependent-launch
 *     wait, overlapping the previous step; PAPER.md:139's per-frame loop).
 *     NGPU-LM calls never write logits, so a loop of NGPU-LM steps over
 *     precomputed logits always qualifies; a logits producer launched with
 *     programmatic dependent launch that triggers early does not.
 *   NGPULM_STEP_INPUTS_READY: the caller guarantees that no kernel which may
 *     still be running when this call's kernel starts writes ANY of its
 *     inputs (logits, states, prev, active) — e.g. a transducer / AED loop
 *     whose network kernel before each step is a plain launch (not a
 *     programmatic dependent launch: every cuBLAS / PyTorch kernel), so the
 *     step starts only after it has completed. The kernel then copies the
 *     logits and builds the LM row from the state it reads at its start,
 *     without re-reading the state after its programmatic-dependent-launch
 *     wait. Results are identical to flags == 0 whenever the guarantee holds;
 *     consecutive NGPU-LM steps (which write states) do not qualify.
 *     Ignored by the ILM variant, by models held in shared memory (tiny-LM
 *     path) and by models without packed arcs and a chain table (they run
 *     their flags == 0 kernels; results are the same).
 * flags == 0 is ngpulm_fused_greedy_step. EUSAGE for unknown flags. */
enum { NGPULM_STEP_LOGITS_READY = 1, NGPULM_STEP_INPUTS_READY = 2 };
int ngpulm_fused_greedy_step_ex(const ngpulm_model* model, int32_t mode, const float* logits,
                                int64_t row_stride, int32_t B, int32_t* states, int32_t* prev,
                                const uint8_t* active, float lambda, int32_t blank_id, int32_t* tokens_out,
                                uint32_t flags, ngpulm_stream stream);

/* ngpulm_fused_greedy_step with internal-LM subtraction ("-ILM+LM" for HAT
 * transducers, Table 3; SPEC.md:298-306 fuse_scores): every
 * LM-rescored column (CTC: not blank, not prev; RNN-T stage 2: non-blank;
 * AED: token columns — the eos column takes no ILM term) gets
 *     fmaf(-lambda_ilm, ilm[b*ilm_stride + v], fmaf(lambda, lm, asr))
 * (two single roundings in this order, R21; lambda_ilm = 0 gives
 * exactly the plain fused step's decisions). ilm: dev float32, row b at
 * ilm + b*ilm_stride, indexed by LM token v in [0, V) (not by column). All
 * other arguments and rules as ngpulm_fused_greedy_step. */
int ngpulm_fused_greedy_step_ilm(const ngpulm_model* model, int32_t mode, const float* logits,
                                 int64_t row_stride, int32_t B, int32_t* states, int32_t* prev,
                                 const uint8_t* active, float lambda, int32_t blank_id, const float* ilm,
                                 int64_t ilm_stride, float lambda_ilm, int32_t* tokens_out,
                                 ngpulm_stream stream);

/* One iteration of batched label-looping greedy transducer decoding with
 * fusion. Each row
 * carries a loop state (frame_idx, sym_count, emit_len, last_token); the
 * caller's joint network produces row b's logits for (frame_idx[b],
 * u = emit_len[b], last_token[b]) before each call. A row is active while
 * frame_idx[b] < lengths[b]; for an active row the call makes the RNN-T
 * two-stage decision of ngpulm_fused_greedy_step (with the ILM term when ilm
 * != NULL, as ngpulm_fused_greedy_step_ilm), then:
 *   blank        -> frame_idx += 1, sym_count = 0;
 *   a label (col)-> emit_out[b*max_len + emit_len[b]] = col (if emit_len[b] <
 *                   max_len), emit_len += 1, last_token = its LM token,
 *                   states[b] = next state, sym_count += 1, and when sym_count
 *                   reaches max_symbols: frame_idx += 1, sym_count = 0.
 * tokens_out[b] = the selected column (-1 for inactive rows). Iterating until
 * no row is active reproduces, row by row, the frame-by-frame greedy loop
 * with at most max_symbols labels per frame. An invalid state sets the
 * bad-row word and ends the row (frame_idx = lengths[b]); an all-NaN logits
 * row counts as blank. All buffers dev int32 [B] except emit_out [B, max_len]
 * and logits (row stride row_stride, V+1 columns, R19); last_token may be
 * NULL. states == NULL (lambda == 0, no ILM): plain greedy label looping
 * without an LM. Needs V % 4 == 0 and V <= 1024. Graph-capturable. */
int ngpulm_transducer_loop_step(const ngpulm_model* model, const float* logits, int64_t row_stride,
                                int32_t B, int32_t* states, int32_t* frame_idx, int32_t* sym_count,
                                const int32_t* lengths, int32_t max_symbols, float lambda,
                                int32_t blank_id, const float* ilm, int64_t ilm_stride, float lambda_ilm,
                                int32_t* tokens_out, int32_t* emit_out, int32_t* emit_len,
                                int32_t* last_token, int32_t max_len, ngpulm_stream stream);

/* One iteration of label-looping greedy Token-and-Duration Transducer (TDT)
 * decoding with fusion (NGPU-LM in the TDT label-looping decoder;
 * DESIGN.md R25). As ngpulm_transducer_loop_step, with D duration logits per
 * row at dur_logits + b*dur_stride (dev float32; typically the joint row's
 * columns V+1 .. V+D), and `durations` (HOST int32 [num_durations], each >= 0,
 * 1 <= num_durations <= NGPULM_MAX_DURATIONS; copied into the launch, so a
 * captured graph keeps the values of capture time): the token is the RNN-T
 * two-stage fused decision; the duration d = durations[j], j = the raw argmax
 * of the duration logits (lowest index on ties; the LM does not touch them);
 * blank -> frame_idx += max(d, 1), sym_count = 0; a label -> emitted and LM
 * advanced as for RNN-T, then d > 0 -> frame_idx += d, sym_count = 0, and
 * d == 0 -> the frame is kept, sym_count += 1, and at max_symbols the frame
 * advances by 1. durations = {1} gives the RNN-T loop with max_symbols = 1,
 * durations = {0} the RNN-T loop with max_symbols. */
int ngpulm_tdt_loop_step(const ngpulm_model* model, const float* logits, int64_t row_stride,
                         const float* dur_logits, int64_t dur_stride, const int32_t* durations,
                         int32_t num_durations, int32_t B, int32_t* states, int32_t* frame_idx,
                         int32_t* sym_count, const int32_t* lengths, int32_t max_symbols, float lambda,
                         int32_t blank_id, const float* ilm, int64_t ilm_stride, float lambda_ilm,
                         int32_t* tokens_out, int32_t* emit_out, int32_t* emit_len, int32_t* last_token,
                         int32_t max_len, ngpulm_stream stream);

/* ngpulm_transducer_loop_step / ngpulm_tdt_loop_step with flags:
 *   NGPULM_STEP_INPUTS_READY: as for ngpulm_fused_greedy_step_ex — no kernel
 *     which may still be running when this call's kernel starts writes any of
 *     its inputs (logits, duration logits, states, frame_idx, sym_count,
 *     lengths, last_token), e.g. a label-looping decoder whose joint kernel
 *     before each step is a plain launch. The step then copies the logits and
 *     builds the LM row from the state read at its start (no re-read after its
 *     programmatic-dependent-launch wait). Results are identical to flags == 0
 *     whenever the guarantee holds. Ignored with an ILM, for models held in
 *     shared memory (tiny-LM path) and for models without packed arcs and a
 *     chain table.
 * flags == 0 are the calls above. EUSAGE for unknown flags. */
int ngpulm_transducer_loop_step_ex(const ngpulm_model* model, const float* logits, int64_t row_stride,
                                   int32_t B, int32_t* states, int32_t* frame_idx, int32_t* sym_count,
                                   const int32_t* lengths, int32_t max_symbols, float lambda,
                                   int32_t blank_id, const float* ilm, int64_t ilm_stride, float lambda_ilm,
                                   int32_t* tokens_out, int32_t* emit_out, int32_t* emit_len,
                                   int32_t* last_token, int32_t max_len, uint32_t flags, ngpulm_stream stream);
int ngpulm_tdt_loop_step_ex(const ngpulm_model* model, const float* logits, int64_t row_stride,
                            const float* dur_logits, int64_t dur_stride, const int32_t* durations,
                            int32_t num_durations, int32_t B, int32_t* states, int32_t* frame_idx,
                            int32_t* sym_count, const int32_t* lengths, int32_t max_symbols, float lambda,
                            int32_t blank_id, const float* ilm, int64_t ilm_stride, float lambda_ilm,
                            int32_t* tokens_out, int32_t* emit_out, int32_t* emit_len, int32_t* last_token,
                            int32_t max_len, uint32_t flags, ngpulm_stream stream);

/* The fused greedy step of ngpulm_fused_greedy_step (same modes, rules and
 * outputs) from LM rows computed beforehand by ngpulm_advance on the SAME
 * states: lm_scores/lm_next dev [B, *] (row b at b*lm_stride, V entries),
 * lm_final dev [B] (AED only, else may be NULL). Overlap mode:
 * in a decode loop the LM query of a step depends only on the states left by
 * the previous step, so the caller runs ngpulm_advance on a second stream while
 * its network computes the step's logits, and this call then only reads the
 * two rows and decides; the LM's cost leaves the loop's critical path. A row
 * whose LM row carries the advance's invalid-state mark (next = -1) gets
 * tokens_out = -1 and is untouched. Needs V <= 1024. */
int ngpulm_fused_greedy_step_rows(const ngpulm_model* model, int32_t mode, const float* logits,
                                  int64_t row_stride, int32_t B, const float* lm_scores,
                                  const int32_t* lm_next, const float* lm_final, int64_t lm_stride,
                                  int32_t* states, int32_t* prev, const uint8_t* active, float lambda,
                                  int32_t blank_id, int32_t* tokens_out, ngpulm_stream stream);

/* The k best fused expansions of each row, for AED beam search with NGPU-LM
 * shallow fusion. Fused value of a
 * token column: fmaf(lambda, lm, asr) [then fmaf(-lambda_ilm, ilm[v], .) when
 * ilm != NULL]; of the eos column `eos_id`: fmaf(lambda, final(state), asr).
 *   logits:      dev float32, row b at logits + b*row_stride, V+1 columns (R19).
 *   states:      dev [B] int32 (read only).
 *   ilm:         dev float32 or NULL, row b at ilm + b*ilm_stride, V token entries.
 *   topk_scores: dev [B,k] float32: the k largest fused values, descending
 *                (ties: lower column first, R14; NaN never selected; slots
 *                past the selectable columns: -inf with column -1).
 *   topk_cols:   dev [B,k] int32: their columns.
 *   topk_next:   dev [B,k] int32 or NULL: the LM state after each candidate
 *                (the state itself for eos, -1 for an empty slot).
 * 1 <= k <= NGPULM_MAX_TOPK; needs V % 4 == 0 and V <= 1024 (EUSAGE
 * otherwise). Invalid states: NaN scores, columns -1, bad-row word set. */
int ngpulm_fused_topk(const ngpulm_model* model, const float* logits, int64_t row_stride, int32_t B,
                      const int32_t* states, const float* ilm, int64_t ilm_stride, float lambda,
                      float lambda_ilm, int32_t eos_id, int32_t k, float* topk_scores,
                      int32_t* topk_cols, int32_t* topk_next, ngpulm_stream stream);

/* Whole-utterance greedy CTC decoding with shallow fusion in ONE launch
 * (the CTC rule of PAPER.md:138-139). The result is
 * identical to T calls of ngpulm_fused_greedy_step(NGPULM_CTC) for
 * t = 0..T-1 with active[b] = (t < lengths[b]): the LM row of a state is
 * computed on chip only when an emission changes the state and is reused
 * across the frames in between.
 *   logits:     dev float32; frame t of row b starts at
 *               logits + b*row_stride + t*frame_stride and has V+1 columns
 *               (column layout as for the fused step, R19). A [B,T,V+1]
 *               contiguous tensor has row_stride = T*(V+1), frame_stride = V+1.
 *   lengths:    dev [B] int32 (frames of each row, clamped to [0,T]) or NULL (= T).
 *   states:     dev [B] int32 in/out: LM state before frame 0 / after the last frame.
 *   prev:       dev [B] int32 in/out: column selected at the frame before
 *               frame 0 (-1 = none), and at the row's last frame (R17).
 *   frames_out: dev [B,T] int32 (row stride T) or NULL: the column selected at
 *               each frame, -1 at t >= lengths[b] (and for invalid states).
 *   emit_out:   dev [B,T] int32 (row stride T) or NULL: the emitted columns of
 *               row b (selections that are neither blank nor prev), in order,
 *               in emit_out[b*T .. b*T + emit_len[b]).
 *   emit_len:   dev [B] int32 or NULL: number of emissions of each row.
 * Needs V % 4 == 0, V <= 1024 and a finite lambda (EUSAGE otherwise); row_stride/frame_stride
 * must be multiples of 1 float (any alignment). Asynchronous, no allocation,
 * CUDA-graph capturable. An invalid start state sets the bad-row word and the
 * row decides nothing (frames -1, no emissions, state and prev unchanged).
 * states == NULL (lambda == 0): plain greedy CTC decoding without an LM. */
int ngpulm_ctc_greedy_decode(const ngpulm_model* model, const float* logits, int64_t row_stride,
                             int64_t frame_stride, int32_t B, int32_t T, const int32_t* lengths,
                             int32_t* states, int32_t* prev, float lambda, int32_t blank_id,
                             int32_t* frames_out, int32_t* emit_out, int32_t* emit_len,
                             ngpulm_stream stream);

/* Synchronizes `stream`, reads and clears the sticky bad-row word:
 * *first_bad_row = smallest row index that carried an invalid state since the
 * last check, or -1. */
int ngpulm_check(const ngpulm_model* model, ngpulm_stream stream, int64_t* first_bad_row);

/* End-to-end convenience for callers holding HOST buffers (ideally pinned):
 * copies states_host [B] in, runs ngpulm_advance on model-owned device
 * scratch, copies scores_host [B,V], next_host [B,V] and final_host [B] (may
 * be NULL) back, and synchronizes `stream`. Allocates scratch on first use. */
int ngpulm_advance_host(ngpulm_model* model, const int32_t* states_host, int32_t B,
                        float* scores_host, int32_t* next_host, float* final_host,
                        ngpulm_stream stream);

/* Measurement support (host only): unique model bytes a call on this batch
 * must read — state records and arc ranges of every distinct state on the
 * rows' back-off chains, the V root arcs once, and the finals. */
int ngpulm_touched_bytes(const ngpulm_model* model, const int32_t* states_host, int32_t B,
                         int64_t* out_bytes);

#ifdef __cplusplus
}
#endif
#endif /* NGPULM_H */
