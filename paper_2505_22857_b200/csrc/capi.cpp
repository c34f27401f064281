// C ABI of libngpulm (include/ngpulm.h): argument checks, model residency in
// HBM, launches. No host synchronization or allocation on the hot-path calls.
#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <unordered_set>
#include <vector>

#include "ngpulm_internal.h"

struct ngpulm_model {
  ngpulm::HostModel h;
  int32_t device = -1;
  void* blob = nullptr;
  size_t blob_bytes = 0;
  ngpulm::DevModel dm{};
  const void* chain_dev = nullptr;  // chain table inside blob
  int32_t chain_mode = NGPULM_CHAIN_TABLE;
  void* scratch = nullptr;  // ngpulm_advance_host only
  size_t scratch_bytes = 0;
  std::mutex mu;
};

namespace {

thread_local std::string g_err;

int err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_err(cudaError_t e, const char* what) {
  return err(NGPULM_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct DeviceGuard {  // restores the caller's current device
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (dev >= 0 && dev != prev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// One allocation holds the whole resident model.
int upload(ngpulm_model* m, int device) {
  const ngpulm::HostModel& h = m->h;
  const size_t S = (size_t)h.num_states;
  std::vector<int32_t> dbeg;
  const size_t A = ngpulm::device_arc_layout(h, dbeg);  // padded arc count
  const bool pack = ngpulm::packable(h);
  const int32_t pk_bits = ngpulm::packed_token_bits(h.V);
  if (A > (size_t)INT32_MAX) return err(NGPULM_EUSAGE, "too many arcs for 32-bit arc indices");
  const size_t o_srec = 0;
  const size_t o_fin = align256(o_srec + S * sizeof(ngpulm::StateRec));
  const size_t o_tok = align256(o_fin + S * 4);
  const size_t o_w = align256(o_tok + A * 4);
  const size_t o_to = align256(o_w + A * 4);
  std::vector<int32_t> chain;
  int32_t slots = 1;
  ngpulm::build_chain_table(h, dbeg, chain, slots);
  const size_t o_q = align256(o_to + A * 4);
  const size_t o_chain = align256(o_q + (pack ? A * 8 : 0));
  std::vector<float> lm_ub;
  ngpulm::build_row_bounds(h, lm_ub);
  const size_t o_hi = align256(o_chain + chain.size() * 4);
  const size_t o_bad = align256(o_hi + S * 4);
  const size_t total = align256(o_bad + 8);
  std::vector<unsigned char> stage(total, 0);
  auto* rec = reinterpret_cast<ngpulm::StateRec*>(stage.data() + o_srec);
  auto* tok = reinterpret_cast<int32_t*>(stage.data() + o_tok);
  auto* wt = reinterpret_cast<float*>(stage.data() + o_w);
  auto* to = reinterpret_cast<int32_t*>(stage.data() + o_to);
  auto* aq = reinterpret_cast<uint32_t*>(stage.data() + o_q);  // [A/4][8]
  for (size_t s = 0; s < S; ++s) {
    const int32_t b = h.arc_off[s], cnt = h.arc_off[s + 1] - b;
    rec[s] = {dbeg[s], dbeg[s] + cnt, h.boff_to[s], h.boff_w[s]};
    const int32_t end = s + 1 < S ? dbeg[s + 1] : (int32_t)A;
    for (int32_t j = 0; j < end - dbeg[s]; ++j) {  // the padding repeats the last arc
      const int32_t src = b + std::min(j, cnt - 1);
      tok[dbeg[s] + j] = h.arc_tok[src];
      wt[dbeg[s] + j] = h.arc_w[src];
      to[dbeg[s] + j] = h.arc_to[src];
      if (pack) {
        const size_t a = (size_t)dbeg[s] + j, unit = a / 4, k = a % 4;
        aq[unit * 8 + k] = ((uint32_t)h.arc_to[src] << pk_bits) | (uint32_t)h.arc_tok[src];
        std::memcpy(&aq[unit * 8 + 4 + k], &h.arc_w[src], 4);
      }
    }
  }
  std::memcpy(stage.data() + o_fin, h.final_w.data(), S * 4);
  std::memcpy(stage.data() + o_chain, chain.data(), chain.size() * 4);
  std::memcpy(stage.data() + o_hi, lm_ub.data(), S * 4);
  std::memset(stage.data() + o_bad, 0xff, 8);

  DeviceGuard g(device);
  void* d = nullptr;
  cudaError_t e = cudaMalloc(&d, total);
  if (e != cudaSuccess) return cuda_err(e, "cudaMalloc(model)");
  e = cudaMemcpy(d, stage.data(), total, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { cudaFree(d); return cuda_err(e, "cudaMemcpy(model)"); }
  auto* base = static_cast<unsigned char*>(d);
  m->blob = d;
  m->blob_bytes = total;
  m->device = device;
  m->dm.srec = reinterpret_cast<const ngpulm::StateRec*>(base + o_srec);
  m->dm.final_w = reinterpret_cast<const float*>(base + o_fin);
  m->dm.arc_tok = reinterpret_cast<const int32_t*>(base + o_tok);
  m->dm.arc_w = reinterpret_cast<const float*>(base + o_w);
  m->dm.arc_to = reinterpret_cast<const int32_t*>(base + o_to);
  m->dm.bad_row = reinterpret_cast<unsigned long long*>(base + o_bad);
  m->chain_dev = base + o_chain;
  m->dm.chain = m->chain_mode == NGPULM_CHAIN_TABLE ? m->chain_dev : nullptr;
  m->dm.chain_slots = slots;
  m->dm.S = h.num_states;
  m->dm.V = h.V;
  m->dm.order = h.order;
  m->dm.arc_q = pack ? static_cast<const void*>(base + o_q) : nullptr;
  m->dm.pk_bits = pk_bits;
  m->dm.adv_kind = NGPULM_ADVANCE_AUTO;
  m->dm.lm_ub = reinterpret_cast<const float*>(base + o_hi);
  // tiny LM (keyword-biasing size): chain table + packed quads <= 96 KiB stay in shared memory
  const size_t chain_bytes = chain.size() * 4, arcq_bytes = pack ? A * 8 : 0;
  const bool tiny = pack && h.V <= 1024 && h.V % 4 == 0 && chain_bytes + arcq_bytes <= ((size_t)96 << 10);
  m->dm.tiny_chain_bytes = tiny ? (int32_t)chain_bytes : 0;
  m->dm.tiny_arcq_bytes = tiny ? (int32_t)arcq_bytes : 0;
  return NGPULM_OK;
}

int check_hot(const ngpulm_model* m, int32_t B) {
  if (!m) return err(NGPULM_EUSAGE, "model is NULL");
  if (m->device < 0) return err(NGPULM_EUSAGE, "host-only model (loaded with cuda_device = -1)");
  if (B < 0) return err(NGPULM_EUSAGE, "B < 0");
  if (m->h.V > ngpulm::max_vocab_supported()) return err(NGPULM_EUSAGE, "vocabulary larger than supported");
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != m->device) return err(NGPULM_EUSAGE, "current CUDA device differs from the model's device");
  return NGPULM_OK;
}

}  // namespace

extern "C" {

const char* ngpulm_last_error(void) { return g_err.c_str(); }

int ngpulm_load_arpa(const char* arpa_path, const char* vocab_path, int32_t vocab_size, int32_t cuda_device,
                     ngpulm_model** out) {
  if (!arpa_path || !out) return err(NGPULM_EUSAGE, "NULL argument");
  *out = nullptr;
  std::unique_ptr<ngpulm_model> m(new (std::nothrow) ngpulm_model());
  if (!m) return err(NGPULM_EUSAGE, "out of host memory");
  std::string e;
  int r = ngpulm::build_from_arpa(arpa_path, vocab_path, vocab_size, m->h, e);
  if (r != NGPULM_OK) return err(r, e);
  if (cuda_device >= 0) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || cuda_device >= n)
      return err(NGPULM_EUSAGE, "no such CUDA device");
    r = upload(m.get(), cuda_device);
    if (r != NGPULM_OK) return r;
  }
  *out = m.release();
  return NGPULM_OK;
}

int ngpulm_save(const ngpulm_model* m, const char* path) {
  if (!m || !path) return err(NGPULM_EUSAGE, "NULL argument");
  std::string e;
  int r = ngpulm::save_binary(m->h, path, e);
  return r == NGPULM_OK ? r : err(r, e);
}

int ngpulm_load_binary(const char* path, int32_t cuda_device, ngpulm_model** out) {
  if (!path || !out) return err(NGPULM_EUSAGE, "NULL argument");
  *out = nullptr;
  std::unique_ptr<ngpulm_model> m(new (std::nothrow) ngpulm_model());
  if (!m) return err(NGPULM_EUSAGE, "out of host memory");
  std::string e;
  int r = ngpulm::load_binary(path, m->h, e);
  if (r != NGPULM_OK) return err(r, e);
  if (cuda_device >= 0) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || cuda_device >= n) return err(NGPULM_EUSAGE, "no such CUDA device");
    r = upload(m.get(), cuda_device);
    if (r != NGPULM_OK) return r;
  }
  *out = m.release();
  return NGPULM_OK;
}

int ngpulm_replicate(const ngpulm_model* src, int32_t cuda_device, ngpulm_model** out) {
  if (!src || !out || cuda_device < 0) return err(NGPULM_EUSAGE, "bad argument");
  *out = nullptr;
  std::unique_ptr<ngpulm_model> m(new (std::nothrow) ngpulm_model());
  if (!m) return err(NGPULM_EUSAGE, "out of host memory");
  m->h = src->h;
  int r = upload(m.get(), cuda_device);
  if (r != NGPULM_OK) return r;
  *out = m.release();
  return NGPULM_OK;
}

void ngpulm_free(ngpulm_model* m) {
  if (!m) return;
  if (m->blob || m->scratch) {
    DeviceGuard g(m->device);
    if (m->blob) cudaFree(m->blob);
    if (m->scratch) cudaFree(m->scratch);
  }
  delete m;
}

int ngpulm_set_advance_kernel(ngpulm_model* m, int32_t kind) {
  if (!m) return err(NGPULM_EUSAGE, "model is NULL");
  if (kind != NGPULM_ADVANCE_AUTO && kind != NGPULM_ADVANCE_WARP && kind != NGPULM_ADVANCE_CTA)
    return err(NGPULM_EUSAGE, "bad advance kernel kind");
  m->dm.adv_kind = kind;
  return NGPULM_OK;
}

int ngpulm_set_chain_mode(ngpulm_model* m, int32_t mode) {
  if (!m) return err(NGPULM_EUSAGE, "model is NULL");
  if (mode != NGPULM_CHAIN_TABLE && mode != NGPULM_CHAIN_WALK) return err(NGPULM_EUSAGE, "bad chain mode");
  m->chain_mode = mode;
  m->dm.chain = mode == NGPULM_CHAIN_TABLE ? m->chain_dev : nullptr;
  return NGPULM_OK;
}

int ngpulm_get_info(const ngpulm_model* m, ngpulm_info* out) {
  if (!m || !out) return err(NGPULM_EUSAGE, "NULL argument");
  std::memset(out, 0, sizeof *out);
  out->order = m->h.order;
  out->vocab_size = m->h.V;
  out->num_states = m->h.num_states;
  out->root_state = 0;
  out->bos_state = m->h.bos_state;
  out->device = m->device;
  out->num_arcs = (int64_t)m->h.arc_tok.size();
  out->num_unk_filled = m->h.num_unk_filled;
  out->num_dropped = m->h.num_dropped;
  out->device_bytes = (int64_t)m->blob_bytes;
  out->max_vocab = ngpulm::max_vocab_supported();
  out->max_fused_vocab = ngpulm::max_fused_vocab();
  out->tiny_resident = m->dm.tiny_chain_bytes > 0;
  out->chain_mode = m->chain_mode;
  out->advance_kernel = m->dm.adv_kind;
  out->packed_arcs = m->dm.arc_q != nullptr;
  return NGPULM_OK;
}

int ngpulm_host_view_get(const ngpulm_model* m, ngpulm_host_view* out) {
  if (!m || !out) return err(NGPULM_EUSAGE, "NULL argument");
  out->arc_tokens = m->h.arc_tok.data();
  out->arc_weights = m->h.arc_w.data();
  out->arc_to_states = m->h.arc_to.data();
  out->arc_offsets = m->h.arc_off.data();
  out->boff_to_states = m->h.boff_to.data();
  out->boff_weights = m->h.boff_w.data();
  out->final_weights = m->h.final_w.data();
  return NGPULM_OK;
}

int ngpulm_state_of(const ngpulm_model* m, int32_t with_bos, const int32_t* tokens, int32_t n,
                    int32_t* out_state) {
  if (!m || !out_state || n < 0 || (n > 0 && !tokens)) return err(NGPULM_EUSAGE, "bad argument");
  std::vector<int32_t> hist;
  if (with_bos) hist.push_back(m->h.V);  // <s>
  for (int32_t i = 0; i < n; ++i) {
    if (tokens[i] < 0 || tokens[i] >= m->h.V) return err(NGPULM_EUSAGE, "token out of range");
    hist.push_back(tokens[i]);
  }
  // longest suffix that is a state: follow prefix edges from the root
  const size_t L = hist.size();
  const size_t first = L > (size_t)m->h.order ? L - (size_t)m->h.order : 0;
  for (size_t j = first; j <= L; ++j) {
    int32_t s = 0;
    size_t i = j;
    for (; i < L; ++i) {
      s = m->h.child(s, hist[i]);
      if (s < 0) break;
    }
    if (i == L) { *out_state = s; return NGPULM_OK; }
  }
  *out_state = 0;
  return NGPULM_OK;
}

int ngpulm_advance(const ngpulm_model* m, const int32_t* states, int32_t B, float* scores, int32_t* next,
                   float* final_out, ngpulm_stream stream) {
  return ngpulm_advance_ex(m, states, B, scores, next, final_out, 0u, stream);
}

int ngpulm_advance_ex(const ngpulm_model* m, const int32_t* states, int32_t B, float* scores, int32_t* next,
                      float* final_out, uint32_t flags, ngpulm_stream stream) {
  if (int r = check_hot(m, B)) return r;
  if (flags & ~(uint32_t)NGPULM_ADVANCE_INDEPENDENT) return err(NGPULM_EUSAGE, "unknown flags");
  if (B == 0) return NGPULM_OK;
  if (!states || !scores || !next) return err(NGPULM_EUSAGE, "NULL device buffer");
  {  // the outputs must not overlap the states (rows re-read their state after others are written)
    auto overlap = [](const void* a, size_t na, const void* b, size_t nb) {
      const uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
      return x < y + nb && y < x + na;
    };
    const size_t sb = (size_t)B * 4, ob = (size_t)B * m->h.V * 4;
    if (overlap(states, sb, scores, ob) || overlap(states, sb, next, ob) || (final_out && overlap(states, sb, final_out, sb)))
      return err(NGPULM_EUSAGE, "advance outputs overlap the states");
  }
  int e = ngpulm::launch_advance(m->dm, states, B, scores, next, final_out, stream, flags);
  if (e) return cuda_err((cudaError_t)e, "advance launch");
  return NGPULM_OK;
}

int ngpulm_final(const ngpulm_model* m, const int32_t* states, int32_t B, float* final_out,
                 ngpulm_stream stream) {
  if (int r = check_hot(m, B)) return r;
  if (B == 0) return NGPULM_OK;
  if (!states || !final_out) return err(NGPULM_EUSAGE, "NULL device buffer");
  int e = ngpulm::launch_final(m->dm, states, B, final_out, stream);
  if (e) return cuda_err((cudaError_t)e, "final launch");
  return NGPULM_OK;
}

int ngpulm_fused_greedy_step(const ngpulm_model* m, int32_t mode, const float* logits, int64_t row_stride,
                             int32_t B, int32_t* states, int32_t* prev, const uint8_t* active, float lambda,
                             int32_t blank_id, int32_t* tokens_out, ngpulm_stream stream) {
  return ngpulm_fused_greedy_step_ex(m, mode, logits, row_stride, B, states, prev, active, lambda, blank_id,
                                     tokens_out, 0u, stream);
}

int ngpulm_fused_greedy_step_ex(const ngpulm_model* m, int32_t mode, const float* logits, int64_t row_stride,
                                int32_t B, int32_t* states, int32_t* prev, const uint8_t* active, float lambda,
                                int32_t blank_id, int32_t* tokens_out, uint32_t flags, ngpulm_stream stream) {
  if (int r = check_hot(m, B)) return r;
  if (flags & ~(uint32_t)(NGPULM_STEP_LOGITS_READY | NGPULM_STEP_INPUTS_READY)) return err(NGPULM_EUSAGE, "unknown flags");
  if (mode != NGPULM_CTC && mode != NGPULM_RNNT && mode != NGPULM_AED) return err(NGPULM_EUSAGE, "bad mode");
  if (blank_id < 0 || blank_id > m->h.V) return err(NGPULM_EUSAGE, "blank_id outside [0, V]");
  if (m->h.V > ngpulm::max_fused_vocab()) return err(NGPULM_EUSAGE, "fused step: the row must fit in shared memory");
  if (B == 0) return NGPULM_OK;
  if (!states && lambda != 0.f) return err(NGPULM_EUSAGE, "states NULL (plain greedy, no LM) needs lambda == 0");
  if (!logits || !tokens_out || (mode == NGPULM_CTC && !prev))
    return err(NGPULM_EUSAGE, "NULL device buffer");
  if (B > 1 && row_stride < (int64_t)m->h.V + 1) return err(NGPULM_EUSAGE, "row_stride < V+1");
  int e = ngpulm::launch_fused(m->dm, mode, logits, row_stride, B, states, prev, active, lambda, blank_id, nullptr,
                               0, 0.f, tokens_out, stream, flags);
  if (e) return cuda_err((cudaError_t)e, "fused step launch");
  return NGPULM_OK;
}

int ngpulm_fused_greedy_step_ilm(const ngpulm_model* m, int32_t mode, const float* logits, int64_t row_stride,
                                 int32_t B, int32_t* states, int32_t* prev, const uint8_t* active, float lambda,
                                 int32_t blank_id, const float* ilm, int64_t ilm_stride, float lambda_ilm,
                                 int32_t* tokens_out, ngpulm_stream stream) {
  if (int r = check_hot(m, B)) return r;
  if (mode != NGPULM_CTC && mode != NGPULM_RNNT && mode != NGPULM_AED) return err(NGPULM_EUSAGE, "bad mode");
  if (blank_id < 0 || blank_id > m->h.V) return err(NGPULM_EUSAGE, "blank_id outside [0, V]");
  if (m->h.V > ngpulm::max_fused_vocab()) return err(NGPULM_EUSAGE, "fused step: the row must fit in shared memory");
  if (B == 0) return NGPULM_OK;
  if (!logits || !states || !tokens_out || !ilm || (mode == NGPULM_CTC && !prev))
    return err(NGPULM_EUSAGE, "NULL device buffer");
  if (B > 1 && row_stride < (int64_t)m->h.V + 1) return err(NGPULM_EUSAGE, "row_stride < V+1");
  if (B > 1 && ilm_stride < (int64_t)m->h.V) return err(NGPULM_EUSAGE, "ilm_stride < V");
  int e = ngpulm::launch_fused(m->dm, mode, logits, row_stride, B, states, prev, active, lambda, blank_id, ilm,
                               ilm_stride, lambda_ilm, tokens_out, stream);
  if (e) return cuda_err((cudaError_t)e, "fused step launch");
  return NGPULM_OK;
}

static int loop_step(const ngpulm_model* m, const float* logits, int64_t row_stride, const float* dur_logits,
                     int64_t dur_stride, const int32_t* durations, int32_t D, int32_t B, int32_t* states,
                     int32_t* frame_idx, int32_t* sym_count, const int32_t* lengths, int32_t max_symbols, float lambda,
                     int32_t blank_id, const float* ilm, int64_t ilm_stride, float lambda_ilm, int32_t* tokens_out,
                     int32_t* emit_out, int32_t* emit_len, int32_t* last_token, int32_t max_len, uint32_t flags,
                     ngpulm_stream stream) {
  if (int r = check_hot(m, B)) return r;
  if (blank_id < 0 || blank_id > m->h.V) return err(NGPULM_EUSAGE, "blank_id outside [0, V]");
  if (max_symbols < 1 || max_len < 0) return err(NGPULM_EUSAGE, "max_symbols < 1 or max_len < 0");
  if (m->h.V % 4 != 0 || m->h.V > 1024) return err(NGPULM_EUSAGE, "loop step needs V % 4 == 0 and V <= 1024");
  if (D < 0 || D > NGPULM_MAX_DURATIONS) return err(NGPULM_EUSAGE, "number of durations outside [1, NGPULM_MAX_DURATIONS]");
  if (D > 0) {
    if (!durations) return err(NGPULM_EUSAGE, "NULL durations");
    for (int32_t j = 0; j < D; ++j)
      if (durations[j] < 0) return err(NGPULM_EUSAGE, "negative duration");
  }
  if (B == 0) return NGPULM_OK;
  if (!states && (lambda != 0.f || ilm)) return err(NGPULM_EUSAGE, "states NULL (plain greedy, no LM) needs lambda == 0 and no ILM");
  if (!logits || !frame_idx || !sym_count || !lengths || !tokens_out || !emit_len ||
      (max_len > 0 && !emit_out) || (D > 0 && !dur_logits))
    return err(NGPULM_EUSAGE, "NULL device buffer");
  if (B > 1 && row_stride < (int64_t)m->h.V + 1) return err(NGPULM_EUSAGE, "row_stride < V+1");
  if (ilm && B > 1 && ilm_stride < (int64_t)m->h.V) return err(NGPULM_EUSAGE, "ilm_stride < V");
  if (D > 0 && B > 1 && dur_stride < D) return err(NGPULM_EUSAGE, "dur_stride < number of durations");
  int e = ngpulm::launch_transducer_loop(m->dm, logits, row_stride, B, states, frame_idx, sym_count, lengths,
                                         max_symbols, lambda, blank_id, ilm, ilm_stride, lambda_ilm, tokens_out,
                                         emit_out, emit_len, last_token, max_len, dur_logits, dur_stride, durations,
                                         D, flags, stream);
  if (e) return cuda_err((cudaError_t)e, "transducer loop step launch");
  return NGPULM_OK;
}

int ngpulm_transducer_loop_step_ex(const ngpulm_model* m, const float* logits, int64_t row_stride, int32_t B,
                                   int32_t* states, int32_t* frame_idx, int32_t* sym_count, const int32_t* lengths,
                                   int32_t max_symbols, float lambda, int32_t blank_id, const float* ilm,
                                   int64_t ilm_stride, float lambda_ilm, int32_t* tokens_out, int32_t* emit_out,
                                   int32_t* emit_len, int32_t* last_token, int32_t max_len, uint32_t flags,
                                   ngpulm_stream stream) {
  if (flags & ~(uint32_t)NGPULM_STEP_INPUTS_READY) return err(NGPULM_EUSAGE, "unknown flags");
  return loop_step(m, logits, row_stride, nullptr, 0, nullptr, 0, B, states, frame_idx, sym_count, lengths,
                   max_symbols, lambda, blank_id, ilm, ilm_stride, lambda_ilm, tokens_out, emit_out, emit_len,
                   last_token, max_len, flags, stream);
}

int ngpulm_transducer_loop_step(const ngpulm_model* m, const float* logits, int64_t row_stride, int32_t B,
                                int32_t* states, int32_t* frame_idx, int32_t* sym_count, const int32_t* lengths,
                                int32_t max_symbols, float lambda, int32_t blank_id, const float* ilm,
                                int64_t ilm_stride, float lambda_ilm, int32_t* tokens_out, int32_t* emit_out,
                                int32_t* emit_len, int32_t* last_token, int32_t max_len, ngpulm_stream stream) {
  return ngpulm_transducer_loop_step_ex(m, logits, row_stride, B, states, frame_idx, sym_count, lengths, max_symbols,
                                        lambda, blank_id, ilm, ilm_stride, lambda_ilm, tokens_out, emit_out, emit_len,
                                        last_token, max_len, 0u, stream);
}

int ngpulm_tdt_loop_step_ex(const ngpulm_model* m, const float* logits, int64_t row_stride, const float* dur_logits,
                            int64_t dur_stride, const int32_t* durations, int32_t num_durations, int32_t B,
                            int32_t* states, int32_t* frame_idx, int32_t* sym_count, const int32_t* lengths,
                            int32_t max_symbols, float lambda, int32_t blank_id, const float* ilm, int64_t ilm_stride,
                            float lambda_ilm, int32_t* tokens_out, int32_t* emit_out, int32_t* emit_len,
                            int32_t* last_token, int32_t max_len, uint32_t flags, ngpulm_stream stream) {
  if (flags & ~(uint32_t)NGPULM_STEP_INPUTS_READY) return err(NGPULM_EUSAGE, "unknown flags");
  if (num_durations < 1) return err(NGPULM_EUSAGE, "number of durations outside [1, NGPULM_MAX_DURATIONS]");
  return loop_step(m, logits, row_stride, dur_logits, dur_stride, durations, num_durations, B, states, frame_idx,
                   sym_count, lengths, max_symbols, lambda, blank_id, ilm, ilm_stride, lambda_ilm, tokens_out,
                   emit_out, emit_len, last_token, max_len, flags, stream);
}

int ngpulm_tdt_loop_step(const ngpulm_model* m, const float* logits, int64_t row_stride, const float* dur_logits,
                         int64_t dur_stride, const int32_t* durations, int32_t num_durations, int32_t B,
                         int32_t* states, int32_t* frame_idx, int32_t* sym_count, const int32_t* lengths,
                         int32_t max_symbols, float lambda, int32_t blank_id, const float* ilm, int64_t ilm_stride,
                         float lambda_ilm, int32_t* tokens_out, int32_t* emit_out, int32_t* emit_len,
                         int32_t* last_token, int32_t max_len, ngpulm_stream stream) {
  return ngpulm_tdt_loop_step_ex(m, logits, row_stride, dur_logits, dur_stride, durations, num_durations, B, states,
                                 frame_idx, sym_count, lengths, max_symbols, lambda, blank_id, ilm, ilm_stride,
                                 lambda_ilm, tokens_out, emit_out, emit_len, last_token, max_len, 0u, stream);
}

int ngpulm_fused_greedy_step_rows(const ngpulm_model* m, int32_t mode, const float* logits, int64_t row_stride,
                                  int32_t B, const float* lm_scores, const int32_t* lm_next, const float* lm_final,
                                  int64_t lm_stride, int32_t* states, int32_t* prev, const uint8_t* active,
                                  float lambda, int32_t blank_id, int32_t* tokens_out, ngpulm_stream stream) {
  if (int r = check_hot(m, B)) return r;
  if (mode != NGPULM_CTC && mode != NGPULM_RNNT && mode != NGPULM_AED) return err(NGPULM_EUSAGE, "bad mode");
  if (blank_id < 0 || blank_id > m->h.V) return err(NGPULM_EUSAGE, "blank_id outside [0, V]");
  if (m->h.V > 1024) return err(NGPULM_EUSAGE, "fused step from rows needs V <= 1024");
  if (B == 0) return NGPULM_OK;
  if (!logits || !lm_scores || !lm_next || !states || !tokens_out || (mode == NGPULM_CTC && !prev) ||
      (mode == NGPULM_AED && !lm_final))
    return err(NGPULM_EUSAGE, "NULL device buffer");
  if (B > 1 && row_stride < (int64_t)m->h.V + 1) return err(NGPULM_EUSAGE, "row_stride < V+1");
  if (B > 1 && lm_stride < (int64_t)m->h.V) return err(NGPULM_EUSAGE, "lm_stride < V");
  int e = ngpulm::launch_fused_rows(mode, logits, row_stride, lm_scores, lm_next, lm_final, lm_stride, B, m->h.V,
                                    states, prev, active, lambda, blank_id, tokens_out, stream);
  if (e) return cuda_err((cudaError_t)e, "fused step (rows) launch");
  return NGPULM_OK;
}

int ngpulm_fused_topk(const ngpulm_model* m, const float* logits, int64_t row_stride, int32_t B,
                      const int32_t* states, const float* ilm, int64_t ilm_stride, float lambda, float lambda_ilm,
                      int32_t eos_id, int32_t k, float* topk_scores, int32_t* topk_cols, int32_t* topk_next,
                      ngpulm_stream stream) {
  if (int r = check_hot(m, B)) return r;
  if (eos_id < 0 || eos_id > m->h.V) return err(NGPULM_EUSAGE, "eos_id outside [0, V]");
  if (k < 1 || k > NGPULM_MAX_TOPK) return err(NGPULM_EUSAGE, "k outside [1, NGPULM_MAX_TOPK]");
  if (m->h.V % 4 != 0 || m->h.V > 1024) return err(NGPULM_EUSAGE, "top-k needs V % 4 == 0 and V <= 1024");
  if (B == 0) return NGPULM_OK;
  if (!logits || !states || !topk_scores || !topk_cols) return err(NGPULM_EUSAGE, "NULL device buffer");
  if (B > 1 && row_stride < (int64_t)m->h.V + 1) return err(NGPULM_EUSAGE, "row_stride < V+1");
  if (ilm && B > 1 && ilm_stride < (int64_t)m->h.V) return err(NGPULM_EUSAGE, "ilm_stride < V");
  int e = ngpulm::launch_topk(m->dm, logits, row_stride, B, states, ilm, ilm_stride, lambda, lambda_ilm, eos_id, k,
                              topk_scores, topk_cols, topk_next, stream);
  if (e) return cuda_err((cudaError_t)e, "top-k launch");
  return NGPULM_OK;
}

int ngpulm_ctc_greedy_decode(const ngpulm_model* m, const float* logits, int64_t row_stride, int64_t frame_stride,
                             int32_t B, int32_t T, const int32_t* lengths, int32_t* states, int32_t* prev,
                             float lambda, int32_t blank_id, int32_t* frames_out, int32_t* emit_out,
                             int32_t* emit_len, ngpulm_stream stream) {
  if (int r = check_hot(m, B)) return r;
  if (T < 0) return err(NGPULM_EUSAGE, "T < 0");
  if (blank_id < 0 || blank_id > m->h.V) return err(NGPULM_EUSAGE, "blank_id outside [0, V]");
  if (m->h.V % 4 != 0 || m->h.V > 1024) return err(NGPULM_EUSAGE, "ctc decode needs V % 4 == 0 and V <= 1024");
  if (!std::isfinite(lambda)) return err(NGPULM_EUSAGE, "lambda must be finite");
  if (B == 0) return NGPULM_OK;
  if (!states && lambda != 0.f) return err(NGPULM_EUSAGE, "states NULL (plain greedy, no LM) needs lambda == 0");
  if (!prev || (T > 0 && !logits)) return err(NGPULM_EUSAGE, "NULL device buffer");
  if (T > 1 && frame_stride < (int64_t)m->h.V + 1 && row_stride < (int64_t)m->h.V + 1)
    return err(NGPULM_EUSAGE, "frames overlap: frame_stride and row_stride < V+1");
  int e = ngpulm::launch_ctc_decode(m->dm, logits, row_stride, frame_stride, B, T, lengths, states, prev, lambda,
                                    blank_id, frames_out, emit_out, emit_len, stream);
  if (e) return cuda_err((cudaError_t)e, "ctc decode launch");
  return NGPULM_OK;
}

int ngpulm_check(const ngpulm_model* m, ngpulm_stream stream, int64_t* first_bad_row) {
  if (!m || !first_bad_row) return err(NGPULM_EUSAGE, "NULL argument");
  if (m->device < 0) return err(NGPULM_EUSAGE, "host-only model");
  DeviceGuard g(m->device);
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_err(e, "stream synchronize");
  unsigned long long v = 0, none = ULLONG_MAX;
  e = cudaMemcpy(&v, m->dm.bad_row, 8, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(m->dm.bad_row, &none, 8, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_err(e, "read bad-row word");
  *first_bad_row = v == ULLONG_MAX ? -1 : (int64_t)v;
  return NGPULM_OK;
}

int ngpulm_advance_host(ngpulm_model* m, const int32_t* states_host, int32_t B, float* scores_host,
                        int32_t* next_host, float* final_host, ngpulm_stream stream) {
  if (int r = check_hot(m, B)) return r;
  if (B == 0) return NGPULM_OK;
  if (!states_host || !scores_host || !next_host) return err(NGPULM_EUSAGE, "NULL host buffer");
  const size_t V = (size_t)m->h.V;
  const size_t o_sc = align256((size_t)B * 4), o_nx = align256(o_sc + (size_t)B * V * 4),
               o_fi = align256(o_nx + (size_t)B * V * 4);
  const size_t need = align256(o_fi + (size_t)B * 4);
  std::lock_guard<std::mutex> lk(m->mu);
  if (m->scratch_bytes < need) {
    if (m->scratch) cudaFree(m->scratch);
    m->scratch = nullptr;
    m->scratch_bytes = 0;
    cudaError_t e = cudaMalloc(&m->scratch, need);
    if (e != cudaSuccess) return cuda_err(e, "cudaMalloc(scratch)");
    m->scratch_bytes = need;
  }
  auto* base = static_cast<unsigned char*>(m->scratch);
  auto* d_st = reinterpret_cast<int32_t*>(base);
  auto* d_sc = reinterpret_cast<float*>(base + o_sc);
  auto* d_nx = reinterpret_cast<int32_t*>(base + o_nx);
  auto* d_fi = reinterpret_cast<float*>(base + o_fi);
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(d_st, states_host, (size_t)B * 4, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_err(e, "H2D states");
  int k = ngpulm::launch_advance(m->dm, d_st, B, d_sc, d_nx, final_host ? d_fi : nullptr, stream);
  if (k) return cuda_err((cudaError_t)k, "advance launch");
  e = cudaMemcpyAsync(scores_host, d_sc, (size_t)B * V * 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(next_host, d_nx, (size_t)B * V * 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && final_host) e = cudaMemcpyAsync(final_host, d_fi, (size_t)B * 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_err(e, "D2H results");
  return NGPULM_OK;
}

#ifdef NGPULM_PHASE_TIMING
int ngpulm_debug_probe(const ngpulm::DevModel* m, const int32_t* states, int32_t B, long long* out_dev);
int ngpulm_debug_probe_model(const ngpulm_model* m, const int32_t* states, int32_t B, long long* out_dev) {
  return ngpulm_debug_probe(&m->dm, states, B, out_dev);
}
#endif

int ngpulm_touched_bytes(const ngpulm_model* m, const int32_t* states_host, int32_t B, int64_t* out_bytes) {
  if (!m || !out_bytes || B < 0 || (B > 0 && !states_host)) return err(NGPULM_EUSAGE, "bad argument");
  std::unordered_set<int32_t> seen;
  int64_t bytes = (int64_t)m->h.V * 12 + (int64_t)B * 4;  // root arcs once + finals read
  for (int32_t b = 0; b < B; ++b) {
    int32_t s = states_host[b];
    if (s < 0 || s >= m->h.num_states) continue;
    for (int it = 0; it <= NGPULM_MAX_ORDER && s != 0; ++it) {
      if (!seen.insert(s).second) break;  // the rest of this chain is already counted
      bytes += 16 + 12 * (int64_t)(m->h.arc_off[s + 1] - m->h.arc_off[s]);
      s = m->h.boff_to[s];
    }
  }
  *out_bytes = bytes;
  return NGPULM_OK;
}

}  // extern "C"
