// NGPU-LM ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, obviously-correct CPU statement of what the hot path computes.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// `--impl reference` legs may load it. It shares no code with the CUDA path
// (paper_2505_22857_b200/): it has its own ARPA reader, works on token-sequence
// contexts held in hash maps (the "hash tables" design of PAPER.md:106, the
// OracleLM of SPEC.md:222-225) and never builds the flat trie.
//
// What it computes (each function cites the passage it follows):
//   score64(ctx, v)   textbook ARPA back-off in double                 PAPER.md:98 §2.1
//   score32(s, v)     the same value associated the way Algorithm 1
//                     accumulates it, in float                         PAPER.md:65-84 Alg. 1
//   next(s, v)        longest suffix of ctx(s)+v that is a state       PAPER.md:101-102 §2.1
//   final32/64(s)     </s> weight reached through back-offs            PAPER.md:142-143 §2.3
//   fused step        RNN-T two-stage / CTC three-group / AED eos      PAPER.md:132-143 §2.3
// Readings of the paper where it is silent are DESIGN.md §Readings R1..R20
// (= SURVEY.md §8(c) points 1..20); each is cited as [Rn] below.
//
// Pins (tests/test_oracle_*.py, -m "not gpu"): Fig. 1 worked example with exact
// rational values (tests/golden/fig1.*), Witten-Bell interpolation recomputed
// from corpus counts, per-state normalization, sentence replay, depth bound,
// N=1/N=2 special cases, f32-vs-f64 error bound, decoder identities.
// Parity unpinned: none of the functions above.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

namespace {

thread_local std::string g_err;

struct VecHash {
  size_t operator()(const std::vector<int32_t>& v) const {
    uint64_t h = 1469598103934665603ull;  // FNV-1a over the ids
    for (int32_t x : v) { h ^= (uint32_t)x; h *= 1099511628211ull; }
    return (size_t)h;
  }
};

struct Entry {
  double log10p = 0;    // as written in the ARPA
  bool has_bo = false;
  double log10bo = 0;
};

constexpr double kLn10 = 2.302585092994045684;  // [R1] ln(10) in double

// [R1] log10 -> ln: one double multiply; [R3] ARPA's -99 dummy -> -1e30 sentinel
double to_ln64(double log10v) { return log10v <= -99.0 ? -1e30 : log10v * kLn10; }
float to_ln32(double log10v) { return (float)to_ln64(log10v); }

struct Oracle {
  int32_t V = 0, N = 0;
  int32_t BOS = 0, EOS = 0, UNK = 0;  // [R6] meta ids <s>=V, </s>=V+1, <unk>=V+2
  std::unordered_map<std::vector<int32_t>, Entry, VecHash> ngram;  // full n-gram -> entry
  std::unordered_map<std::string, int32_t> vocab;
  int64_t M = 0;            // vocabulary tokens without a unigram  [R2]
  double unk_log10 = 0;     // the <unk> unigram (log10)
  bool has_unk = false;
  // states  [R5],[R6]
  std::vector<std::vector<int32_t>> ctx;          // state id -> context
  std::map<std::vector<int32_t>, int32_t> state;  // context -> state id
  int32_t bos_state = 0;

  const Entry* find(const std::vector<int32_t>& g) const {
    auto it = ngram.find(g);
    return it == ngram.end() ? nullptr : &it->second;
  }
  bool is_state(const std::vector<int32_t>& c) const { return state.count(c) != 0; }

  // [R2] normalized <unk>: log p_unk - ln M, evaluated in double
  double unk_norm64() const { return to_ln64(unk_log10) - std::log((double)M); }

  // ---------------------------------------------------------------- definitions
  // W(t|c) = B(c) + W(t|c[1:]); at the empty context an absent
  // token gets the (normalized, [R2]) <unk> weight. B(c) = 0 when c has no entry.
  double score64(const std::vector<int32_t>& c, int32_t v) const {
    std::vector<int32_t> g(c);
    g.push_back(v);
    if (const Entry* e = find(g)) return to_ln64(e->log10p);
    if (c.empty()) return unk_norm64();
    double b = 0.0;
    if (const Entry* ce = find(c)) b = ce->has_bo ? to_ln64(ce->log10bo) : 0.0;
    return b + score64(std::vector<int32_t>(c.begin() + 1, c.end()), v);
  }

  // [R8] back-off target: longest proper suffix of c that is a state
  std::vector<int32_t> boff_ctx(const std::vector<int32_t>& c) const {
    for (size_t j = 1; j <= c.size(); ++j) {
      std::vector<int32_t> s(c.begin() + j, c.end());
      if (s.empty() || is_state(s)) return s;
    }
    return {};
  }

  // PAPER.md:65-84 Algorithm 1, value of token v in state s, in float:
  //   acc_boff = 0; per level: score = acc_boff + arc_weight (first level that
  //   has an arc for v wins, lines 77-79); acc_boff += boff_weights[state];
  //   state = boff_to_states[state].  [R10] left-associated, round-to-nearest.
  // The root level has an arc for every token ([R2]).
  // Also returns the number of levels visited (Algorithm 1 iterations).
  float score32(int32_t s, int32_t v, int* levels = nullptr) const {
    std::vector<int32_t> c = ctx[s];
    float acc = 0.0f;
    for (int lvl = 1;; ++lvl) {
      std::vector<int32_t> g(c);
      g.push_back(v);
      const Entry* e = find(g);
      if (e || c.empty()) {
        if (levels) *levels = lvl;
        float w = e ? to_ln32(e->log10p) : (float)unk_norm64();
        return acc + w;
      }
      const Entry* ce = find(c);
      float bo = (ce && ce->has_bo) ? to_ln32(ce->log10bo) : 0.0f;
      acc = acc + bo;
      c = boff_ctx(c);
    }
  }

  // next state: longest suffix of ctx(s)+v that is a state ([R7])
  int32_t next(int32_t s, int32_t v) const {
    std::vector<int32_t> g(ctx[s]);
    g.push_back(v);
    for (size_t j = 0; j <= g.size(); ++j) {
      std::vector<int32_t> suf(g.begin() + j, g.end());
      auto it = state.find(suf);
      if (it != state.end()) return it->second;
    }
    return 0;  // unreachable: the empty context is the root state
  }

  // longest suffix of an arbitrary history that is a state (decoder start states)
  int32_t state_of(const std::vector<int32_t>& hist) const {
    for (size_t j = 0; j <= hist.size(); ++j) {
      std::vector<int32_t> suf(hist.begin() + j, hist.end());
      auto it = state.find(suf);
      if (it != state.end()) return it->second;
    }
    return 0;
  }

  // PAPER.md:142-143 final weight = </s> reached "by traversing backoff
  // transitions"; [R9] associated like Algorithm 1 (final = column "</s>").
  float final32(int32_t s) const { return score32(s, EOS); }
  double final64(int32_t s) const { return score64(ctx[s], EOS); }

  // ---------------------------------------------------------------- fused step
  // PAPER.md:131-143 §2.3. [R13] fused = fmaf(lambda, lm, asr) single rounding;
  // [R14] argmax ties -> lowest column; [R19] token v <-> column v (v < blank)
  // or v+1; [R16] stage 2 without renormalization; [R17] prev = frame-level
  // selection at t-1 (-1 = none).
  int32_t tok_of(int32_t col, int32_t sp) const { return col < sp ? col : col - 1; }

  // [R21] internal-LM subtraction ("-ILM+LM"; SPEC.md:301
  // fuse_scores: out = asr + lambda*lm - lambda_ilm*aux): on the LM-rescored
  // columns, fmaf(-lambda_ilm, ilm[v], fmaf(lambda, lm[v], asr[c])).
  float rescore(float lambda, float lmv, float asr, const float* ilm, float lam_ilm, int32_t v) const {
    const float y = std::fmaf(lambda, lmv, asr);
    return ilm ? std::fmaf(-lam_ilm, ilm[v], y) : y;
  }

  void fused_step(int mode, const float* asr, int32_t sp, float lambda, int32_t* st,
                  int32_t* prev, int32_t* token_out, const float* ilm = nullptr, float lam_ilm = 0.f) const {
    const int32_t ncols = V + 1, s = *st;
    std::vector<float> lm(V);
    for (int32_t v = 0; v < V; ++v) lm[v] = score32(s, v);
    auto argmax = [&](const std::vector<float>& val, int32_t skip) {
      int32_t best = -1;
      for (int32_t c = 0; c < ncols; ++c) {
        if (c == skip) continue;
        if (best < 0 || val[c] > val[best]) best = c;  // strict: earliest column wins ties
      }
      return best;
    };
    std::vector<float> val(ncols);
    if (mode == 1) {  // RNN-T / TDT two-stage
      for (int32_t c = 0; c < ncols; ++c) val[c] = asr[c];
      int32_t c1 = argmax(val, -1);
      if (c1 == sp) { *token_out = sp; return; }  // "If blank is predicted, we retain it"
      for (int32_t c = 0; c < ncols; ++c)
        if (c != sp) val[c] = rescore(lambda, lm[tok_of(c, sp)], asr[c], ilm, lam_ilm, tok_of(c, sp));
      int32_t c2 = argmax(val, sp);  // "greedy selection among non-blank symbols"
      *token_out = c2;
      *st = next(s, tok_of(c2, sp));
      return;
    }
    if (mode == 0) {  // CTC three groups
      const int32_t p = *prev;
      for (int32_t c = 0; c < ncols; ++c)
        val[c] = (c == sp || c == p) ? asr[c] : rescore(lambda, lm[tok_of(c, sp)], asr[c], ilm, lam_ilm, tok_of(c, sp));
      int32_t c = argmax(val, -1);
      *token_out = c;
      if (c == sp) { *prev = -1; return; }
      if (c == p) return;  // repeated token: collapsed, no LM advance
      *st = next(s, tok_of(c, sp));
      *prev = c;
      return;
    }
    // AED: eos column scored with the final weight
    for (int32_t c = 0; c < ncols; ++c)
      val[c] = (c == sp) ? std::fmaf(lambda, final32(s), asr[c])
                         : rescore(lambda, lm[tok_of(c, sp)], asr[c], ilm, lam_ilm, tok_of(c, sp));
    int32_t c = argmax(val, -1);
    *token_out = c;
    if (c != sp) *st = next(s, tok_of(c, sp));
  }

  // The k best AED expansions (beam search with fusion): all
  // V+1 fused values by the AED rule, ordered by value descending then
  // column ascending; NaN values are never candidates (R14, R15).
  void topk(const float* asr, int32_t sp, float lambda, int32_t s, const float* ilm, float lam_ilm, int32_t k,
            float* sc, int32_t* cols, int32_t* nxt) const {
    const int32_t ncols = V + 1;
    std::vector<std::pair<float, int32_t>> cand;
    for (int32_t c = 0; c < ncols; ++c) {
      const float v = (c == sp) ? std::fmaf(lambda, final32(s), asr[c])
                                : rescore(lambda, score32(s, tok_of(c, sp)), asr[c], ilm, lam_ilm, tok_of(c, sp));
      if (!std::isnan(v)) cand.emplace_back(v, c);
    }
    std::sort(cand.begin(), cand.end(), [](const std::pair<float, int32_t>& a, const std::pair<float, int32_t>& b) {
      return a.first > b.first || (a.first == b.first && a.second < b.second);
    });
    for (int32_t i = 0; i < k; ++i) {
      if (i < (int32_t)cand.size()) {
        sc[i] = cand[i].first;
        cols[i] = cand[i].second;
        nxt[i] = cand[i].second == sp ? s : next(s, tok_of(cand[i].second, sp));
      } else {
        sc[i] = -INFINITY; cols[i] = -1; nxt[i] = -1;
      }
    }
  }
};

// ---------------------------------------------------------------- ARPA reader
bool fail(const std::string& m) { g_err = m; return false; }

bool load(Oracle& o, const char* arpa, const char* vocab_path, int32_t V) {
  if (vocab_path && *vocab_path) {
    std::ifstream vf(vocab_path);
    if (!vf) return fail(std::string("cannot open vocab ") + vocab_path);
    std::string line;
    int32_t id = 0;
    while (std::getline(vf, line)) {
      while (!line.empty() && (line.back() == '\r' || line.back() == ' ')) line.pop_back();
      o.vocab[line] = id++;
    }
    if (V > 0 && V != id) return fail("vocab size mismatch");
    V = id;
  } else {
    if (V <= 0) return fail("vocab_size required without a vocab file");
    for (int32_t i = 0; i < V; ++i) o.vocab[std::to_string(i)] = i;
  }
  o.V = V; o.BOS = V; o.EOS = V + 1; o.UNK = V + 2;
  o.vocab["<s>"] = o.BOS; o.vocab["</s>"] = o.EOS; o.vocab["<unk>"] = o.UNK;

  std::ifstream f(arpa);
  if (!f) return fail(std::string("cannot open ") + arpa);
  std::string line;
  std::map<int, long long> declared, seen;
  int section = -1;  // -1 before \data\, 0 in \data\, k in \k-grams:
  bool ended = false;
  long long lineno = 0;
  while (std::getline(f, line)) {
    ++lineno;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    if (line == "\\data\\") { section = 0; continue; }
    if (line == "\\end\\") { ended = true; break; }
    if (section < 0) continue;
    if (line[0] == '\\') {
      int k = 0;
      if (std::sscanf(line.c_str(), "\\%d-grams:", &k) != 1) return fail("bad section " + line);
      section = k;
      continue;
    }
    if (section == 0) {
      int k = 0; long long n = 0;
      if (std::sscanf(line.c_str(), "ngram %d=%lld", &k, &n) != 2) return fail("bad header " + line);
      declared[k] = n;
      continue;
    }
    std::istringstream ss(line);
    std::vector<std::string> fld;
    std::string x;
    while (ss >> x) fld.push_back(x);
    const int k = section;
    if ((int)fld.size() != k + 1 && (int)fld.size() != k + 2)
      return fail("malformed line " + std::to_string(lineno));
    Entry e;
    e.log10p = std::strtod(fld[0].c_str(), nullptr);
    if ((int)fld.size() == k + 2) { e.has_bo = true; e.log10bo = std::strtod(fld[k + 1].c_str(), nullptr); }
    std::vector<int32_t> g;
    for (int i = 1; i <= k; ++i) {
      auto it = o.vocab.find(fld[i]);
      if (it == o.vocab.end()) return fail("OOV token '" + fld[i] + "' line " + std::to_string(lineno));
      g.push_back(it->second);
    }
    seen[k] += 1;
    if (k == 1 && g[0] == o.UNK) { o.has_unk = true; o.unk_log10 = e.log10p; continue; }
    // [R5] n-grams containing <unk> beyond the unigram are unreachable: dropped
    if (std::find(g.begin(), g.end(), o.UNK) != g.end()) continue;
    if (!o.ngram.emplace(g, e).second) return fail("duplicate n-gram line " + std::to_string(lineno));
  }
  if (!ended) return fail("missing \\end\\");
  for (auto& d : declared) {
    if (seen[d.first] != d.second) return fail("count mismatch for order " + std::to_string(d.first));
    if (d.second > 0) o.N = std::max(o.N, d.first);  // order N = highest declared non-empty order
  }
  if (!o.find({o.EOS})) return fail("missing </s> unigram");
  // [R4] the <s> unigram's probability is never used: "<s>" is a state, not a token

  for (int32_t v = 0; v < V; ++v)
    if (!o.find({v})) ++o.M;
  if (o.M > 0 && !o.has_unk) return fail("<unk> unigram needed but missing");

  // [R5] states: root + every entry of order < N whose last token is a vocab
  // token, plus the <s> unigram. [R6] ids: root = 0, then (order, ids lexicographic).
  std::vector<std::vector<int32_t>> st;
  for (auto& kv : o.ngram) {
    const auto& g = kv.first;
    if ((int)g.size() >= o.N) continue;
    int32_t last = g.back();
    if (last < V || (g.size() == 1 && last == o.BOS)) st.push_back(g);
  }
  std::sort(st.begin(), st.end(), [](const std::vector<int32_t>& a, const std::vector<int32_t>& b) {
    if (a.size() != b.size()) return a.size() < b.size();
    return a < b;
  });
  o.ctx.push_back({});
  o.state[{}] = 0;
  for (auto& g : st) { o.state[g] = (int32_t)o.ctx.size(); o.ctx.push_back(g); }
  auto b = o.state.find({o.BOS});
  o.bos_state = b == o.state.end() ? 0 : b->second;  // [R4]
  return true;
}

template <class F>
void parallel_rows(int64_t n, int nthreads, F fn) {
  if (nthreads <= 0) nthreads = (int)std::max(1u, std::thread::hardware_concurrency());
  nthreads = (int)std::min<int64_t>(nthreads, std::max<int64_t>(1, n));
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; ++t)
    th.emplace_back([&, t] { for (int64_t i = t; i < n; i += nthreads) fn(i); });
  for (auto& x : th) x.join();
}

}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

void* oracle_load(const char* arpa, const char* vocab, int32_t V) {
  auto o = std::make_unique<Oracle>();
  if (!load(*o, arpa, vocab, V)) return nullptr;
  return o.release();
}
void oracle_free(void* h) { delete (Oracle*)h; }

int32_t oracle_vocab_size(void* h) { return ((Oracle*)h)->V; }
int32_t oracle_order(void* h) { return ((Oracle*)h)->N; }
int32_t oracle_num_states(void* h) { return (int32_t)((Oracle*)h)->ctx.size(); }
int32_t oracle_bos_state(void* h) { return ((Oracle*)h)->bos_state; }
int64_t oracle_num_unk_filled(void* h) { return ((Oracle*)h)->M; }

// context of state s (meta id V = <s>); returns its length, copies up to cap ids
int32_t oracle_state_context(void* h, int32_t s, int32_t* out, int32_t cap) {
  auto& c = ((Oracle*)h)->ctx[s];
  for (int32_t i = 0; i < (int32_t)c.size() && i < cap; ++i) out[i] = c[i];
  return (int32_t)c.size();
}

// longest suffix of ("<s>" if with_bos) + tokens that is a state
int32_t oracle_state_of(void* h, int32_t with_bos, const int32_t* tokens, int32_t n) {
  auto* o = (Oracle*)h;
  std::vector<int32_t> hist;
  if (with_bos) hist.push_back(o->BOS);
  hist.insert(hist.end(), tokens, tokens + n);
  return o->state_of(hist);
}

// full rows for states[0..n): score32 [n,V] (Algorithm-1 order, float),
// score64 [n,V] (definition, double; may be NULL), next [n,V], levels [n]
// (Algorithm 1 iterations = max over tokens; may be NULL)
void oracle_rows(void* h, const int32_t* states, int64_t n, float* s32, double* s64,
                 int32_t* next, int32_t* levels, int nthreads) {
  auto* o = (Oracle*)h;
  const int32_t V = o->V;
  parallel_rows(n, nthreads, [&](int64_t i) {
    int32_t s = states[i];
    int maxlv = 0;
    for (int32_t v = 0; v < V; ++v) {
      int lv = 0;
      s32[i * V + v] = o->score32(s, v, &lv);
      maxlv = std::max(maxlv, lv);
      if (s64) s64[i * V + v] = o->score64(o->ctx[s], v);
      next[i * V + v] = o->next(s, v);
    }
    if (levels) levels[i] = maxlv;
  });
}

void oracle_finals(void* h, const int32_t* states, int64_t n, float* f32, double* f64) {
  auto* o = (Oracle*)h;
  for (int64_t i = 0; i < n; ++i) {
    f32[i] = o->final32(states[i]);
    if (f64) f64[i] = o->final64(states[i]);
  }
}

// one fused greedy step for n rows; row i of the logits at logits + i*row_stride
// (V+1 columns). mode 0 = CTC, 1 = RNN-T, 2 = AED. active may be NULL (all).
// Inactive rows are untouched and get token -1.
void oracle_fused_step(void* h, int mode, const float* logits, int64_t row_stride, int64_t n,
                       int32_t* states, int32_t* prev, const uint8_t* active, float lambda,
                       int32_t blank_id, int32_t* tokens_out, int nthreads) {
  auto* o = (Oracle*)h;
  parallel_rows(n, nthreads, [&](int64_t i) {
    if (active && !active[i]) { tokens_out[i] = -1; return; }
    int32_t dummy = -1;
    o->fused_step(mode, logits + i * row_stride, blank_id, lambda, &states[i],
                  prev ? &prev[i] : &dummy, &tokens_out[i]);
  });
}

// fused step with the ILM term (R21); ilm row i at ilm + i*ilm_stride, V entries
void oracle_fused_step_ilm(void* h, int mode, const float* logits, int64_t row_stride, int64_t n,
                           int32_t* states, int32_t* prev, const uint8_t* active, float lambda, int32_t blank_id,
                           const float* ilm, int64_t ilm_stride, float lam_ilm, int32_t* tokens_out, int nthreads) {
  auto* o = (Oracle*)h;
  parallel_rows(n, nthreads, [&](int64_t i) {
    if (active && !active[i]) { tokens_out[i] = -1; return; }
    int32_t dummy = -1;
    o->fused_step(mode, logits + i * row_stride, blank_id, lambda, &states[i], prev ? &prev[i] : &dummy,
                  &tokens_out[i], ilm + i * ilm_stride, lam_ilm);
  });
}

// k best AED expansions per row (ilm may be NULL)
void oracle_topk(void* h, const float* logits, int64_t row_stride, int64_t n, const int32_t* states,
                 const float* ilm, int64_t ilm_stride, float lambda, float lam_ilm, int32_t eos_id, int32_t k,
                 float* sc, int32_t* cols, int32_t* nxt, int nthreads) {
  auto* o = (Oracle*)h;
  parallel_rows(n, nthreads, [&](int64_t i) {
    o->topk(logits + i * row_stride, eos_id, lambda, states[i], ilm ? ilm + i * ilm_stride : nullptr, lam_ilm, k,
            sc + i * k, cols + i * k, nxt + i * k);
  });
}

// The synthetic joint (test input, not the method; the oracle's own copy of
// the counter-based generator of synth/joint.cu).
static uint64_t smix(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static void joint_row(uint64_t seed, int32_t t, int32_t u, int32_t last, int32_t ncols, int32_t blank, float bias,
                      float temp, float* out) {
  uint64_t h = seed;
  h = smix(h ^ (uint64_t)(int64_t)t);
  h = smix(h ^ (uint64_t)(int64_t)u);
  h = smix(h ^ (uint64_t)(int64_t)(last + 1));
  for (int32_t v = 0; v < ncols; ++v) {
    float x = (float)(smix(h ^ (uint64_t)v) >> 40) * 5.9604644775390625e-08f;
    if (v == blank) x = x + bias;
    out[v] = x * temp;
  }
}

// Greedy transducer decoding with fusion (SPEC.md:317-325
// transducer_greedy_fused): per utterance, frame loop t <
// lengths[i]; on each frame up to max_sym labels: the joint row for (t, u,
// last) -> the two-stage fused step; blank -> next frame; else emit (u += 1,
// last = the label's LM token, LM state advanced). emitted [n, max_len]
// (columns; emissions past max_len are counted, not stored), emit_len [n],
// states in/out.
void oracle_transducer_decode(void* h, uint64_t seed, float temp, float blank_bias, const int32_t* lengths, int64_t n,
                              int32_t* states, float lambda, int32_t blank_id, int32_t max_sym, int32_t max_len,
                              const float* ilm_rows, float lam_ilm, int32_t* emitted, int32_t* emit_len,
                              int nthreads) {
  auto* o = (Oracle*)h;
  const int32_t ncols = o->V + 1;
  parallel_rows(n, nthreads, [&](int64_t i) {
    std::vector<float> row(ncols);
    int32_t u = 0, last = -1;
    for (int32_t t = 0; t < lengths[i]; ++t) {
      for (int32_t k = 0; k < max_sym; ++k) {
        joint_row(seed, t, u, last, ncols, blank_id, blank_bias, temp, row.data());
        int32_t tok = -1, dummy = -1;
        o->fused_step(1, row.data(), blank_id, lambda, &states[i], &dummy, &tok,
                      ilm_rows ? ilm_rows + (size_t)i * o->V : nullptr, lam_ilm);
        if (tok == blank_id) break;  // "If blank is predicted, we retain it": next frame
        if (u < max_len) emitted[i * max_len + u] = tok;
        ++u;
        last = o->tok_of(tok, blank_id);
      }
    }
    emit_len[i] = u;
  });
}

// Greedy Token-and-Duration Transducer (TDT) decoding with fusion (PAPER.md:135:
// NGPU-LM in "the Token-and-Duration Transducer (TDT)" label-looping greedy
// decoder; R25). The joint row for (t, u, last) has V+1 token columns
// followed by D duration columns (duration index j <-> durations[j] frames).
// Per step: the token is the RNN-T two-stage fused decision over the token
// columns; the duration is the raw argmax over the duration
// columns (lowest index on ties, R14), untouched by the LM. A blank advances
// the frame by max(d, 1) (a blank must consume a frame); a label is emitted
// (LM state advanced) and advances the frame by d; a label with d = 0 stays on
// the frame, and after max_sym labels on one frame the frame advances by 1.
void oracle_tdt_decode(void* h, uint64_t seed, float temp, float blank_bias, const int32_t* lengths, int64_t n,
                       int32_t* states, float lambda, int32_t blank_id, const int32_t* durations, int32_t D,
                       int32_t max_sym, int32_t max_len, int32_t* emitted, int32_t* emit_len, int32_t* steps_out,
                       int nthreads) {
  auto* o = (Oracle*)h;
  const int32_t ntok = o->V + 1, ncols = ntok + D;
  parallel_rows(n, nthreads, [&](int64_t i) {
    std::vector<float> row(ncols);
    int32_t u = 0, last = -1, sym = 0, steps = 0;
    for (int32_t t = 0; t < lengths[i];) {
      joint_row(seed, t, u, last, ncols, blank_id, blank_bias, temp, row.data());
      int32_t tok = -1, dummy = -1;
      o->fused_step(1, row.data(), blank_id, lambda, &states[i], &dummy, &tok);
      int32_t j = 0;  // duration: raw argmax, lowest index on ties
      for (int32_t k = 1; k < D; ++k)
        if (row[ntok + k] > row[ntok + j]) j = k;
      const int32_t d = durations[j];
      ++steps;
      if (tok == blank_id) {
        t += std::max(d, 1);
        sym = 0;
        continue;
      }
      if (u < max_len) emitted[i * max_len + u] = tok;
      ++u;
      last = o->tok_of(tok, blank_id);
      if (d > 0) {
        t += d;
        sym = 0;
      } else if (++sym >= max_sym) {
        t += 1;
        sym = 0;
      }
    }
    emit_len[i] = u;
    if (steps_out) steps_out[i] = steps;
  });
}

// Greedy CTC decoding of whole utterances (SPEC.md:307-316 ctc_greedy_fused;
// PAPER.md:138-139): for t = 0..T-1, frame t of row i (logits + i*row_stride +
// t*frame_stride) gets one fused CTC step while t < lengths[i] (NULL: T).
// frames [n,T]: the column selected at each frame (-1 past the length);
// emitted [n,T]: the selections that are neither blank nor prev, in order;
// emit_len [n]. states / prev in/out.
void oracle_ctc_decode(void* h, const float* logits, int64_t row_stride, int64_t frame_stride, int64_t n,
                       int32_t T, const int32_t* lengths, int32_t* states, int32_t* prev, float lambda,
                       int32_t blank_id, int32_t* frames, int32_t* emitted, int32_t* emit_len, int nthreads) {
  auto* o = (Oracle*)h;
  parallel_rows(n, nthreads, [&](int64_t i) {
    const int32_t len = lengths ? std::min(T, std::max(0, lengths[i])) : T;
    int32_t ne = 0;
    for (int32_t t = 0; t < T; ++t) {
      int32_t tok = -1;
      if (t < len) {
        const int32_t p0 = prev[i];
        o->fused_step(0, logits + i * row_stride + (int64_t)t * frame_stride, blank_id, lambda, &states[i],
                      &prev[i], &tok);
        if (tok != blank_id && tok != p0) emitted[i * T + ne++] = tok;  // "blank ... and repeated tokens" collapse
      }
      frames[i * T + t] = tok;
    }
    emit_len[i] = ne;
  });
}

}  // extern "C"
