// Host side of libngpulm: ARPA parsing, validation and flat-trie construction.
//
// Off the hot path (SURVEY.md §3 call stack 1). Produces the tensors of
// PAPER.md:114-122 (§2.2): arcs sorted by (from_state, token) with per-state
// ranges, back-off targets/weights, the root state filled to all V tokens with
// the normalized <unk> weight, and final weights precomputed by walking
// back-offs. Readings of the paper: DESIGN.md R1-R20.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <unordered_map>
#include <vector>

#include "ngpulm_internal.h"

namespace ngpulm {
namespace {

constexpr uint64_t kEmpty = ~0ull;
constexpr double kLn10 = 2.302585092994045684;

uint64_t hmix(uint64_t k) {
  k ^= k >> 33; k *= 0xff51afd7ed558ccdull; k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ull; k ^= k >> 33;
  return k;
}
uint64_t ckey(int32_t parent, int32_t tok) { return ((uint64_t)(uint32_t)parent << 32) | (uint32_t)tok; }

void child_insert(HostModel& m, uint64_t key, int32_t val) {
  if ((uint64_t)(m.num_states + 1) * 10 > (m.child_mask + 1) * 6 || m.child_keys.empty()) {
    uint64_t cap = m.child_keys.empty() ? 1024 : (m.child_mask + 1) * 2;
    std::vector<uint64_t> ok; std::vector<int32_t> ov;
    ok.swap(m.child_keys); ov.swap(m.child_vals);
    m.child_keys.assign(cap, kEmpty); m.child_vals.assign(cap, -1); m.child_mask = cap - 1;
    for (size_t i = 0; i < ok.size(); ++i) {
      if (ok[i] == kEmpty) continue;
      uint64_t j = hmix(ok[i]) & m.child_mask;
      while (m.child_keys[j] != kEmpty) j = (j + 1) & m.child_mask;
      m.child_keys[j] = ok[i]; m.child_vals[j] = ov[i];
    }
  }
  uint64_t j = hmix(key) & m.child_mask;
  while (m.child_keys[j] != kEmpty) j = (j + 1) & m.child_mask;
  m.child_keys[j] = key; m.child_vals[j] = val;
}

// [R1] log10 -> ln (one double multiply, one rounding); [R3] -99 -> -1e30
double ln64(double log10v) { return log10v <= -99.0 ? -1e30 : log10v * kLn10; }
float ln32(double log10v) { return (float)ln64(log10v); }

struct Pending { int32_t parent, tok; float bo; };
struct Arc { int32_t from, tok; float w; int32_t to; };  // to: state, or -(pending+3), or -2

}  // namespace

int32_t HostModel::child(int32_t parent, int32_t tok) const {
  if (child_keys.empty()) return -1;
  uint64_t key = ckey(parent, tok);
  for (uint64_t i = hmix(key) & child_mask;; i = (i + 1) & child_mask) {
    if (child_keys[i] == key) return child_vals[i];
    if (child_keys[i] == kEmpty) return -1;
  }
}

int build_from_arpa(const char* arpa_path, const char* vocab_path, int32_t V, HostModel& m,
                    std::string& err) {
  auto fail = [&](int code, const std::string& msg) { err = msg; return code; };
  // ---------------------------------------------------------------- vocabulary
  std::unordered_map<std::string, int32_t> vocab;
  if (vocab_path) {
    FILE* vf = std::fopen(vocab_path, "r");
    if (!vf) return fail(NGPULM_EIO, std::string("cannot open vocabulary ") + vocab_path);
    char line[4096];
    int32_t id = 0;
    while (std::fgets(line, sizeof line, vf)) {
      size_t n = std::strlen(line);
      while (n && (line[n - 1] == '\n' || line[n - 1] == '\r' || line[n - 1] == ' ')) line[--n] = 0;
      std::string w(line, n);
      if (w == "<s>" || w == "</s>" || w == "<unk>")
        { std::fclose(vf); return fail(NGPULM_EDOMAIN, "vocabulary contains reserved token " + w); }
      if (!vocab.emplace(w, id).second)
        { std::fclose(vf); return fail(NGPULM_EDOMAIN, "duplicate vocabulary token " + w); }
      ++id;
    }
    std::fclose(vf);
    if (V > 0 && V != id) return fail(NGPULM_EUSAGE, "vocab_size does not match the vocabulary file");
    V = id;
  }
  if (V <= 0) return fail(NGPULM_EUSAGE, "vocab_size must be > 0 without a vocabulary file");
  const int32_t BOS = V, EOS = V + 1, UNK = V + 2;
  m = HostModel();
  m.V = V;

  // ---------------------------------------------------------------- read file
  std::vector<char> buf;
  {
    FILE* f = std::fopen(arpa_path, "rb");
    if (!f) return fail(NGPULM_EIO, std::string("cannot open ") + arpa_path + ": " + std::strerror(errno));
    std::fseek(f, 0, SEEK_END);
    long sz = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    buf.resize((size_t)sz + 1);
    if (sz > 0 && std::fread(buf.data(), 1, (size_t)sz, f) != (size_t)sz)
      { std::fclose(f); return fail(NGPULM_EIO, "short read"); }
    std::fclose(f);
    buf[(size_t)sz] = 0;
  }

  auto map_token = [&](const char* a, const char* b) -> int32_t {
    size_t n = (size_t)(b - a);
    if (n == 3 && !std::memcmp(a, "<s>", 3)) return BOS;
    if (n == 4 && !std::memcmp(a, "</s>", 4)) return EOS;
    if (n == 5 && !std::memcmp(a, "<unk>", 5)) return UNK;
    if (!vocab_path) {  // canonical decimal ids only
      if (n == 0 || n > 10 || (n > 1 && a[0] == '0')) return -1;
      int64_t x = 0;
      for (const char* p = a; p < b; ++p) {
        if (*p < '0' || *p > '9') return -1;
        x = x * 10 + (*p - '0');
      }
      return x < V ? (int32_t)x : -1;
    }
    auto it = vocab.find(std::string(a, n));
    return it == vocab.end() ? -1 : it->second;
  };

  // ---------------------------------------------------------------- parse + build
  std::vector<int64_t> declared;  // declared[k]
  std::vector<int64_t> seen;
  std::vector<uint8_t> has_uni(V, 0);
  std::vector<float> uni_w(V, 0.f);
  bool has_unk = false;
  double unk_log10 = 0;
  // per-state data by final id (root = 0)
  std::vector<int32_t> st_parent{-1}, st_tok{-1};
  std::vector<float> st_bo{0.f};
  std::vector<float> fin{0.f};
  std::vector<uint8_t> has_fin{0};
  m.num_states = 1;
  std::vector<Arc> arcs;
  std::vector<Pending> pend;
  std::vector<size_t> pend_arc;  // index of the arc created with each pending state (k>=2)
  int N = 0;
  int section = -1;  // -1 before \data\, 0 header, k = \k-grams:
  int last_section = 0;
  bool ended = false;
  // context cache: tokens and resolved states of the previous line's context
  std::vector<int32_t> cache_tok, cache_st;

  auto finish_section = [&](int k) -> int {
    // [R6] ids of this order's states: sorted by (parent id, token), which is
    // the lexicographic order of the token tuples because parents are sorted.
    std::vector<int32_t> idx(pend.size());
    std::iota(idx.begin(), idx.end(), 0);
    std::sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) {
      if (pend[a].parent != pend[b].parent) return pend[a].parent < pend[b].parent;
      return pend[a].tok < pend[b].tok;
    });
    std::vector<int32_t> id_of(pend.size());
    for (size_t i = 0; i < idx.size(); ++i) {
      const Pending& p = pend[idx[i]];
      if (i > 0 && pend[idx[i - 1]].parent == p.parent && pend[idx[i - 1]].tok == p.tok)
        return fail(NGPULM_EDOMAIN, "duplicate " + std::to_string(k) + "-gram");
      int32_t id = m.num_states++;
      id_of[idx[i]] = id;
      st_parent.push_back(p.parent); st_tok.push_back(p.tok); st_bo.push_back(p.bo);
      fin.push_back(0.f); has_fin.push_back(0);
      child_insert(m, ckey(p.parent, p.tok), id);
    }
    for (size_t i = 0; i < pend_arc.size(); ++i)
      if (pend_arc[i] != (size_t)-1) arcs[pend_arc[i]].to = id_of[i];
    pend.clear(); pend_arc.clear();
    return NGPULM_OK;
  };

  long long lineno = 0;
  const char* p = buf.data();
  const char* end = buf.data() + buf.size() - 1;
  while (p < end && !ended) {
    const char* ls = p;
    const char* le = (const char*)std::memchr(p, '\n', (size_t)(end - p));
    if (!le) le = end;
    p = le + 1;
    ++lineno;
    const char* e = le;
    while (e > ls && (e[-1] == '\r' || e[-1] == ' ' || e[-1] == '\t')) --e;
    const char* s = ls;
    while (s < e && (*s == ' ' || *s == '\t')) ++s;
    if (s == e) continue;
    std::string where = " (line " + std::to_string(lineno) + ")";
    if (*s == '\\') {
      std::string tag(s, e);
      if (tag == "\\data\\") { section = 0; continue; }
      if (section < 0) continue;
      if (tag == "\\end\\") {
        if (last_section > 0) { int r = finish_section(last_section); if (r) return r; }
        ended = true;
        continue;
      }
      int k = 0;
      if (std::sscanf(tag.c_str(), "\\%d-grams:", &k) != 1) return fail(NGPULM_EDOMAIN, "bad section header " + tag + where);
      if (k != last_section + 1) return fail(NGPULM_EDOMAIN, "n-gram sections out of order" + where);
      if (last_section > 0) { int r = finish_section(last_section); if (r) return r; }
      if (k == 1) {
        N = 0;
        for (size_t j = 1; j < declared.size(); ++j) if (declared[j] > 0) N = (int)j;  // [R5'] order
        if (N <= 0) return fail(NGPULM_EDOMAIN, "no n-grams declared");
        if (N > NGPULM_MAX_ORDER) return fail(NGPULM_EDOMAIN, "order above NGPULM_MAX_ORDER");
        m.order = N;
        seen.assign(declared.size(), 0);
      }
      if (k >= (int)declared.size()) return fail(NGPULM_EDOMAIN, "section not declared in \\data\\" + where);
      section = last_section = k;
      cache_tok.clear(); cache_st.clear();
      continue;
    }
    if (section < 0) continue;  // text before \data\ is ignored
    if (section == 0) {
      int k = 0; long long n = 0;
      if (std::sscanf(std::string(s, e).c_str(), "ngram %d=%lld", &k, &n) != 2 || k <= 0 || n < 0)
        return fail(NGPULM_EDOMAIN, "bad \\data\\ line" + where);
      if ((int)declared.size() <= k) declared.resize(k + 1, 0);
      declared[k] = n;
      continue;
    }
    const int k = section;
    // a section above the order N is declared empty (N = highest non-empty order,
    // <= NGPULM_MAX_ORDER): any line in it is a count mismatch, rejected before
    // its tokens are read into toks[NGPULM_MAX_ORDER]
    if (k > N) return fail(NGPULM_EDOMAIN, "n-gram in a section declared empty in \\data\\" + where);
    // ---- one n-gram line: log10p tokens... [log10bo]
    char* q = nullptr;
    double lp = std::strtod(s, &q);
    if (q == s) return fail(NGPULM_EDOMAIN, "malformed n-gram line" + where);
    const char* c = q;
    int32_t toks[NGPULM_MAX_ORDER];
    for (int i = 0; i < k; ++i) {
      while (c < e && (*c == ' ' || *c == '\t')) ++c;
      const char* a = c;
      while (c < e && *c != ' ' && *c != '\t') ++c;
      if (a == c) return fail(NGPULM_EDOMAIN, "malformed n-gram line (too few tokens)" + where);
      toks[i] = map_token(a, c);
      if (toks[i] < 0) return fail(NGPULM_EDOMAIN, "token '" + std::string(a, c) + "' not in vocabulary" + where);
    }
    while (c < e && (*c == ' ' || *c == '\t')) ++c;
    bool has_bo = false;
    double bo = 0;
    if (c < e) {
      bo = std::strtod(c, &q);
      if (q == c) return fail(NGPULM_EDOMAIN, "malformed back-off field" + where);
      has_bo = true;
      c = q;
      while (c < e && (*c == ' ' || *c == '\t')) ++c;
      if (c != e) return fail(NGPULM_EDOMAIN, "malformed n-gram line (extra fields)" + where);
    }
    seen[k] += 1;
    const float w32 = ln32(lp), bo32 = has_bo ? ln32(bo) : 0.0f;
    const int32_t last = toks[k - 1];
    // validation of meta tokens
    bool dropped = false;
    for (int i = 0; i < k; ++i) {
      if (toks[i] == BOS && i > 0) return fail(NGPULM_EDOMAIN, "n-gram predicts <s>" + where);
      if (toks[i] == EOS && i < k - 1) return fail(NGPULM_EDOMAIN, "</s> inside an n-gram context" + where);
      if (toks[i] == UNK && !(k == 1)) dropped = true;
    }
    if (dropped) { ++m.num_dropped; continue; }  // [R5] unreachable
    if (k == 1) {
      if (last == UNK) { has_unk = true; unk_log10 = lp; continue; }
      if (last == EOS) {
        if (has_fin[0]) return fail(NGPULM_EDOMAIN, "duplicate </s> unigram" + where);
        has_fin[0] = 1; fin[0] = w32;
        continue;
      }
      if (last == BOS) {  // [R4] probability discarded, back-off kept
        if (N > 1) { pend.push_back({0, BOS, bo32}); pend_arc.push_back((size_t)-1); }
        continue;
      }
      if (has_uni[last]) return fail(NGPULM_EDOMAIN, "duplicate unigram" + where);
      has_uni[last] = 1; uni_w[last] = w32;
      if (N > 1) { pend.push_back({0, last, bo32}); pend_arc.push_back((size_t)-1); }
      continue;
    }
    // context state: walk the prefix edges (cached from the previous line)
    int32_t ctx = 0;
    {
      size_t common = 0;
      while (common < cache_tok.size() && common < (size_t)(k - 1) && cache_tok[common] == toks[common]) ++common;
      cache_tok.resize(common); cache_st.resize(common);
      ctx = common ? cache_st[common - 1] : 0;
      for (int i = (int)common; i < k - 1; ++i) {
        ctx = m.child(ctx, toks[i]);
        if (ctx < 0) return fail(NGPULM_EDOMAIN, "context of n-gram is not an n-gram (ARPA not prefix-closed)" + where);
        cache_tok.push_back(toks[i]); cache_st.push_back(ctx);
      }
    }
    if (last == EOS) {  // final-weight carrier
      if (has_fin[ctx]) return fail(NGPULM_EDOMAIN, "duplicate n-gram" + where);
      has_fin[ctx] = 1; fin[ctx] = w32;
      continue;
    }
    if (!has_uni[last]) return fail(NGPULM_EDOMAIN, "token without a unigram" + where);
    if (k < N) {
      pend.push_back({ctx, last, bo32});
      pend_arc.push_back(arcs.size());
      arcs.push_back({ctx, last, w32, -1});
    } else {
      arcs.push_back({ctx, last, w32, -2});  // highest order: target resolved below
    }
  }
  if (!ended) return fail(NGPULM_EDOMAIN, "missing \\end\\");
  if (section < 0) return fail(NGPULM_EDOMAIN, "missing \\data\\");
  for (size_t k = 1; k < declared.size(); ++k)
    if (k < seen.size() && seen[k] != declared[k])
      return fail(NGPULM_EDOMAIN, "count mismatch for order " + std::to_string(k) + ": declared " +
                  std::to_string(declared[k]) + ", found " + std::to_string(seen[k]));
  if (last_section < N) return fail(NGPULM_EDOMAIN, "missing n-gram section");
  if (!has_fin[0]) return fail(NGPULM_EDOMAIN, "missing </s> unigram");

  const int32_t S = m.num_states;
  // ---- [R2] normalized <unk> for the M vocabulary tokens without a unigram
  int64_t M = 0;
  for (int32_t v = 0; v < V; ++v) M += !has_uni[v];
  m.num_unk_filled = M;
  if (M > 0 && !has_unk) return fail(NGPULM_EDOMAIN, "<unk> unigram missing but some vocabulary tokens lack a unigram");
  const float w_unk = M > 0 ? (float)(ln64(unk_log10) - std::log((double)M)) : 0.0f;
  { int32_t b = m.child(0, BOS); m.bos_state = b >= 0 ? b : 0; }

  // ---- [R8] back-off target: longest proper suffix state, via the parent's chain
  m.boff_to.assign(S, 0);
  m.boff_w.assign(S, 0.f);
  for (int32_t s = 1; s < S; ++s) {
    m.boff_w[s] = st_bo[s];
    int32_t par = st_parent[s], t = st_tok[s];
    if (par == 0) { m.boff_to[s] = 0; continue; }
    for (int32_t x = m.boff_to[par];; x = m.boff_to[x]) {
      int32_t y = m.child(x, t);
      if (y >= 0) { m.boff_to[s] = y; break; }
      if (x == 0) { m.boff_to[s] = 0; break; }
    }
  }
  // ---- [R7] highest-order arcs point to the longest proper suffix state of c+v
  for (Arc& a : arcs) {
    if (a.to != -2) continue;
    for (int32_t x = m.boff_to[a.from];; x = m.boff_to[x]) {
      int32_t y = m.child(x, a.tok);
      if (y >= 0) { a.to = y; break; }
      if (x == 0) { a.to = 0; break; }
    }
  }
  // ---- CSR: root owns [0, V), then states in id order, tokens sorted
  m.arc_off.assign((size_t)S + 1, 0);
  std::vector<int64_t> cnt(S, 0);
  cnt[0] = V;
  for (const Arc& a : arcs) cnt[a.from] += 1;
  int64_t A = 0;
  for (int32_t s = 0; s < S; ++s) {
    if (A > INT32_MAX) return fail(NGPULM_EDOMAIN, "more than 2^31 arcs");
    m.arc_off[s] = (int32_t)A;
    A += cnt[s];
  }
  if (A > INT32_MAX) return fail(NGPULM_EDOMAIN, "more than 2^31 arcs");
  m.arc_off[S] = (int32_t)A;
  m.arc_tok.assign((size_t)A, 0); m.arc_w.assign((size_t)A, 0.f); m.arc_to.assign((size_t)A, 0);
  for (int32_t v = 0; v < V; ++v) {
    m.arc_tok[v] = v;
    if (has_uni[v]) {
      m.arc_w[v] = uni_w[v];
      int32_t y = m.child(0, v);
      m.arc_to[v] = y >= 0 ? y : 0;
    } else {
      m.arc_w[v] = w_unk;
      m.arc_to[v] = 0;
    }
  }
  {
    std::vector<int64_t> pos(m.arc_off.begin(), m.arc_off.end() - 1);
    pos[0] = V;
    for (const Arc& a : arcs) {
      int64_t i = pos[a.from]++;
      m.arc_tok[i] = a.tok; m.arc_w[i] = a.w; m.arc_to[i] = a.to;
    }
    std::vector<Arc>().swap(arcs);
    std::vector<int64_t> perm;
    for (int32_t s = 1; s < S; ++s) {
      int64_t b = m.arc_off[s], e = m.arc_off[s + 1];
      if (e - b < 2) continue;
      bool sorted = true;
      for (int64_t i = b + 1; i < e; ++i) if (m.arc_tok[i] <= m.arc_tok[i - 1]) { sorted = false; break; }
      if (sorted) continue;
      perm.resize(e - b);
      std::iota(perm.begin(), perm.end(), b);
      std::sort(perm.begin(), perm.end(), [&](int64_t x, int64_t y) { return m.arc_tok[x] < m.arc_tok[y]; });
      std::vector<int32_t> t2(e - b), to2(e - b);
      std::vector<float> w2(e - b);
      for (int64_t i = 0; i < e - b; ++i) { t2[i] = m.arc_tok[perm[i]]; w2[i] = m.arc_w[perm[i]]; to2[i] = m.arc_to[perm[i]]; }
      for (int64_t i = 0; i < e - b; ++i) {
        if (i > 0 && t2[i] == t2[i - 1]) return fail(NGPULM_EDOMAIN, "duplicate " + std::to_string(N) + "-gram");
        m.arc_tok[b + i] = t2[i]; m.arc_w[b + i] = w2[i]; m.arc_to[b + i] = to2[i];
      }
    }
  }
  // ---- [R9] finals: Algorithm-1 order walk of the back-off chain
  m.final_w.assign(S, 0.f);
  for (int32_t s = 0; s < S; ++s) {
    float acc = 0.0f;
    int32_t x = s;
    for (int it = 0; it <= N + 1; ++it) {
      if (has_fin[x]) { m.final_w[s] = acc + fin[x]; break; }
      acc = acc + m.boff_w[x];
      x = m.boff_to[x];
    }
  }
  return NGPULM_OK;
}

size_t device_arc_layout(const HostModel& m, std::vector<int32_t>& arc_begin) {
  const int32_t S = m.num_states;
  arc_begin.assign((size_t)S, 0);
  size_t cur = 0;
  for (int32_t s = 0; s < S; ++s) {
    arc_begin[(size_t)s] = (int32_t)cur;
    cur = (cur + (size_t)(m.arc_off[s + 1] - m.arc_off[s]) + 3) & ~(size_t)3;
  }
  return cur;
}

int32_t packed_token_bits(int32_t V) {
  int32_t b = 1;
  while ((int64_t)1 << b < (int64_t)V) ++b;
  return b;
}

bool packable(const HostModel& m) {
  const int32_t b = packed_token_bits(m.V);
  return b < 32 && (int64_t)m.num_states <= ((int64_t)1 << (32 - b));
}

void build_chain_table(const HostModel& m, const std::vector<int32_t>& arc_begin, std::vector<int32_t>& out,
                       int32_t& slots) {
  slots = std::max(1, m.order);
  const int32_t S = m.num_states;
  out.assign((size_t)S * slots * 4, 0);
  for (int32_t s = 0; s < S; ++s) {
    int32_t* rec = out.data() + (size_t)s * slots * 4;
    float acc = 0.0f;
    int32_t n = 0, pre = 0, x = s;
    for (int it = 0; it < slots && x != 0; ++it) {  // Algorithm 1 lines 72-82, at load time
      const int32_t cnt = m.arc_off[x + 1] - m.arc_off[x];
      if (cnt > 0 && n + 1 < slots) {
        int32_t* lv = rec + (size_t)(n + 1) * 4;
        lv[0] = arc_begin[x];
        lv[1] = pre;
        std::memcpy(&lv[2], &acc, 4);
        pre += cnt;
        ++n;
      }
      acc = acc + m.boff_w[x];
      x = m.boff_to[x];
    }
    // field 3 of a level: (first slot << 16) | quads, for the one-warp-per-row
    // kernel: level i covers the 16-byte quads [begin/4, (begin+count-1)/4],
    // cut into slots of 32 quads; slots are numbered from the last level.
    for (int32_t i = n - 1, start = 0; i >= 0; --i) {
      int32_t* lv = rec + (size_t)(i + 1) * 4;
      const int32_t b = lv[0], cnt = (i + 1 < n ? lv[4 + 1] : pre) - lv[1];
      const int32_t nq = ((b + cnt - 1) >> 2) - (b >> 2) + 1;
      lv[3] = (start << 16) | nq;
      start += (nq + 31) >> 5;
    }
    rec[0] = n;
    std::memcpy(&rec[1], &acc, 4);
    std::memcpy(&rec[2], &m.final_w[s], 4);
    rec[3] = pre;
    for (int32_t i = n + 1; i < slots; ++i) rec[(size_t)i * 4 + 1] = pre;
  }
}

void build_row_bounds(const HostModel& m, std::vector<float>& ub) {
  const int32_t S = m.num_states;
  std::vector<float> maxw((size_t)S, -INFINITY);
  for (int32_t s = 0; s < S; ++s)
    for (int32_t a = m.arc_off[s]; a < m.arc_off[s + 1]; ++a) maxw[s] = std::max(maxw[s], m.arc_w[a]);
  ub.assign((size_t)S, -INFINITY);
  const int32_t cap = std::max(1, m.order);
  for (int32_t s = 0; s < S; ++s) {  // the chain of build_chain_table, Algorithm 1 order
    float acc = 0.0f, u = -INFINITY;
    int32_t x = s;
    for (int it = 0; it < cap && x != 0; ++it) {
      if (m.arc_off[x + 1] > m.arc_off[x]) u = std::max(u, acc + maxw[x]);
      acc = acc + m.boff_w[x];
      x = m.boff_to[x];
    }
    ub[s] = std::max(u, acc + maxw[0]);  // the root level
  }
}

// The context trie's prefix edges (state_of) from the flat arrays alone, for
// models loaded from NGLM files: state ids are ordered by context length
// (R6), so walking states in id order, an arc (s, v) whose target has no
// length yet reaches the state of context(s)+v — its child (a target of
// length <= |context(s)| was reached before). <s> is the root's child V.
bool rebuild_child_map(HostModel& m, std::string& err) {
  const int32_t S = m.num_states, V = m.V;
  std::vector<int32_t> len((size_t)S, -1);
  m.child_keys.clear();
  m.child_vals.clear();
  m.child_mask = 0;
  len[0] = 0;
  if (m.bos_state != 0) {
    len[(size_t)m.bos_state] = 1;
    child_insert(m, ckey(0, V), m.bos_state);
  }
  for (int32_t s = 0; s < S; ++s) {
    if (len[(size_t)s] < 0) { err = "state " + std::to_string(s) + " is not reachable by a prefix arc"; return false; }
    for (int32_t a = m.arc_off[s]; a < m.arc_off[s + 1]; ++a) {
      const int32_t t = m.arc_to[a];
      if (t != 0 && len[(size_t)t] < 0) {
        len[(size_t)t] = len[(size_t)s] + 1;
        child_insert(m, ckey(s, m.arc_tok[a]), t);
      }
    }
  }
  if (m.order >= 2) {  // root arcs that fall back to the root: tokens without a unigram (R2)
    int64_t M = 0;
    for (int32_t v = 0; v < V; ++v) M += m.arc_to[v] == 0;
    m.num_unk_filled = M;
  }
  return true;
}

}  // namespace ngpulm
