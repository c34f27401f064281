// lmgen — seeded synthetic token-level corpus -> interpolated Witten-Bell ARPA LM.
//
// INPUT GENERATOR ONLY. This file is shared input plumbing for both the oracle
// (oracle/) and the CUDA path (paper_2505_22857_b200/): it writes ARPA text and
// plain corpus files. It contains none of NGPU-LM's query arithmetic (no
// back-off walk, no Algorithm 1, no fusion); it only *estimates* an LM the way a
// toolkit would, so that the LM under test is (a) shaped like the paper's
// token-level BPE-1024 n-gram LMs (§3.1) and (b) exactly
// normalized per context, which the oracle pins rely on (SURVEY.md §8(d)
// "LM generator recipe"; SPEC.md:245-253 estimate_fixture).
//
// Estimator (interpolated Witten-Bell):
//   unigram  P(v)   = C(v) / (Ntok + u),  P(<unk>) = u / (Ntok + u)        (u = 1)
//   k >= 2   P(v|c) = (C(c,v) + T(c) * P(v|c[1:])) / (C(c) + T(c))
//   back-off alpha(c) = T(c) / (C(c) + T(c))
// where C(c) = sum_v C(c,v) over successors v (tokens and </s>) and T(c) the
// number of distinct successors. With these back-offs the ARPA back-off model
// reproduces the interpolated model exactly, so every context is normalized.
//
// Corpus source: word lexicon of W words with Zipf(1.07)
// frequencies; word length in tokens 1 + Poisson(0.9 ln(1 + rank/50)) clipped to
// [1,8]; tokens Zipf(0.9) over the V - absent usable ids (the last `absent` ids
// never occur, so M >= 1 vocabulary tokens need the normalized <unk> weight);
// word order from a sparse word-bigram chain (40 successors per word, Zipf(1.2)
// slot weights) mixed 70/30 with unigram draws; sentences have U[5,25) words.
//
// All randomness is splitmix64/xoshiro256** with hand-written samplers, so the
// output is bit-identical on every platform and libstdc++ version.
//
// Usage:
//   lmgen --arpa OUT --V 1024 --order 6 --tokens 430000 --seed 1
//         [--absent 1] [--lexicon 20000] [--minlen 5 --maxlen 25]
//         [--corpus-out FILE] [--heldout N --heldout-out FILE]
//         [--corpus-in FILE]   (use these sentences instead of sampling)
#include <algorithm>
#include <functional>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

namespace {

// ---------------------------------------------------------------- RNG
struct Rng {
  uint64_t s[4];
  static uint64_t splitmix(uint64_t& x) {
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  explicit Rng(uint64_t seed) {
    uint64_t x = seed;
    for (auto& v : s) v = splitmix(x);
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    uint64_t r = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t; s[3] = rotl(s[3], 45);
    return r;
  }
  double uniform() { return (next() >> 11) * (1.0 / 9007199254740992.0); }  // [0,1)
  int range(int lo, int hi) { return lo + (int)(uniform() * (hi - lo)); }  // [lo,hi)
  int poisson(double lam) {  // Knuth; lam is small (< 6)
    double L = std::exp(-lam), p = 1.0;
    int k = 0;
    do { ++k; p *= uniform(); } while (p > L);
    return k - 1;
  }
};

struct Zipf {  // P(rank r) ~ 1/(r+1)^a, r in [0,n)
  std::vector<double> cdf;
  Zipf(int n, double a) : cdf(n) {
    double acc = 0;
    for (int r = 0; r < n; ++r) { acc += 1.0 / std::pow(r + 1.0, a); cdf[r] = acc; }
    for (auto& c : cdf) c /= acc;
  }
  int sample(Rng& g) const {
    double u = g.uniform();
    int r = (int)(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
    return r < (int)cdf.size() ? r : (int)cdf.size() - 1;
  }
};

// ---------------------------------------------------------------- corpus
using Sentence = std::vector<int32_t>;

struct Source {
  std::vector<std::vector<int32_t>> words;  // token sequence per word
  std::vector<std::vector<int32_t>> succ;   // 40 successors per word
  Zipf word_zipf, slot_zipf;
  int minlen, maxlen;
  Source(int V_usable, int W, uint64_t seed, int minlen_, int maxlen_)
      : word_zipf(W, 1.07), slot_zipf(40, 1.2), minlen(minlen_), maxlen(maxlen_) {
    Rng g(seed ^ 0x5157A11CE5ull);
    Zipf tok_zipf(V_usable, 0.9);
    words.resize(W);
    for (int w = 0; w < W; ++w) {
      int len = 1 + g.poisson(0.9 * std::log(1.0 + w / 50.0));
      len = std::max(1, std::min(8, len));
      for (int i = 0; i < len; ++i) words[w].push_back(tok_zipf.sample(g));
    }
    succ.resize(W);
    for (int w = 0; w < W; ++w)
      for (int j = 0; j < 40; ++j) succ[w].push_back(word_zipf.sample(g));
  }
  Sentence sentence(Rng& g) const {
    int nw = g.range(minlen, maxlen);
    Sentence s;
    int w = word_zipf.sample(g);
    for (int i = 0; i < nw; ++i) {
      if (i > 0) w = (g.uniform() < 0.7) ? succ[w][slot_zipf.sample(g)] : word_zipf.sample(g);
      s.insert(s.end(), words[w].begin(), words[w].end());
    }
    return s;
  }
};

// ---------------------------------------------------------------- n-gram trie of counts
struct HashMap {  // open addressing u64 -> u32
  std::vector<uint64_t> keys;
  std::vector<uint32_t> vals;
  uint64_t mask = 0, size = 0;
  static constexpr uint64_t kEmpty = ~0ull;
  explicit HashMap(uint64_t cap_pow2 = 1u << 16) { reset(cap_pow2); }
  void reset(uint64_t cap) { keys.assign(cap, kEmpty); vals.assign(cap, 0); mask = cap - 1; size = 0; }
  static uint64_t h(uint64_t k) {
    k ^= k >> 33; k *= 0xff51afd7ed558ccdull; k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ull; k ^= k >> 33;
    return k;
  }
  uint32_t* find(uint64_t k) {
    for (uint64_t i = h(k) & mask;; i = (i + 1) & mask) {
      if (keys[i] == k) return &vals[i];
      if (keys[i] == kEmpty) return nullptr;
    }
  }
  void insert(uint64_t k, uint32_t v) {
    if ((size + 1) * 10 > (mask + 1) * 6) grow();
    for (uint64_t i = h(k) & mask;; i = (i + 1) & mask) {
      if (keys[i] == kEmpty) { keys[i] = k; vals[i] = v; ++size; return; }
      if (keys[i] == k) { vals[i] = v; return; }
    }
  }
  void grow() {
    std::vector<uint64_t> ok; std::vector<uint32_t> ov;
    ok.swap(keys); ov.swap(vals);
    reset((mask + 1) * 2);
    for (size_t i = 0; i < ok.size(); ++i)
      if (ok[i] != kEmpty) insert(ok[i], ov[i]);
  }
};

struct Trie {
  uint64_t radix;  // token ids in [0, radix)
  std::vector<uint32_t> parent, count, suf;
  std::vector<int32_t> tok;
  std::vector<uint8_t> depth;
  HashMap child;
  explicit Trie(uint64_t radix_) : radix(radix_) {
    parent.push_back(0); count.push_back(0); tok.push_back(-1); depth.push_back(0); suf.push_back(0);
  }
  uint64_t key(uint32_t p, int32_t t) const { return (uint64_t)p * radix + (uint64_t)t; }
  uint32_t get(uint32_t p, int32_t t) {
    uint32_t* f = child.find(key(p, t));
    return f ? *f : ~0u;
  }
  uint32_t get_or_add(uint32_t p, int32_t t) {
    uint32_t* f = child.find(key(p, t));
    if (f) return *f;
    uint32_t id = (uint32_t)parent.size();
    parent.push_back(p); count.push_back(0); tok.push_back(t); depth.push_back(depth[p] + 1); suf.push_back(0);
    child.insert(key(p, t), id);
    return id;
  }
};

void usage() {
  std::fprintf(stderr,
               "lmgen --arpa OUT --V V --order N (--tokens T | --corpus-in FILE) --seed S\n"
               "      [--absent A] [--lexicon W] [--minlen a --maxlen b] [--corpus-out F]\n"
               "      [--heldout H --heldout-out F]\n");
  std::exit(2);
}

}  // namespace

int main(int argc, char** argv) {
  std::string arpa_out, corpus_out, heldout_out, corpus_in;
  std::string prune_arg;  // "t1,t2,...": drop n-grams of order k with count <= t_k (k >= 2)
  int V = 0, order = 0, absent = 1, W = 20000, minlen = 5, maxlen = 25, heldout = 0;
  long long target_tokens = 0;
  uint64_t seed = 1;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    auto nxt = [&]() -> const char* { if (i + 1 >= argc) usage(); return argv[++i]; };
    if (a == "--arpa") arpa_out = nxt();
    else if (a == "--V") V = std::atoi(nxt());
    else if (a == "--order") order = std::atoi(nxt());
    else if (a == "--tokens") target_tokens = std::atoll(nxt());
    else if (a == "--seed") seed = std::strtoull(nxt(), nullptr, 10);
    else if (a == "--absent") absent = std::atoi(nxt());
    else if (a == "--lexicon") W = std::atoi(nxt());
    else if (a == "--minlen") minlen = std::atoi(nxt());
    else if (a == "--maxlen") maxlen = std::atoi(nxt());
    else if (a == "--corpus-out") corpus_out = nxt();
    else if (a == "--corpus-in") corpus_in = nxt();
    else if (a == "--heldout") heldout = std::atoi(nxt());
    else if (a == "--heldout-out") heldout_out = nxt();
    else if (a == "--prune") prune_arg = nxt();
    else usage();
  }
  if (arpa_out.empty() || V <= 0 || order <= 0 || (target_tokens <= 0 && corpus_in.empty())) usage();
  if (absent < 0 || absent >= V) { std::fprintf(stderr, "lmgen: need 0 <= absent < V\n"); return 2; }

  // ---- corpus
  std::vector<Sentence> corpus, held;
  if (!corpus_in.empty()) {
    FILE* f = std::fopen(corpus_in.c_str(), "r");
    if (!f) { std::perror(corpus_in.c_str()); return 2; }
    char line[1 << 16];
    while (std::fgets(line, sizeof line, f)) {
      Sentence s;
      for (char* p = std::strtok(line, " \t\r\n"); p; p = std::strtok(nullptr, " \t\r\n")) {
        int t = std::atoi(p);
        if (t < 0 || t >= V) { std::fprintf(stderr, "lmgen: token %d out of range\n", t); return 2; }
        s.push_back(t);
      }
      if (!s.empty()) corpus.push_back(s);
    }
    std::fclose(f);
  } else {
    Source src(V - absent, W, seed, minlen, maxlen);
    Rng g(seed);
    long long n = 0;
    while (n < target_tokens) { corpus.push_back(src.sentence(g)); n += (long long)corpus.back().size(); }
    Rng gh(seed * 0x100000001B3ull + 1000003ull);
    for (int i = 0; i < heldout; ++i) held.push_back(src.sentence(gh));
  }
  auto write_sents = [](const std::string& path, const std::vector<Sentence>& ss) {
    FILE* f = std::fopen(path.c_str(), "w");
    if (!f) { std::perror(path.c_str()); std::exit(2); }
    for (auto& s : ss) {
      for (size_t i = 0; i < s.size(); ++i) std::fprintf(f, i ? " %d" : "%d", s[i]);
      std::fputc('\n', f);
    }
    std::fclose(f);
  };
  if (!corpus_out.empty()) write_sents(corpus_out, corpus);
  if (!heldout_out.empty()) write_sents(heldout_out, held);

  // ---- count all windows of length <= order in "<s> w1 .. wn </s>"
  const int32_t BOS = V, EOS = V + 1;
  Trie tr((uint64_t)V + 3);
  std::vector<int32_t> pad;
  for (auto& s : corpus) {
    pad.assign(1, BOS);
    pad.insert(pad.end(), s.begin(), s.end());
    pad.push_back(EOS);
    for (size_t i = 0; i < pad.size(); ++i) {
      uint32_t node = 0;
      for (size_t k = i; k < pad.size() && (int)(k - i) < order; ++k) {
        node = tr.get_or_add(node, pad[k]);
        tr.count[node] += 1;
      }
    }
  }
  const size_t nn = tr.parent.size();
  // context statistics: C(c) = sum of successor counts, T(c) = #distinct successors
  std::vector<uint64_t> C(nn, 0);
  std::vector<uint32_t> T(nn, 0);
  for (size_t n = 1; n < nn; ++n) { C[tr.parent[n]] += tr.count[n]; T[tr.parent[n]] += 1; }
  uint64_t ntok = 0;  // predicted unigram events: every token and </s>, not <s>
  for (size_t n = 1; n < nn; ++n)
    if (tr.depth[n] == 1 && tr.tok[n] != BOS) ntok += tr.count[n];
  const double u = 1.0;

  // nodes bucketed by depth, lexicographic within depth (by parent rank, then token id)
  std::vector<std::vector<uint32_t>> byd(order + 1);
  for (size_t n = 1; n < nn; ++n) byd[tr.depth[n]].push_back((uint32_t)n);
  std::vector<uint32_t> rank(nn, 0);
  for (int d = 1; d <= order; ++d) {
    auto& v = byd[d];
    std::sort(v.begin(), v.end(), [&](uint32_t a, uint32_t b) {
      if (rank[tr.parent[a]] != rank[tr.parent[b]]) return rank[tr.parent[a]] < rank[tr.parent[b]];
      return tr.tok[a] < tr.tok[b];
    });
    for (size_t i = 0; i < v.size(); ++i) rank[v[i]] = (uint32_t)i;
  }
  // interpolated probabilities, increasing depth (suffix links first)
  std::vector<double> P(nn, 0.0);
  for (int d = 1; d <= order; ++d) {
    for (uint32_t n : byd[d]) {
      uint32_t p = tr.parent[n];
      if (d == 1) {
        tr.suf[n] = 0;
        P[n] = (double)tr.count[n] / ((double)ntok + u);
      } else {
        uint32_t s = tr.get(tr.suf[p], tr.tok[n]);  // suffix n-gram c[1:]+v is always observed
        if (s == ~0u) { std::fprintf(stderr, "lmgen: internal: missing suffix\n"); return 3; }
        tr.suf[n] = s;
        P[n] = ((double)tr.count[n] + (double)T[p] * P[s]) / ((double)C[p] + (double)T[p]);
      }
    }
  }

  // ---- optional count pruning (the paper's SPGI LM is pruned):
  // an n-gram of order k >= 2 is dropped when its count <= t_k, unless it is a
  // prefix of a kept n-gram (ARPA contexts must exist). Kept n-grams keep their
  // interpolated probability; back-off weights are renormalized so that every
  // context still sums to one:  bo(c) = (1 - sum_{kept v} P(v|c)) /
  // (1 - sum_{kept v} Pm(v|c[1:])), Pm = the pruned model's back-off
  // probability (a missing context contributes a weight of 1, i.e. log 0).
  // Thresholds that are not monotone (t_2 > t_3) leave kept n-grams whose
  // suffix was dropped: missing back-off contexts (R7/R8).
  std::vector<char> keep(nn, 1);
  std::vector<double> BO(nn, 0.0);  // natural back-off of kept contexts (probability ratio)
  bool pruned = false;
  if (!prune_arg.empty()) {
    std::vector<uint64_t> th(order + 1, 0);
    size_t pos = 0;
    for (int k = 1; k <= order && pos <= prune_arg.size(); ++k) {
      size_t e = prune_arg.find(',', pos);
      if (e == std::string::npos) e = prune_arg.size();
      th[k] = std::strtoull(prune_arg.substr(pos, e - pos).c_str(), nullptr, 10);
      pos = e + 1;
    }
    pruned = true;
    for (int d = order; d >= 2; --d)
      for (uint32_t n : byd[d]) {
        if (tr.count[n] <= th[d] && !keep[n]) continue;
        if (tr.count[n] <= th[d]) keep[n] = 0;
      }
    for (int d = order; d >= 2; --d)  // prefix closure
      for (uint32_t n : byd[d])
        if (keep[n]) keep[tr.parent[n]] = 1;
    // Pm(v | context node c): kept (c, v) -> P; else bo(c) * Pm(v | c[1:]); the
    // suffix context of a node is tr.suf (the node of context[1:], always observed)
    std::function<double(uint32_t, int32_t)> pm = [&](uint32_t c, int32_t v) -> double {
      const uint32_t x = tr.get(c, v);
      if (x != ~0u && keep[x]) return P[x];
      if (c == 0) return 0.0;  // (children of a context are observed unigrams: not reached)
      const double b = (keep[c] && BO[c] > 0) ? BO[c] : 1.0;
      return b * pm(tr.suf[c], v);
    };
    std::vector<std::vector<uint32_t>> kids(nn);
    for (size_t n = 1; n < nn; ++n) kids[tr.parent[n]].push_back((uint32_t)n);
    for (int d = 1; d < order; ++d)
      for (uint32_t c : byd[d]) {
        if (!keep[c]) continue;
        double num = 1.0, den = 1.0;
        bool any = false;
        for (uint32_t x : kids[c]) {
          if (!keep[x]) continue;
          any = true;
          num -= P[x];
          den -= pm(tr.suf[c], tr.tok[x]);
        }
        BO[c] = any ? (den > 1e-12 ? num / den : 1.0) : 1.0;
      }
  }

  // ---- write ARPA
  FILE* f = std::fopen(arpa_out.c_str(), "w");
  if (!f) { std::perror(arpa_out.c_str()); return 2; }
  std::vector<char> buf(1 << 24);
  std::setvbuf(f, buf.data(), _IOFBF, buf.size());
  auto tokstr = [&](int32_t t, char* out) {
    if (t == BOS) std::strcpy(out, "<s>");
    else if (t == EOS) std::strcpy(out, "</s>");
    else std::sprintf(out, "%d", t);
  };
  std::fprintf(f, "\\data\\\n");
  for (int d = 1; d <= order; ++d) {
    size_t cnt = 0;
    for (uint32_t n : byd[d]) cnt += keep[n] ? 1 : 0;
    std::fprintf(f, "ngram %d=%zu\n", d, cnt + (d == 1 ? 1 : 0));  // + <unk>
  }
  std::vector<int32_t> tup(order);
  char tb[32];
  for (int d = 1; d <= order; ++d) {
    std::fprintf(f, "\n\\%d-grams:\n", d);
    for (uint32_t n : byd[d]) {
      if (!keep[n]) continue;
      uint32_t x = n;
      for (int k = d - 1; k >= 0; --k) { tup[k] = tr.tok[x]; x = tr.parent[x]; }
      bool is_bos_unigram = (d == 1 && tr.tok[n] == BOS);
      if (is_bos_unigram) std::fprintf(f, "-99\t");
      else std::fprintf(f, "%.10g\t", std::log10(P[n]));
      for (int k = 0; k < d; ++k) { tokstr(tup[k], tb); std::fprintf(f, k ? " %s" : "%s", tb); }
      if (pruned) {
        if (d < order && BO[n] > 0 && BO[n] != 1.0) std::fprintf(f, "\t%.10g", std::log10(BO[n]));
      } else if (d < order && T[n] > 0) {
        std::fprintf(f, "\t%.10g", std::log10((double)T[n] / ((double)C[n] + (double)T[n])));
      }
      std::fputc('\n', f);
    }
    if (d == 1) std::fprintf(f, "%.10g\t<unk>\n", std::log10(u / ((double)ntok + u)));
  }
  std::fprintf(f, "\n\\end\\\n");
  std::fclose(f);

  size_t total = 0;
  for (int d = 1; d <= order; ++d) total += byd[d].size();
  std::fprintf(stderr, "lmgen: %zu sentences, %llu predicted unigram events, %zu n-grams (+<unk>)\n",
               corpus.size(), (unsigned long long)ntok, total);
  return 0;
}
