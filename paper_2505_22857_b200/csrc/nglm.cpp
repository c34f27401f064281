// NGLM binary model files (format at SPEC.md:209): a parsed,
// built model saved once and reloaded without the ARPA parse (a 20M n-gram
// ARPA takes tens of seconds to parse; its binary loads at disk speed).
//
// Layout (little-endian, version 1): "NGLM" magic (0x4E474C4D as the first
// four bytes 'N','G','L','M'), u32 version, u32 order, u32 vocab_size,
// u32 num_states, u64 num_arcs, u32 root_state, u32 bos_state; arrays
// arc_tokens u32[A], arc_weights f32[A], arc_to_states u32[A],
// start_arcs u64[S], end_arcs u64[S], boff_weights f32[S],
// boff_to_states u32[S], final_weights f32[S]; CRC-32 (IEEE, reflected
// 0xEDB88320) of every preceding byte, u32.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "ngpulm_internal.h"

namespace ngpulm {
namespace {

uint32_t crc_table[256];
bool crc_ready = false;

uint32_t crc32_update(uint32_t crc, const unsigned char* p, size_t n) {
  if (!crc_ready) {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      crc_table[i] = c;
    }
    crc_ready = true;
  }
  crc = ~crc;
  for (size_t i = 0; i < n; ++i) crc = crc_table[(crc ^ p[i]) & 0xff] ^ (crc >> 8);
  return ~crc;
}

struct Writer {
  std::vector<unsigned char> buf;
  template <class T>
  void put(const T& x) {
    const auto* p = reinterpret_cast<const unsigned char*>(&x);
    buf.insert(buf.end(), p, p + sizeof(T));
  }
  template <class T>
  void put_array(const T* a, size_t n) {
    const auto* p = reinterpret_cast<const unsigned char*>(a);
    buf.insert(buf.end(), p, p + n * sizeof(T));
  }
};

struct Reader {
  const unsigned char* p;
  size_t n, at = 0;
  bool get(void* dst, size_t bytes) {
    if (at + bytes > n) return false;
    std::memcpy(dst, p + at, bytes);
    at += bytes;
    return true;
  }
};

}  // namespace

int save_binary(const HostModel& m, const char* path, std::string& err) {
  const size_t S = (size_t)m.num_states, A = m.arc_tok.size();
  Writer w;
  w.buf.reserve(40 + A * 12 + S * 28 + 4);
  w.put_array("NGLM", 4);
  w.put<uint32_t>(1);
  w.put<uint32_t>((uint32_t)m.order);
  w.put<uint32_t>((uint32_t)m.V);
  w.put<uint32_t>((uint32_t)m.num_states);
  w.put<uint64_t>((uint64_t)A);
  w.put<uint32_t>(0);  // root_state
  w.put<uint32_t>((uint32_t)m.bos_state);
  w.put_array(m.arc_tok.data(), A);
  w.put_array(m.arc_w.data(), A);
  w.put_array(m.arc_to.data(), A);
  std::vector<uint64_t> se(S);
  for (size_t s = 0; s < S; ++s) se[s] = (uint64_t)m.arc_off[s];
  w.put_array(se.data(), S);
  for (size_t s = 0; s < S; ++s) se[s] = (uint64_t)m.arc_off[s + 1];
  w.put_array(se.data(), S);
  w.put_array(m.boff_w.data(), S);
  w.put_array(m.boff_to.data(), S);
  w.put_array(m.final_w.data(), S);
  const uint32_t crc = crc32_update(0, w.buf.data(), w.buf.size());
  w.put(crc);
  FILE* f = std::fopen(path, "wb");
  if (!f) { err = std::string("cannot open ") + path + " for writing"; return NGPULM_EIO; }
  const size_t wrote = std::fwrite(w.buf.data(), 1, w.buf.size(), f);
  const bool ok = std::fclose(f) == 0 && wrote == w.buf.size();
  if (!ok) { err = std::string("write failed: ") + path; return NGPULM_EIO; }
  return NGPULM_OK;
}

int load_binary(const char* path, HostModel& m, std::string& err) {
  auto fail = [&](int code, const std::string& msg) { err = msg; return code; };
  FILE* f = std::fopen(path, "rb");
  if (!f) return fail(NGPULM_EIO, std::string("cannot open ") + path);
  std::vector<unsigned char> buf;
  {
    unsigned char chunk[1 << 16];
    size_t k;
    while ((k = std::fread(chunk, 1, sizeof chunk, f)) > 0) buf.insert(buf.end(), chunk, chunk + k);
    std::fclose(f);
  }
  Reader r{buf.data(), buf.size()};
  char magic[4];
  if (!r.get(magic, 4) || std::memcmp(magic, "NGLM", 4) != 0) return fail(NGPULM_EDOMAIN, "NGLM: bad magic");
  uint32_t version = 0, order = 0, V = 0, S = 0, root = 0, bos = 0;
  uint64_t A = 0;
  if (!r.get(&version, 4)) return fail(NGPULM_EDOMAIN, "NGLM: truncated header");
  if (version != 1) return fail(NGPULM_EDOMAIN, "NGLM: unsupported version " + std::to_string(version));
  if (!r.get(&order, 4) || !r.get(&V, 4) || !r.get(&S, 4) || !r.get(&A, 8) || !r.get(&root, 4) || !r.get(&bos, 4))
    return fail(NGPULM_EDOMAIN, "NGLM: truncated header");
  const size_t need = 36 + A * 12 + (size_t)S * 28 + 4;
  if (buf.size() < need) return fail(NGPULM_EDOMAIN, "NGLM: truncated payload");
  if (buf.size() > need) return fail(NGPULM_EDOMAIN, "NGLM: trailing bytes after the checksum");
  uint32_t crc_file = 0;
  std::memcpy(&crc_file, buf.data() + need - 4, 4);
  if (crc32_update(0, buf.data(), need - 4) != crc_file) return fail(NGPULM_EDOMAIN, "NGLM: checksum mismatch");
  if (V == 0 || S == 0 || A < V || root != 0 || bos >= S || A > (uint64_t)INT32_MAX || S > (uint32_t)INT32_MAX ||
      order > NGPULM_MAX_ORDER)
    return fail(NGPULM_EDOMAIN, "NGLM: inconsistent header");
  m = HostModel();
  m.V = (int32_t)V;
  m.order = (int32_t)order;
  m.num_states = (int32_t)S;
  m.bos_state = (int32_t)bos;
  m.arc_tok.resize(A);
  m.arc_w.resize(A);
  m.arc_to.resize(A);
  r.get(m.arc_tok.data(), A * 4);
  r.get(m.arc_w.data(), A * 4);
  r.get(m.arc_to.data(), A * 4);
  std::vector<uint64_t> st(S), en(S);
  r.get(st.data(), (size_t)S * 8);
  r.get(en.data(), (size_t)S * 8);
  m.boff_w.resize(S);
  m.boff_to.resize(S);
  m.final_w.resize(S);
  r.get(m.boff_w.data(), (size_t)S * 4);
  r.get(m.boff_to.data(), (size_t)S * 4);
  r.get(m.final_w.data(), (size_t)S * 4);
  // arcs must be the CSR of states sorted by (from_state, token)
  m.arc_off.resize((size_t)S + 1);
  for (uint32_t s = 0; s < S; ++s) {
    if (st[s] != (s == 0 ? 0 : en[s - 1]) || en[s] < st[s] || en[s] > A)
      return fail(NGPULM_EDOMAIN, "NGLM: arc ranges are not contiguous in state order");
    m.arc_off[s] = (int32_t)st[s];
  }
  m.arc_off[S] = (int32_t)en[S - 1];
  if ((uint64_t)m.arc_off[S] != A || m.arc_off[1] != (int32_t)V)
    return fail(NGPULM_EDOMAIN, "NGLM: the root must own exactly arcs [0, V)");
  for (uint64_t a = 0; a < A; ++a)
    if (m.arc_tok[a] < 0 || m.arc_tok[a] >= (int32_t)V || m.arc_to[a] < 0 || m.arc_to[a] >= (int32_t)S)
      return fail(NGPULM_EDOMAIN, "NGLM: arc token or target out of range");
  for (uint32_t s = 0; s < S; ++s)
    if (m.boff_to[s] < 0 || m.boff_to[s] >= (int32_t)S) return fail(NGPULM_EDOMAIN, "NGLM: back-off target out of range");
  // the ARPA-time counters are not part of the format: M is recomputed from
  // the root arcs when N >= 2, the dropped-n-gram count is unknown (-1)
  m.num_unk_filled = -1;
  m.num_dropped = -1;
  std::string e2;
  if (!rebuild_child_map(m, e2)) return fail(NGPULM_EDOMAIN, "NGLM: " + e2);
  return NGPULM_OK;
}

}  // namespace ngpulm
