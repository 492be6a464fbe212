// Host text front-end of Engine.translate_corpus (engine.py:144-164 in the
// reference: preprocess -> whitespace split -> Vocabulary lookup with <unk>
// and an OOV count), native: one call maps a whole corpus's UTF-8 lines to
// the concatenated id array the decoder takes, instead of a Python split
// and a dict lookup per token.  Lowercasing stays on the Python side
// (str.lower(), exact Unicode semantics); this code splits exactly like
// Python's str.split() (every code point Py_UNICODE_ISSPACE accepts) and
// looks tokens up by their UTF-8 bytes.  Host-only code (no device work).
#include <cstdint>
#include <cstring>
#include <string>
#include <algorithm>
#include <functional>
#include <thread>
#include <vector>

#include "../../include/amun_b200.h"
#include "common.cuh"

// Open-addressing hash table over the token bytes (power-of-two slots,
// linear probing, load <= 1/2): one cache line per probe instead of a
// node-based map's pointer chase.
struct amun_vocab {
  std::string bytes;                // every token's UTF-8 bytes back to back
  std::vector<int64_t> off;         // token i = bytes[off[i], off[i+1])
  std::vector<int32_t> slot;        // token id or -1
  std::vector<uint32_t> slot_hash;  // the slot's hash (fast reject)
  uint32_t mask = 0;
};

void amun_set_last_error(const std::string &m);  // api.cu: the thread's amun_last_error() text

namespace {

// Python str.isspace / str.split() whitespace (Py_UNICODE_ISSPACE)
inline bool py_space(uint32_t c) {
  if (c < 0x80) return (c >= 0x09 && c <= 0x0D) || (c >= 0x1C && c <= 0x20);
  return c == 0x85 || c == 0xA0 || c == 0x1680 || (c >= 0x2000 && c <= 0x200A) || c == 0x2028 || c == 0x2029 ||
         c == 0x202F || c == 0x205F || c == 0x3000;
}

// code point starting at p (< end) and its byte length; malformed bytes
// decode as themselves (never whitespace)
inline uint32_t utf8_at(const unsigned char *p, const unsigned char *end, int *n) {
  const unsigned char c = p[0];
  if (c < 0x80) {
    *n = 1;
    return c;
  }
  const int len = c >= 0xF0 ? 4 : c >= 0xE0 ? 3 : c >= 0xC0 ? 2 : 1;
  if (len == 1 || p + len > end) {
    *n = 1;
    return 0xFFFFFFFFu;
  }
  uint32_t v = c & (0xFF >> (len + 1));
  for (int i = 1; i < len; ++i) v = (v << 6) | (p[i] & 0x3F);
  *n = len;
  return v;
}

inline uint32_t hash_bytes(const unsigned char *p, size_t n) {  // FNV-1a
  uint32_t h = 2166136261u;
  for (size_t i = 0; i < n; ++i) h = (h ^ p[i]) * 16777619u;
  return h ^ (h >> 15);
}

// id of token bytes [p, p + n), or -1
inline int32_t vocab_find(const amun_vocab &v, const unsigned char *p, size_t n) {
  const uint32_t h = hash_bytes(p, n);
  for (uint32_t s = h & v.mask;; s = (s + 1) & v.mask) {
    const int32_t id = v.slot[s];
    if (id < 0) return -1;
    if (v.slot_hash[s] == h && (size_t)(v.off[id + 1] - v.off[id]) == n &&
        std::memcmp(v.bytes.data() + v.off[id], p, n) == 0)
      return id;
  }
}

}  // namespace

extern "C" int amun_vocab_create(const char *bytes, const int64_t *offsets, int32_t n_tokens, amun_vocab **out) {
  try {
    if (!out || n_tokens < 0 || (n_tokens > 0 && (!bytes || !offsets))) {
      amun_set_last_error("amun_vocab_create: null argument");
      return AMUN_ERR_INVALID;
    }
    auto *v = new amun_vocab();
    const int64_t total = n_tokens ? offsets[n_tokens] - offsets[0] : 0;
    v->bytes.assign(n_tokens ? bytes + offsets[0] : "", (size_t)total);
    v->off.resize((size_t)n_tokens + 1);
    for (int32_t i = 0; i <= n_tokens; ++i) v->off[i] = n_tokens ? offsets[i] - offsets[0] : 0;
    size_t cap = 16;
    while (cap < 2 * (size_t)n_tokens) cap *= 2;
    v->slot.assign(cap, -1);
    v->slot_hash.assign(cap, 0);
    v->mask = (uint32_t)(cap - 1);
    const auto *b = reinterpret_cast<const unsigned char *>(v->bytes.data());
    for (int32_t i = 0; i < n_tokens; ++i) {
      const size_t n = (size_t)(v->off[i + 1] - v->off[i]);
      if (vocab_find(*v, b + v->off[i], n) >= 0) {
        amun_set_last_error("vocabulary contains duplicate tokens");
        delete v;
        return AMUN_ERR_INVALID;
      }
      const uint32_t h = hash_bytes(b + v->off[i], n);
      uint32_t s = h & v->mask;
      while (v->slot[s] >= 0) s = (s + 1) & v->mask;
      v->slot[s] = i;
      v->slot_hash[s] = h;
    }
    *out = v;
    return AMUN_OK;
  } catch (const std::exception &e) {
    amun_set_last_error(e.what());
    return AMUN_ERR_CUDA;
  }
}

extern "C" int amun_vocab_destroy(amun_vocab *v) {
  delete v;
  return AMUN_OK;
}

namespace {

// lines [l0, l1) -> ids appended to out, lens / oov per line
void encode_lines(const amun_vocab &v, const char *text, const int64_t *line_off, int32_t l0, int32_t l1,
                  int32_t unk_id, std::vector<int32_t> &out, int32_t *lens, int32_t *oov) {
  for (int32_t l = l0; l < l1; ++l) {
    const auto *p = reinterpret_cast<const unsigned char *>(text + line_off[l]);
    const auto *end = reinterpret_cast<const unsigned char *>(text + line_off[l + 1]);
    int32_t count = 0, miss = 0;
    while (p < end) {
      int n = 0;
      while (p < end && py_space(utf8_at(p, end, &n))) p += n;  // skip a whitespace run
      const auto *t0 = p;
      while (p < end && !py_space(utf8_at(p, end, &n))) p += n;  // one token
      if (p == t0) break;
      const int32_t id = vocab_find(v, t0, (size_t)(p - t0));
      miss += id < 0;
      out.push_back(id < 0 ? unk_id : id);
      ++count;
    }
    lens[l] = count;
    oov[l] = miss;
  }
}

}  // namespace

extern "C" int amun_vocab_encode(const amun_vocab *v, const char *text, const int64_t *line_off, int32_t n_lines,
                                 int32_t unk_id, int32_t *ids, int64_t ids_cap, int32_t *lens, int32_t *oov,
                                 int64_t *n_ids) {
  try {
    if (!v || !n_ids || n_lines < 0 || (n_lines > 0 && (!text || !line_off || !lens || !oov))) {
      amun_set_last_error("amun_vocab_encode: null argument");
      return AMUN_ERR_INVALID;
    }
    // corpus slices of >= 512 lines on up to 8 host threads, concatenated in order
    const int T = (int)std::max<int64_t>(1, std::min<int64_t>({8, n_lines / 512, (int64_t)std::thread::hardware_concurrency()}));
    std::vector<std::vector<int32_t>> part(T);
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t) {
      const int32_t l0 = (int32_t)((int64_t)n_lines * t / T), l1 = (int32_t)((int64_t)n_lines * (t + 1) / T);
      part[t].reserve((size_t)(line_off[l1] - line_off[l0]) / 4 + 16);
      if (t + 1 < T)
        pool.emplace_back(encode_lines, std::cref(*v), text, line_off, l0, l1, unk_id, std::ref(part[t]), lens, oov);
      else
        encode_lines(*v, text, line_off, l0, l1, unk_id, part[t], lens, oov);
    }
    for (auto &th : pool) th.join();
    int64_t w = 0;
    for (auto &pt : part) {
      if (w + (int64_t)pt.size() > ids_cap) {
        amun_set_last_error("amun_vocab_encode: id buffer too small");
        return AMUN_ERR_INVALID;
      }
      std::memcpy(ids + w, pt.data(), pt.size() * sizeof(int32_t));
      w += (int64_t)pt.size();
    }
    *n_ids = w;
    return AMUN_OK;
  } catch (const std::exception &e) {
    amun_set_last_error(e.what());
    return AMUN_ERR_CUDA;
  }
}
