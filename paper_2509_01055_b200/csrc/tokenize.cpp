// F4 — incremental tokenisation of rollout segments (host, multithreaded).
//
// Reference: tokenizer.ToyMergeTokenizer (tokenizer.py:36-87): byte ids
// 0..255 plus an ordered merge table; rule k (left, right) -> id 256 + k, and
// each rule makes ONE left-to-right pass over the current sequence, merging
// every adjacent (left, right) occurrence.  Segments are encoded one at a
// time and never re-encoded as one string (trajectory.py:1-8, the prefix
// stability the packer relies on), then capped at a token budget keeping the
// leading tokens (trajectory._tokenize :97-104; orchestrator.feed_action /
// feed_response :112-117, :156-161).
//
// Output layout: segment i's ids are written at token_pool[text_off[i]...]
// (a segment never has more tokens than bytes), so (token_pool,
// seg_src_off = text_off, seg_len) is directly the segment table that
// tl_pack_varlen consumes — no compaction pass.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/toolloop_b200.h"

namespace tl {
void set_error(const char* fmt, ...);
}

struct tl_tokenizer {
  std::vector<std::string> token_bytes;        // id -> bytes
  std::vector<int32_t> rule_l, rule_r, rule_id;  // merge rules in table order
};

namespace {

// One rule pass, in place: write index never overtakes read index.
inline int64_t merge_pass(int32_t* a, int64_t n, int32_t l, int32_t r, int32_t id) {
  int64_t w = 0, i = 0;
  while (i < n) {
    if (i + 1 < n && a[i] == l && a[i + 1] == r) {
      a[w++] = id;
      i += 2;
    } else {
      a[w++] = a[i++];
    }
  }
  return w;
}

// Encode bytes [s, s + n) into out (capacity n); returns the token count.
int64_t encode_one(const tl_tokenizer& t, const uint8_t* s, int64_t n, int32_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = s[i];
  for (size_t k = 0; k < t.rule_id.size() && n > 1; ++k) {
    // cheap skip: a rule whose left id is absent cannot fire
    const int32_t l = t.rule_l[k];
    bool any = false;
    for (int64_t i = 0; i + 1 < n; ++i)
      if (out[i] == l) {
        any = true;
        break;
      }
    if (any) n = merge_pass(out, n, l, t.rule_r[k], t.rule_id[k]);
  }
  return n;
}

}  // namespace

extern "C" int tl_tokenizer_create(const uint8_t* merge_bytes, const int64_t* merge_off,
                                   int32_t n_merges, tl_tokenizer** out) {
  if (!out || n_merges < 0 || (n_merges > 0 && (!merge_bytes || !merge_off))) {
    tl::set_error("tl_tokenizer_create: bad arguments");
    return TL_ERR_INVALID_ARG;
  }
  auto* t = new tl_tokenizer();
  std::unordered_map<std::string, int32_t> by_bytes;
  for (int i = 0; i < 256; ++i) {
    t->token_bytes.emplace_back(1, static_cast<char>(i));
    by_bytes[t->token_bytes.back()] = i;
  }
  for (int32_t k = 0; k < n_merges; ++k) {
    const std::string left(reinterpret_cast<const char*>(merge_bytes) + merge_off[2 * k],
                           merge_off[2 * k + 1] - merge_off[2 * k]);
    const std::string right(reinterpret_cast<const char*>(merge_bytes) + merge_off[2 * k + 1],
                            merge_off[2 * k + 2] - merge_off[2 * k + 1]);
    auto li = by_bytes.find(left), ri = by_bytes.find(right);
    if (li == by_bytes.end() || ri == by_bytes.end()) {
      // tokenizer.py:55-58
      tl::set_error("merge (%s, %s) references a token that does not exist yet", left.c_str(),
                    right.c_str());
      delete t;
      return TL_ERR_INVALID_ARG;
    }
    const int32_t id = static_cast<int32_t>(t->token_bytes.size());
    t->rule_l.push_back(li->second);
    t->rule_r.push_back(ri->second);
    t->rule_id.push_back(id);
    t->token_bytes.push_back(left + right);
    by_bytes[t->token_bytes.back()] = id;  // a later duplicate spelling wins, as in the dict
  }
  *out = t;
  return TL_OK;
}

extern "C" void tl_tokenizer_free(tl_tokenizer* tok) { delete tok; }

extern "C" int32_t tl_tokenizer_vocab_size(const tl_tokenizer* tok) {
  return tok ? static_cast<int32_t>(tok->token_bytes.size()) : 0;
}

extern "C" int tl_tokenize_segments(const tl_tokenizer* tok, const uint8_t* text,
                                    const int64_t* text_off, int64_t n_segments,
                                    const int32_t* max_tokens, int32_t* token_pool,
                                    int32_t* seg_len, int32_t n_threads) {
  if (!tok || n_segments < 0 || (n_segments > 0 && (!text_off || !token_pool || !seg_len))) {
    tl::set_error("tl_tokenize_segments: bad arguments");
    return TL_ERR_INVALID_ARG;
  }
  if (n_segments == 0) return TL_OK;
  for (int64_t i = 0; i < n_segments; ++i)
    if (text_off[i + 1] < text_off[i]) {
      tl::set_error("tl_tokenize_segments: text_off not non-decreasing at %lld", (long long)i);
      return TL_ERR_INVALID_ARG;
    }
  if (text_off[n_segments] - text_off[0] > 0 && !text) {
    tl::set_error("tl_tokenize_segments: text is NULL");
    return TL_ERR_INVALID_ARG;
  }
  auto run = [&](int64_t s0, int64_t s1) {
    for (int64_t i = s0; i < s1; ++i) {
      const int64_t b0 = text_off[i], nb = text_off[i + 1] - b0;
      int64_t n = encode_one(*tok, text + b0, nb, token_pool + b0);
      if (max_tokens && max_tokens[i] >= 0 && n > max_tokens[i]) n = max_tokens[i];
      seg_len[i] = static_cast<int32_t>(n);
    }
  };
  const int64_t total = text_off[n_segments] - text_off[0];
  int hw = static_cast<int>(std::thread::hardware_concurrency());
  int nt = n_threads > 0 ? n_threads : (hw > 0 ? hw : 1);
  nt = static_cast<int>(std::min<int64_t>(nt, std::max<int64_t>(1, total / (1 << 16))));
  nt = static_cast<int>(std::min<int64_t>(nt, n_segments));
  if (nt <= 1) {
    run(0, n_segments);
    return TL_OK;
  }
  // contiguous segment ranges of ~equal bytes (segments stay whole)
  std::vector<int64_t> cut(nt + 1, n_segments);
  cut[0] = 0;
  for (int k = 1; k < nt; ++k) {
    const int64_t target = text_off[0] + total * k / nt;
    cut[k] = std::lower_bound(text_off, text_off + n_segments, target) - text_off;
    cut[k] = std::max(cut[k], cut[k - 1]);
  }
  std::vector<std::thread> th;
  for (int k = 0; k < nt; ++k)
    if (cut[k + 1] > cut[k]) th.emplace_back(run, cut[k], cut[k + 1]);
  for (auto& x : th) x.join();
  return TL_OK;
}

extern "C" int tl_tokenizer_decode(const tl_tokenizer* tok, const int32_t* ids, int64_t n,
                                   uint8_t* out, int64_t cap, int64_t* len) {
  if (!tok || n < 0 || (n > 0 && !ids) || !len) {
    tl::set_error("tl_tokenizer_decode: bad arguments");
    return TL_ERR_INVALID_ARG;
  }
  const int64_t V = static_cast<int64_t>(tok->token_bytes.size());
  int64_t w = 0;
  bool fits = out != nullptr;  // bytes are copied only while they all fit
  for (int64_t i = 0; i < n; ++i) {
    if (ids[i] < 0 || ids[i] >= V) {
      tl::set_error("token id %d out of range (vocab %lld)", ids[i], (long long)V);
      return TL_ERR_INVALID_ARG;
    }
    const std::string& b = tok->token_bytes[ids[i]];
    fits = fits && w + static_cast<int64_t>(b.size()) <= cap;
    if (fits) memcpy(out + w, b.data(), b.size());
    w += static_cast<int64_t>(b.size());
  }
  *len = w;
  return TL_OK;
}
