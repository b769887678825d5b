// F1 — episode-log / sidecar ingest: JSON lines -> SoA segment table (host).
//
// Reference: rollout/episodes.py:132-147 (read_episodes: one EpisodeRecord per
// non-blank line, any defect -> EpisodeLogError "path:line: ..."),
// EpisodeRecord.from_dict :95-120, trajectory_from_dict trajectory.py:182-200
// (origin / alternation / turn_count checks), cli._read_sidecar cli.py:255-269
// and cli._flat_logps cli.py:233-252, and the task_id grouping of cli.loss
// (cli.py:309-311: first-appearance order).
//
// The whole file is read once; line blocks are parsed by a pool of threads
// with a small recursive-descent JSON parser (numbers via strtod, i.e. the
// same correctly-rounded conversion as CPython's float()); results are merged
// in line order and episodes are permuted so every task_id group is
// contiguous, ready for tl_pack_varlen / tl_group_advantages / tl_loss_f64.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/toolloop_b200.h"

namespace tl {
void set_error(const char* fmt, ...);
}

namespace {

struct JsonError {
  std::string msg;
};

// Minimal JSON reader over [p, end).  Values we need are materialised; all
// others are skipped with full syntax checking.
struct Reader {
  const char* p;
  const char* end;

  [[noreturn]] void fail(const char* what) { throw JsonError{what}; }
  void ws() {
    while (p < end && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
  }
  bool peek(char c) {
    ws();
    return p < end && *p == c;
  }
  void expect(char c) {
    ws();
    if (p >= end || *p != c) {
      static thread_local char buf[64];
      snprintf(buf, sizeof(buf), "expected '%c'", c);
      fail(buf);
    }
    ++p;
  }
  std::string string() {
    ws();
    if (p >= end || *p != '"') fail("expected string");
    ++p;
    std::string out;
    while (true) {
      if (p >= end) fail("unterminated string");
      char c = *p++;
      if (c == '"') break;
      if (c == '\\') {
        if (p >= end) fail("bad escape");
        char e = *p++;
        switch (e) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'n': out += '\n'; break;
          case 'r': out += '\r'; break;
          case 't': out += '\t'; break;
          case 'u': {
            if (end - p < 4) fail("bad \\u escape");
            unsigned cp = 0;
            for (int i = 0; i < 4; ++i) {
              char h = *p++;
              cp <<= 4;
              if (h >= '0' && h <= '9') cp |= h - '0';
              else if (h >= 'a' && h <= 'f') cp |= h - 'a' + 10;
              else if (h >= 'A' && h <= 'F') cp |= h - 'A' + 10;
              else fail("bad \\u escape");
            }
            if (cp >= 0xD800 && cp <= 0xDBFF && end - p >= 6 && p[0] == '\\' && p[1] == 'u') {
              unsigned lo = 0;
              const char* q = p + 2;
              bool ok = true;
              for (int i = 0; i < 4; ++i) {
                char h = q[i];
                lo <<= 4;
                if (h >= '0' && h <= '9') lo |= h - '0';
                else if (h >= 'a' && h <= 'f') lo |= h - 'a' + 10;
                else if (h >= 'A' && h <= 'F') lo |= h - 'A' + 10;
                else ok = false;
              }
              if (ok && lo >= 0xDC00 && lo <= 0xDFFF) {
                cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                p += 6;
              }
            }
            // UTF-8 encode
            if (cp < 0x80) out += static_cast<char>(cp);
            else if (cp < 0x800) {
              out += static_cast<char>(0xC0 | (cp >> 6));
              out += static_cast<char>(0x80 | (cp & 0x3F));
            } else if (cp < 0x10000) {
              out += static_cast<char>(0xE0 | (cp >> 12));
              out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
              out += static_cast<char>(0x80 | (cp & 0x3F));
            } else {
              out += static_cast<char>(0xF0 | (cp >> 18));
              out += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
              out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
              out += static_cast<char>(0x80 | (cp & 0x3F));
            }
            break;
          }
          default: fail("bad escape");
        }
      } else {
        out += c;
      }
    }
    return out;
  }
  // Python float(json number) semantics (also accepts NaN/Infinity like json.loads)
  double number() {
    ws();
    if (end - p >= 3 && !strncmp(p, "NaN", 3)) {
      p += 3;
      return NAN;
    }
    if (end - p >= 8 && !strncmp(p, "Infinity", 8)) {
      p += 8;
      return INFINITY;
    }
    if (end - p >= 9 && !strncmp(p, "-Infinity", 9)) {
      p += 9;
      return -INFINITY;
    }
    const char* s = p;
    if (p < end && *p == '-') ++p;
    if (p >= end || !(*p >= '0' && *p <= '9')) fail("expected number");
    while (p < end && ((*p >= '0' && *p <= '9') || *p == '.' || *p == 'e' || *p == 'E' ||
                       *p == '+' || *p == '-'))
      ++p;
    // std::from_chars: correctly rounded like CPython's float(), no allocation
    double v = 0.0;
    const auto r = std::from_chars(s, p, v);
    if (r.ec != std::errc() || r.ptr != p) fail("bad number");
    return v;
  }
  bool is_null() {
    ws();
    if (end - p >= 4 && !strncmp(p, "null", 4)) {
      p += 4;
      return true;
    }
    return false;
  }
  bool boolean() {
    ws();
    if (end - p >= 4 && !strncmp(p, "true", 4)) {
      p += 4;
      return true;
    }
    if (end - p >= 5 && !strncmp(p, "false", 5)) {
      p += 5;
      return false;
    }
    fail("expected boolean");
  }
  void skip() {
    ws();
    if (p >= end) fail("unexpected end");
    char c = *p;
    if (c == '"') {
      string();
    } else if (c == '{') {
      ++p;
      if (peek('}')) {
        ++p;
        return;
      }
      while (true) {
        string();
        expect(':');
        skip();
        if (peek(',')) {
          ++p;
          continue;
        }
        expect('}');
        return;
      }
    } else if (c == '[') {
      ++p;
      if (peek(']')) {
        ++p;
        return;
      }
      while (true) {
        skip();
        if (peek(',')) {
          ++p;
          continue;
        }
        expect(']');
        return;
      }
    } else if (c == 't' || c == 'f') {
      boolean();
    } else if (c == 'n') {
      if (!is_null()) fail("bad literal");
    } else {
      number();
    }
  }
  // Iterate object members: fn(key) must consume the value.
  template <class F>
  void object(F&& fn) {
    expect('{');
    if (peek('}')) {
      ++p;
      return;
    }
    while (true) {
      std::string k = string();
      expect(':');
      fn(k);
      if (peek(',')) {
        ++p;
        continue;
      }
      expect('}');
      return;
    }
  }
  template <class F>
  void array(F&& fn) {
    expect('[');
    if (peek(']')) {
      ++p;
      return;
    }
    while (true) {
      fn();
      if (peek(',')) {
        ++p;
        continue;
      }
      expect(']');
      return;
    }
  }
};

struct Episode {
  std::string task_id;
  double reward = 0;
  std::vector<uint8_t> seg_action;
  std::vector<int32_t> seg_len;
  std::vector<int32_t> tokens;
  bool has_alog = false;
  std::vector<double> flat;  // _flat_logps (0.0 on observation tokens)
  int line = 0;
};

std::string scalar_to_str(Reader& r) {
  r.ws();
  if (r.p < r.end && *r.p == '"') return r.string();
  const char* s = r.p;
  r.skip();
  return std::string(s, r.p);  // str() of a JSON scalar, close to Python's for ints
}

Episode parse_episode(const char* b, const char* e, int line) {
  Reader r{b, e};
  Episode ep;
  ep.line = line;
  bool have_tid = false, have_reward = false, have_traj = false, have_timings = false,
       have_pid = false, have_rb = false, have_limits = false;
  int n_timings = -1;
  std::vector<std::vector<double>> alog;
  r.object([&](const std::string& k) {
    if (k == "task_id") {
      ep.task_id = scalar_to_str(r);
      have_tid = true;
    } else if (k == "reward") {
      ep.reward = r.number();
      have_reward = true;
    } else if (k == "policy_id") {
      r.skip();
      have_pid = true;
    } else if (k == "reward_breakdown") {
      r.skip();
      have_rb = true;
    } else if (k == "limits") {
      r.skip();
      have_limits = true;
    } else if (k == "timings") {
      n_timings = 0;
      r.array([&] {
        r.skip();
        ++n_timings;
      });
      have_timings = true;
    } else if (k == "action_logprobs") {
      if (r.is_null()) return;
      ep.has_alog = true;
      r.array([&] {
        alog.emplace_back();
        auto& row = alog.back();
        r.array([&] { row.push_back(r.number()); });
      });
    } else if (k == "trajectory") {
      have_traj = true;
      long long declared_turns = -1;
      r.object([&](const std::string& tk) {
        if (tk == "segments") {
          r.array([&] {
            int origin = -1;
            size_t start = ep.tokens.size();
            r.object([&](const std::string& sk) {
              if (sk == "origin") {
                std::string o = r.string();
                if (o == "action") origin = 1;
                else if (o == "observation") origin = 0;
                else throw JsonError{"segment " + std::to_string(ep.seg_len.size()) +
                                     ": unknown origin '" + o + "'"};
              } else if (sk == "tokens") {
                r.array([&] {
                  const double v = r.number();
                  ep.tokens.push_back(static_cast<int32_t>(v));
                });
              } else {
                r.skip();
              }
            });
            if (origin < 0) throw JsonError{"segment without origin"};
            const size_t i = ep.seg_len.size();
            const int prev = i ? ep.seg_action[i - 1] : -1;
            if (origin == prev || (prev == -1 && origin != 1))
              throw JsonError{"segment " + std::to_string(i) + ": broken alternation"};
            ep.seg_action.push_back(static_cast<uint8_t>(origin));
            ep.seg_len.push_back(static_cast<int32_t>(ep.tokens.size() - start));
          });
        } else if (tk == "turn_count") {
          if (!r.is_null()) declared_turns = static_cast<long long>(r.number());
        } else {
          r.skip();
        }
      });
      long long turns = 0;
      for (uint8_t a : ep.seg_action) turns += a ? 0 : 1;
      if (declared_turns >= 0 && declared_turns != turns)
        throw JsonError{"turn_count " + std::to_string(declared_turns) + " does not match " +
                        std::to_string(turns) + " observation segments"};
    } else {
      r.skip();
    }
  });
  r.ws();
  if (r.p != r.end) throw JsonError{"Extra data"};
  if (!have_tid) throw JsonError{"'task_id'"};
  if (!have_pid) throw JsonError{"'policy_id'"};
  if (!have_traj) throw JsonError{"'trajectory'"};
  if (!have_timings) throw JsonError{"'timings'"};
  if (!have_reward) throw JsonError{"'reward'"};
  if (!have_rb) throw JsonError{"'reward_breakdown'"};
  if (!have_limits) throw JsonError{"'limits'"};
  if (n_timings != static_cast<int>(ep.seg_len.size()))
    throw JsonError{"timings has " + std::to_string(n_timings) + " entries for " +
                    std::to_string(ep.seg_len.size()) + " segments"};
  if (ep.has_alog) {
    // cli._flat_logps: rows align with action segments; observation -> 0.0
    ep.flat.reserve(ep.tokens.size());
    size_t row = 0;
    bool aligned = true;
    for (size_t s = 0; s < ep.seg_len.size(); ++s) {
      if (ep.seg_action[s]) {
        if (row >= alog.size() || alog[row].size() != static_cast<size_t>(ep.seg_len[s])) {
          aligned = false;
          break;
        }
        ep.flat.insert(ep.flat.end(), alog[row].begin(), alog[row].end());
        ++row;
      } else {
        ep.flat.insert(ep.flat.end(), ep.seg_len[s], 0.0);
      }
    }
    if (!aligned) {
      ep.flat.clear();
      ep.has_alog = false;
      ep.line = -line;  // marks "does not align" for the flat-logps path
    }
  }
  return ep;
}

struct SideRow {
  std::vector<double> nw, old, ref;
  bool has_old = false, has_ref = false;
};

SideRow parse_side(const char* b, const char* e) {
  Reader r{b, e};
  SideRow s;
  bool have_new = false;
  r.ws();
  if (r.p >= r.end || *r.p != '{') throw JsonError{"expected an object with 'logp_new'"};
  r.object([&](const std::string& k) {
    auto arr = [&](std::vector<double>& v) { r.array([&] { v.push_back(r.number()); }); };
    if (k == "logp_new") {
      arr(s.nw);
      have_new = true;
    } else if (k == "logp_old") {
      if (!r.is_null()) {
        arr(s.old);
        s.has_old = true;
      }
    } else if (k == "logp_ref") {
      if (!r.is_null()) {
        arr(s.ref);
        s.has_ref = true;
      }
    } else {
      r.skip();
    }
  });
  if (!have_new) throw JsonError{"expected an object with 'logp_new'"};
  return s;
}

bool read_file(const char* path, std::string& out) {
  FILE* f = fopen(path, "rb");
  if (!f) return false;
  fseek(f, 0, SEEK_END);
  long n = ftell(f);
  fseek(f, 0, SEEK_SET);
  out.resize(n > 0 ? n : 0);
  size_t got = n > 0 ? fread(&out[0], 1, n, f) : 0;
  fclose(f);
  return got == out.size();
}

struct Line {
  const char* b;
  const char* e;
  int no;
};

std::vector<Line> split_lines(const std::string& s) {
  std::vector<Line> out;
  const char* p = s.data();
  const char* end = p + s.size();
  int no = 0;
  while (p < end) {
    const char* q = static_cast<const char*>(memchr(p, '\n', end - p));
    if (!q) q = end;
    ++no;
    const char* a = p;
    bool blank = true;
    for (const char* c = a; c < q; ++c)
      if (!(*c == ' ' || *c == '\t' || *c == '\r')) {
        blank = false;
        break;
      }
    if (!blank) out.push_back({a, q, no});
    p = q + 1;
  }
  return out;
}

template <class T, class F>
bool parse_parallel(const std::vector<Line>& lines, std::vector<T>& out, F&& fn, std::string& err,
                    int& err_line) {
  const size_t n = lines.size();
  out.resize(n);
  // episodes are long lines (thousands of numbers): one thread per line is fine
  unsigned nt = std::thread::hardware_concurrency();
  nt = std::max(1u, std::min(nt, static_cast<unsigned>(n)));
  std::vector<std::string> errs(nt);
  std::vector<int> eline(nt, 0);
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t) {
    th.emplace_back([&, t] {
      const size_t a = n * t / nt, b = n * (t + 1) / nt;
      for (size_t i = a; i < b; ++i) {
        try {
          out[i] = fn(lines[i]);
        } catch (const JsonError& e) {
          errs[t] = e.msg;
          eline[t] = lines[i].no;
          return;
        }
      }
    });
  }
  for (auto& x : th) x.join();
  for (unsigned t = 0; t < nt; ++t)
    if (!errs[t].empty()) {
      err = errs[t];
      err_line = eline[t];
      return false;
    }
  return true;
}

}  // namespace

struct tl_episode_batch {
  std::vector<int32_t> token_pool, seg_src_off, seg_len, traj_seg_off, group_off;
  std::vector<uint8_t> seg_is_action;
  std::vector<double> rewards, logp_new, logp_old, logp_ref;
  std::vector<std::string> task_ids;  // per group
  int64_t n_episodes = 0;
  int32_t has_ref = 0;
};

extern "C" int tl_ingest_open(const char* episodes_path, const char* sidecar_path,
                              tl_episode_batch** out) {
  *out = nullptr;
  std::string text;
  if (!read_file(episodes_path, text)) {
    tl::set_error("%s: cannot read", episodes_path);
    return TL_ERR_INVALID_ARG;
  }
  const std::vector<Line> lines = split_lines(text);
  std::vector<Episode> eps;
  std::string err;
  int err_line = 0;
  if (!parse_parallel(lines, eps, [](const Line& l) { return parse_episode(l.b, l.e, l.no); }, err,
                      err_line)) {
    tl::set_error("%s:%d: %s", episodes_path, err_line, err.c_str());
    return TL_ERR_EPISODE_LOG;
  }
  const size_t n = eps.size();
  if (n == 0) {
    tl::set_error("%s: no episodes", episodes_path);
    return TL_ERR_INVALID_ARG;
  }
  // per-token log-probs
  std::vector<std::vector<double>> nw(n), old(n), ref(n);
  std::vector<uint8_t> has_ref(n, 0);
  bool any_ref = false;
  if (sidecar_path) {
    std::string side;
    if (!read_file(sidecar_path, side)) {
      tl::set_error("%s: cannot read", sidecar_path);
      return TL_ERR_INVALID_ARG;
    }
    const std::vector<Line> sl = split_lines(side);
    std::vector<SideRow> rows;
    if (!parse_parallel(sl, rows, [](const Line& l) { return parse_side(l.b, l.e); }, err,
                        err_line)) {
      tl::set_error("%s:%d: %s", sidecar_path, err_line, err.c_str());
      return TL_ERR_EPISODE_LOG;
    }
    if (rows.size() != n) {
      tl::set_error("%s: %zu sidecar rows for %zu episodes", sidecar_path, rows.size(), n);
      return TL_ERR_MASK_MISMATCH;
    }
    for (size_t i = 0; i < n; ++i) {
      nw[i] = std::move(rows[i].nw);
      old[i] = rows[i].has_old ? std::move(rows[i].old) : nw[i];
      if (rows[i].has_ref) {
        ref[i] = std::move(rows[i].ref);
        has_ref[i] = 1;
        any_ref = true;
      }
    }
  } else {
    for (size_t i = 0; i < n; ++i) {
      if (!eps[i].has_alog) {
        if (eps[i].line < 0)
          tl::set_error("episode '%s': action_logprobs do not align with action segments",
                        eps[i].task_id.c_str());
        else
          tl::set_error("episode '%s' has no action_logprobs; supply --logprobs",
                        eps[i].task_id.c_str());
        return TL_ERR_MASK_MISMATCH;
      }
      nw[i] = eps[i].flat;
      old[i] = eps[i].flat;
    }
  }
  // token_records length checks (loss.py:85-90)
  for (size_t i = 0; i < n; ++i) {
    const size_t L = eps[i].tokens.size();
    if (nw[i].size() != L || old[i].size() != L) {
      tl::set_error("%zu tokens vs %zu new / %zu old logps", L, nw[i].size(), old[i].size());
      return TL_ERR_MASK_MISMATCH;
    }
    if (has_ref[i] && ref[i].size() != L) {
      tl::set_error("%zu tokens vs %zu ref logps", L, ref[i].size());
      return TL_ERR_MASK_MISMATCH;
    }
  }
  // group by task_id, first-appearance order
  std::unordered_map<std::string, int> gid;
  std::vector<std::vector<int>> members;
  for (size_t i = 0; i < n; ++i) {
    auto it = gid.find(eps[i].task_id);
    if (it == gid.end()) {
      it = gid.emplace(eps[i].task_id, static_cast<int>(members.size())).first;
      members.emplace_back();
    }
    members[it->second].push_back(static_cast<int>(i));
  }
  auto* b = new tl_episode_batch();
  b->n_episodes = static_cast<int64_t>(n);
  b->has_ref = any_ref ? 1 : 0;
  b->group_off.push_back(0);
  b->traj_seg_off.push_back(0);
  for (size_t g = 0; g < members.size(); ++g) {
    b->task_ids.push_back(eps[members[g][0]].task_id);
    for (int i : members[g]) {
      Episode& e = eps[i];
      size_t pos = b->token_pool.size();
      b->token_pool.insert(b->token_pool.end(), e.tokens.begin(), e.tokens.end());
      for (size_t s = 0; s < e.seg_len.size(); ++s) {
        b->seg_src_off.push_back(static_cast<int32_t>(pos));
        b->seg_len.push_back(e.seg_len[s]);
        b->seg_is_action.push_back(e.seg_action[s]);
        pos += e.seg_len[s];
      }
      b->traj_seg_off.push_back(static_cast<int32_t>(b->seg_len.size()));
      b->rewards.push_back(e.reward);
      b->logp_new.insert(b->logp_new.end(), nw[i].begin(), nw[i].end());
      b->logp_old.insert(b->logp_old.end(), old[i].begin(), old[i].end());
      if (any_ref) {
        if (has_ref[i]) b->logp_ref.insert(b->logp_ref.end(), ref[i].begin(), ref[i].end());
        else b->logp_ref.insert(b->logp_ref.end(), e.tokens.size(), NAN);
      }
    }
    b->group_off.push_back(static_cast<int32_t>(b->rewards.size()));
  }
  *out = b;
  return TL_OK;
}

extern "C" int tl_ingest_sizes(const tl_episode_batch* b, int64_t* n_episodes, int64_t* n_segments,
                               int64_t* n_tokens, int64_t* n_groups, int32_t* has_ref) {
  if (!b) return TL_ERR_INVALID_ARG;
  *n_episodes = b->n_episodes;
  *n_segments = static_cast<int64_t>(b->seg_len.size());
  *n_tokens = static_cast<int64_t>(b->token_pool.size());
  *n_groups = static_cast<int64_t>(b->group_off.size()) - 1;
  *has_ref = b->has_ref;
  return TL_OK;
}

extern "C" int tl_ingest_fill(const tl_episode_batch* b, int32_t* token_pool, int32_t* seg_src_off,
                              int32_t* seg_len, uint8_t* seg_is_action, int32_t* traj_seg_off,
                              int32_t* group_off, double* rewards, double* logp_new,
                              double* logp_old, double* logp_ref) {
  if (!b) return TL_ERR_INVALID_ARG;
  auto cp = [](auto* dst, const auto& v) {
    if (dst && !v.empty()) memcpy(dst, v.data(), v.size() * sizeof(v[0]));
  };
  cp(token_pool, b->token_pool);
  cp(seg_src_off, b->seg_src_off);
  cp(seg_len, b->seg_len);
  cp(seg_is_action, b->seg_is_action);
  cp(traj_seg_off, b->traj_seg_off);
  cp(group_off, b->group_off);
  cp(rewards, b->rewards);
  cp(logp_new, b->logp_new);
  cp(logp_old, b->logp_old);
  if (logp_ref && b->has_ref) cp(logp_ref, b->logp_ref);
  return TL_OK;
}

extern "C" void tl_ingest_free(tl_episode_batch* b) { delete b; }
