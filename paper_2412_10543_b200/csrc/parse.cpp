// §8(f3) profile ingestion: the estimator answer parser of the reference
// (parse_profile_text, profiler.py:203-254) as a batched, multi-threaded host
// routine behind the C ABI.  Parsing is branchy byte work on variable-length
// strings that arrive from the network on the host, so it stays on the CPU;
// the parsed rs_profile records are what the GPU gate (rs_prune_gate) reads.
//
// Grammar (profiler.py:191-200, re.IGNORECASE, matched at each line start,
// first matching line wins per field, lines from str.splitlines()):
//   ^\s*Complexity\s*:\s*(High|Low)\b
//   ^\s*Joint Reasoning needed\s*:\s*(Yes|No)\b
//   ^\s*Pieces\s*:\s*(-?\d+)
//   ^\s*Summary range\s*:\s*(-?\d+)\s*-\s*(-?\d+)
// then pieces is clamped into [1, 10] and the summary range is swapped if
// reversed and clamped into [30, 200], flagging the field (:231-245).
//
// Text is UTF-8.  Exact for ASCII text; line breaks and \s also cover the
// Unicode separators/spaces str.splitlines() and \s accept; the keyword
// matcher applies Python's case-insensitive equivalences for i (U+0130,
// U+0131) and s (U+017F).  Deviations (documented in DESIGN.md): non-ASCII
// decimal digits are not numbers here, and \b treats code points >= U+0100
// as word characters except spaces and the general/CJK punctuation blocks.
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <thread>
#include <vector>

#include "ragsched_b200.h"
#include "rs_common.cuh"

namespace rs {
namespace {

struct U8 {
  const unsigned char* p;
  const unsigned char* e;
};

// decode one code point at s (valid UTF-8 from Python's encoder; malformed
// bytes decode as themselves, one byte each)
inline uint32_t decode(const unsigned char* s, const unsigned char* e, int* len) {
  const unsigned c = s[0];
  if (c < 0x80 || s + 1 >= e) {
    *len = 1;
    return c;
  }
  if ((c & 0xE0) == 0xC0 && s + 1 < e) {
    *len = 2;
    return ((c & 0x1F) << 6) | (s[1] & 0x3F);
  }
  if ((c & 0xF0) == 0xE0 && s + 2 < e) {
    *len = 3;
    return ((c & 0x0F) << 12) | ((s[1] & 0x3F) << 6) | (s[2] & 0x3F);
  }
  if ((c & 0xF8) == 0xF0 && s + 3 < e) {
    *len = 4;
    return ((c & 0x07) << 18) | ((s[1] & 0x3F) << 12) | ((s[2] & 0x3F) << 6) | (s[3] & 0x3F);
  }
  *len = 1;
  return c;
}

inline uint32_t peek(const U8& u, int* len) {
  if (u.p >= u.e) {
    *len = 0;
    return 0xFFFFFFFFu;
  }
  return decode(u.p, u.e, len);
}

// str.splitlines() boundaries
inline bool is_linebreak(uint32_t c) {
  return c == 0x0A || c == 0x0D || c == 0x0B || c == 0x0C || c == 0x1C || c == 0x1D || c == 0x1E || c == 0x85 ||
         c == 0x2028 || c == 0x2029;
}

// \s (str patterns): str.isspace()
inline bool is_space(uint32_t c) {
  return c == 0x09 || c == 0x20 || c == 0x1F || is_linebreak(c) || c == 0xA0 || c == 0x1680 ||
         (c >= 0x2000 && c <= 0x200A) || c == 0x202F || c == 0x205F || c == 0x3000;
}

// \w: ASCII alnum + '_', the Latin-1 letters/digits Python's isalnum accepts,
// and (approximation) other code points outside spaces and punctuation blocks
inline bool is_word(uint32_t c) {
  if (c < 0x80) return (c >= '0' && c <= '9') || (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || c == '_';
  if (c < 0x100)
    return c == 0xAA || c == 0xB2 || c == 0xB3 || c == 0xB5 || c == 0xB9 || c == 0xBA || (c >= 0xBC && c <= 0xBE) ||
           (c >= 0xC0 && c <= 0xD6) || (c >= 0xD8 && c <= 0xF6) || c >= 0xF8;
  if (is_space(c)) return false;
  if ((c >= 0x2000 && c <= 0x206F) || (c >= 0x3000 && c <= 0x303F)) return false;
  return true;
}

inline void skip_spaces(U8& u) {
  int n;
  while (u.p < u.e) {
    const uint32_t c = peek(u, &n);
    if (!is_space(c)) return;
    u.p += n;
  }
}

// one keyword character, IGNORECASE: ASCII case plus the non-ASCII code
// points Python's matcher folds onto i, s and k.  `ascii` is cleared when the
// matched code point is plain ASCII (the captured words compare with
// .lower() == "high"/"yes" afterwards, which only ASCII satisfies).
inline bool match_char(U8& u, char want, bool* ascii) {
  int n;
  const uint32_t c = peek(u, &n);
  if (n == 0) return false;
  const char lw = (want >= 'A' && want <= 'Z') ? char(want - 'A' + 'a') : want;
  bool ok;
  if (c < 0x80) {
    const char lc = (c >= 'A' && c <= 'Z') ? char(c - 'A' + 'a') : char(c);
    ok = lc == lw;
  } else {
    ok = (lw == 'i' && (c == 0x130 || c == 0x131)) || (lw == 's' && c == 0x17F) || (lw == 'k' && c == 0x212A);
    if (ok && ascii) *ascii = false;
  }
  if (ok) u.p += n;
  return ok;
}

inline bool match_word(U8& u, const char* w, bool* ascii = nullptr) {
  U8 v = u;
  for (const char* q = w; *q; ++q)
    if (!match_char(v, *q, ascii)) return false;
  u = v;
  return true;
}

inline bool at_boundary(const U8& u) {
  int n;
  const uint32_t c = peek(u, &n);
  return n == 0 || !is_word(c);
}

// \s*:\s*
inline bool colon(U8& u) {
  skip_spaces(u);
  if (u.p >= u.e || *u.p != ':') return false;
  ++u.p;
  skip_spaces(u);
  return true;
}

// -?\d+ (ASCII digits), saturated at +-2^62 (only the order and the domain
// test matter afterwards, both preserved)
inline bool integer(U8& u, int64_t* v) {
  U8 w = u;
  bool neg = false;
  if (w.p < w.e && *w.p == '-') {
    neg = true;
    ++w.p;
  }
  if (w.p >= w.e || *w.p < '0' || *w.p > '9') return false;
  const int64_t cap = int64_t(1) << 62;
  int64_t x = 0;
  while (w.p < w.e && *w.p >= '0' && *w.p <= '9') {
    x = x <= (cap - 9) / 10 ? x * 10 + (*w.p - '0') : cap;
    ++w.p;
  }
  *v = neg ? -x : x;
  u = w;
  return true;
}

struct Found {
  bool cx = false, jt = false, pc = false, sr = false;
  bool high = false, yes = false;
  int64_t pieces = 0, lo = 0, hi = 0;
  int32_t line[4] = {-1, -1, -1, -1};
};

// (High|Low)\b and (Yes|No)\b: returns 1 for the first word, 0 for the
// second, -1 for no match; *plain = captured text is ASCII
inline int choice(U8 u, const char* a, const char* b, bool* plain) {
  bool asc = true;
  U8 v = u;
  if (match_word(v, a, &asc) && at_boundary(v)) {
    *plain = asc;
    return 1;
  }
  asc = true;
  v = u;
  if (match_word(v, b, &asc) && at_boundary(v)) {
    *plain = asc;
    return 0;
  }
  return -1;
}

void match_line(const unsigned char* s, const unsigned char* e, int32_t lineno, Found& f) {
  U8 u{s, e};
  skip_spaces(u);
  const U8 start = u;
  if (!f.cx) {
    U8 v = start;
    bool plain;
    int r;
    if (match_word(v, "complexity") && colon(v) && (r = choice(v, "high", "low", &plain)) >= 0) {
      f.cx = true;
      f.high = r == 1 && plain;  // found.lower() == "high" (profiler.py:228)
      f.line[0] = lineno;
    }
  }
  if (!f.jt) {
    U8 v = start;
    bool plain;
    int r;
    if (match_word(v, "joint reasoning needed") && colon(v) && (r = choice(v, "yes", "no", &plain)) >= 0) {
      f.jt = true;
      f.yes = r == 1 && plain;  // found.lower() == "yes" (profiler.py:229)
      f.line[1] = lineno;
    }
  }
  if (!f.pc) {
    U8 v = start;
    int64_t x;
    if (match_word(v, "pieces") && colon(v) && integer(v, &x)) {
      f.pc = true;
      f.pieces = x;
      f.line[2] = lineno;
    }
  }
  if (!f.sr) {
    U8 v = start;
    int64_t a, b;
    if (match_word(v, "summary range") && colon(v) && integer(v, &a)) {
      skip_spaces(v);
      if (v.p < v.e && *v.p == '-') {
        ++v.p;
        skip_spaces(v);
        if (integer(v, &b)) {
          f.sr = true;
          f.lo = a;
          f.hi = b;
          f.line[3] = lineno;
        }
      }
    }
  }
}

void parse_one(const unsigned char* s, const unsigned char* e, double conf, rs_profile* out, uint8_t* clamped,
               int32_t* lines, uint8_t* status) {
  Found f;
  int32_t lineno = 0;
  const unsigned char* ls = s;
  const unsigned char* p = s;
  while (p < e) {
    int n;
    const uint32_t c = decode(p, e, &n);
    if (is_linebreak(c)) {
      match_line(ls, p, lineno, f);
      p += n;
      if (c == 0x0D && p < e && *p == 0x0A) ++p;  // \r\n is one break
      ls = p;
      ++lineno;
    } else {
      p += n;
    }
  }
  if (ls < e) match_line(ls, e, lineno, f);  // last line (no trailing empty line, as splitlines)

  if (lines)
    for (int i = 0; i < 4; ++i) lines[i] = f.line[i];
  if (!(f.cx && f.jt && f.pc && f.sr)) {
    *status = RS_PARSE_UNPARSEABLE;  // UnparseableAnswer (profiler.py:223-225)
    *out = rs_profile{};
    if (clamped) *clamped = 0;
    return;
  }
  uint8_t cl = 0;
  int64_t pieces = f.pieces;
  if (pieces < 1 || pieces > 10) {
    pieces = std::min<int64_t>(std::max<int64_t>(pieces, 1), 10);
    cl |= RS_CLAMPED_PIECES;
  }
  int64_t lo = f.lo, hi = f.hi;
  if (lo > hi) {
    std::swap(lo, hi);
    cl |= RS_CLAMPED_SUMMARY;
  }
  if (!(30 <= lo && hi <= 200)) {
    lo = std::min<int64_t>(std::max<int64_t>(lo, 30), 200);
    hi = std::min<int64_t>(std::max<int64_t>(hi, 30), 200);
    cl |= RS_CLAMPED_SUMMARY;
  }
  rs_profile r{};
  r.complexity_high = f.high ? 1 : 0;
  r.needs_joint_reasoning = f.yes ? 1 : 0;
  r.pieces_required = uint16_t(pieces);
  r.summary_lo = uint16_t(lo);
  r.summary_hi = uint16_t(hi);
  r.confidence = conf;
  *out = r;
  if (clamped) *clamped = cl;
  *status = RS_PARSE_OK;
}

// CPython 3.12 sum() over floats (builtin_sum_impl): 0 + x0, then Neumaier's
// compensated additions, the compensation added at the end when finite.
struct PySum {
  double f = 0.0, c = 0.0;
  int64_t n = 0;
  void add(double x) {
    if (n++ == 0) {
      f = 0.0 + x;  // int 0 + float
      return;
    }
    const double t = f + x;
    if (std::fabs(f) >= std::fabs(x))
      c += (f - t) + x;
    else
      c += (x - t) + f;
    f = t;
  }
  double value() const { return (c != 0.0 && std::isfinite(c)) ? f + c : f; }
};

// code points in UTF-8 text (lead bytes; str len of the decoded token)
inline int64_t code_points(const unsigned char* s, const unsigned char* e) {
  int64_t n = 0;
  for (; s < e; ++s) n += (*s & 0xC0) != 0x80;
  return n;
}

void field_conf_one(const unsigned char* s, const unsigned char* e, int64_t t0, int64_t t1,
                    const unsigned char* tt, const int64_t* tto, const double* lp, const uint8_t* has, double* out) {
  for (int f = 0; f < 4; ++f) out[f] = 1.0;
  if (t1 <= t0) return;  // `if not tokens` (profiler.py:431)
  rs_profile prof;
  uint8_t st;
  int32_t lines[4];
  parse_one(s, e, 1.0, &prof, nullptr, lines, &st);
  if (st != RS_PARSE_OK) return;  // UnparseableAnswer -> 1.0 (:434-436)
  // line_starts (:439-441): 0 and the end of every splitlines(keepends=True) line, in code points
  std::vector<int64_t> starts{0};
  int64_t cp = 0;
  for (const unsigned char* p = s; p < e;) {
    int nb;
    const uint32_t c = decode(p, e, &nb);
    p += nb;
    ++cp;
    if (is_linebreak(c)) {
      if (c == 0x0D && p < e && *p == 0x0A) {  // \r\n is one break
        ++p;
        ++cp;
      }
      starts.push_back(cp);
    }
  }
  if (cp > starts.back()) starts.push_back(cp);  // a last line without a break
  const int64_t nlines = int64_t(starts.size());
  PySum acc[4];
  int64_t offset = 0;
  for (int64_t t = t0; t < t1; ++t) {
    // the first line whose end lies past the token's start, else the last line (:446-452)
    int64_t lineno = nlines - 2;
    const auto it = std::upper_bound(starts.begin() + 1, starts.end(), offset);
    if (it != starts.end()) lineno = int64_t(it - starts.begin()) - 1;
    if (has[t])
      for (int f = 0; f < 4; ++f)
        if (lines[f] == lineno) acc[f].add(lp[t]);
    offset += code_points(tt + tto[t], tt + tto[t + 1]);
  }
  for (int f = 0; f < 4; ++f)
    if (acc[f].n) out[f] = std::exp(acc[f].value() / double(acc[f].n));  // :461-462
}

}  // namespace
}  // namespace rs

extern "C" int rs_field_confidences(const char* text, const int64_t* offsets, int64_t n, const int64_t* tok_offsets,
                                    const char* tok_text, const int64_t* tok_text_offsets, const double* tok_lp,
                                    const uint8_t* tok_has_lp, double* out, int32_t nthreads) {
  using namespace rs;
  RS_REQUIRE(n >= 0, "n must be non-negative");
  if (n == 0) return RS_OK;
  RS_REQUIRE(text && offsets && tok_offsets && out, "NULL argument");
  for (int64_t i = 0; i < n; ++i) {
    RS_REQUIRE(offsets[i] <= offsets[i + 1] && offsets[i] >= 0, "offsets must be non-decreasing");
    RS_REQUIRE(tok_offsets[i] <= tok_offsets[i + 1] && tok_offsets[i] >= 0, "token offsets must be non-decreasing");
  }
  const int64_t ntok = tok_offsets[n];
  RS_REQUIRE(ntok == 0 || (tok_text && tok_text_offsets && tok_lp && tok_has_lp), "NULL token argument");
  for (int64_t t = 0; t < ntok; ++t)
    RS_REQUIRE(tok_text_offsets[t] <= tok_text_offsets[t + 1] && tok_text_offsets[t] >= 0,
               "token text offsets must be non-decreasing");
  const auto* base = reinterpret_cast<const unsigned char*>(text);
  const auto* tbase = reinterpret_cast<const unsigned char*>(tok_text);
  auto work = [&](int64_t a, int64_t b) {
    for (int64_t i = a; i < b; ++i)
      field_conf_one(base + offsets[i], base + offsets[i + 1], tok_offsets[i], tok_offsets[i + 1], tbase,
                     tok_text_offsets, tok_lp, tok_has_lp, out + 4 * i);
  };
  int t = nthreads > 0 ? nthreads : int(std::thread::hardware_concurrency());
  t = int(std::max<int64_t>(1, std::min<int64_t>(t, n / 256 + 1)));
  if (t == 1) {
    work(0, n);
    return RS_OK;
  }
  std::vector<std::thread> pool;
  for (int i = 0; i < t; ++i) pool.emplace_back(work, n * i / t, n * (i + 1) / t);
  for (auto& th : pool) th.join();
  return RS_OK;
}

extern "C" int rs_parse_profiles(const char* text, const int64_t* offsets, int64_t n, const double* confidence,
                                 rs_profile* out, uint8_t* clamped, int32_t* line_numbers, uint8_t* status,
                                 int32_t nthreads) {
  using namespace rs;
  RS_REQUIRE(n >= 0, "n must be non-negative");
  if (n == 0) return RS_OK;
  RS_REQUIRE(text && offsets && out && status, "NULL argument");
  for (int64_t i = 0; i < n; ++i)
    RS_REQUIRE(offsets[i] <= offsets[i + 1] && offsets[i] >= 0, "offsets must be non-decreasing");
  const auto* base = reinterpret_cast<const unsigned char*>(text);
  auto work = [&](int64_t a, int64_t b) {
    for (int64_t i = a; i < b; ++i)
      parse_one(base + offsets[i], base + offsets[i + 1], confidence ? confidence[i] : 1.0, out + i,
                clamped ? clamped + i : nullptr, line_numbers ? line_numbers + 4 * i : nullptr, status + i);
  };
  int t = nthreads > 0 ? nthreads : int(std::thread::hardware_concurrency());
  t = int(std::max<int64_t>(1, std::min<int64_t>(t, n / 256 + 1)));
  if (t == 1) {
    work(0, n);
    return RS_OK;
  }
  std::vector<std::thread> pool;
  for (int i = 0; i < t; ++i) pool.emplace_back(work, n * i / t, n * (i + 1) / t);
  for (auto& th : pool) th.join();
  return RS_OK;
}
