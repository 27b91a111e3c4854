// Host-side front end of the C-ABI (no device code): the reference's point
// file format and input validation, so files feed the GPU build directly.
//
//   hood_parse_points     cli.cpp:62-99   (parse_points: count, then x y pairs;
//                                          '#' comments; strtod/strtoll tokens;
//                                          count <= 2^26, cli.cpp:17)
//   hood_format_points    cli.cpp:101-106 (write_point_set, "%.17g" coords)
//   hood_format_section   cli.cpp:47-52   (write_section of the run output)
//   hood_format_trace_round cli.cpp:108-118 (write_trace_round)
//   hood_validate_points  hoodbuf.cpp:30-70 (power of two, x in (0,1) strictly
//                                          increasing, collinearity margin
//                                          1e-9 over all triples for n <= 64,
//                                          else consecutive + 10n sampled)
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../include/hood_b200.h"

namespace {

constexpr long long kMaxPointCount = 1LL << 26;  // cli.cpp:17
constexpr double kCollinearMargin = 1e-9;        // hoodbuf.hpp:15

struct Tok {
  const char* p;
  int len;
  int line;
};

// Whitespace-separated tokens, '#' to end of line ignored.
std::vector<Tok> tokens_of(const char* text, long long len) {
  std::vector<Tok> out;
  int line = 1;
  long long i = 0;
  while (i < len) {
    const char c = text[i];
    if (c == '\n') {
      ++line;
      ++i;
    } else if (c == '#') {
      while (i < len && text[i] != '\n') ++i;
    } else if (c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f') {
      ++i;
    } else {
      const long long s = i;
      while (i < len && !(text[i] == ' ' || text[i] == '\t' || text[i] == '\r' || text[i] == '\v' ||
                          text[i] == '\f' || text[i] == '\n' || text[i] == '#'))
        ++i;
      out.push_back({text + s, (int)(i - s), line});
    }
  }
  return out;
}

bool to_double(const Tok& t, double& v) {
  const std::string s(t.p, (size_t)t.len);
  char* end = nullptr;
  v = std::strtod(s.c_str(), &end);
  return end != s.c_str() && *end == '\0';
}

// geom.hpp:22-24, evaluated as written (no contraction: this file is built
// without -ffast-math and host FMA contraction is off for x86-64 by default).
double orient(const double* r, const double* p, const double* q) {
  const volatile double a = (q[0] - p[0]) * (r[1] - p[1]);
  const volatile double b = (q[1] - p[1]) * (r[0] - p[0]);
  return a - b;
}

}  // namespace

extern "C" {

int hood_parse_points(const char* text, int64_t len, double* xy, int64_t cap, int64_t* count, int64_t* err_line) {
  if (!text || len < 0 || !count) return HOOD_ERR_INVALID_ARG;
  if (err_line) *err_line = 0;
  const std::vector<Tok> toks = tokens_of(text, len);
  auto fail = [&](int line) {
    if (err_line) *err_line = line;
    return HOOD_ERR_PARSE;
  };
  size_t pos = 0;
  if (toks.empty()) return fail(1);
  {
    const std::string s(toks[0].p, (size_t)toks[0].len);
    char* end = nullptr;
    errno = 0;
    const long long c = std::strtoll(s.c_str(), &end, 10);
    if (end == s.c_str() || *end != '\0' || c < 0) return fail(toks[0].line);
    if (c > kMaxPointCount) return fail(toks[0].line);
    *count = c;
    pos = 1;
  }
  const long long n = *count;
  if (!xy || cap < n) return HOOD_ERR_CAPACITY;  // *count tells the caller how much to allocate
  for (long long k = 0; k < 2 * n; ++k) {
    if (pos >= toks.size()) return fail(toks.back().line);
    double v;
    if (!to_double(toks[pos], v)) return fail(toks[pos].line);
    xy[k] = v;
    ++pos;
  }
  if (pos != toks.size()) return fail(toks[pos].line);
  return HOOD_OK;
}

int64_t hood_format_points(const double* xy, int64_t n, char* buf, int64_t cap) {
  if (n < 0 || (n > 0 && !xy)) return -1;
  std::string out = std::to_string(n) + "\n";
  char tmp[96];
  for (int64_t i = 0; i < n; ++i) {
    const int k = std::snprintf(tmp, sizeof tmp, "%.17g %.17g\n", xy[2 * i], xy[2 * i + 1]);
    out.append(tmp, (size_t)k);
  }
  if (buf && cap >= (int64_t)out.size()) std::memcpy(buf, out.data(), out.size());
  return (int64_t)out.size();
}

int64_t hood_format_section(const char* label, const double* xy, int64_t n, char* buf, int64_t cap) {
  if (!label || n < 0 || (n > 0 && !xy)) return -1;
  std::string out = std::string(label) + " " + std::to_string(n) + "\n";
  char tmp[96];
  for (int64_t i = 0; i < n; ++i) {
    const int k = std::snprintf(tmp, sizeof tmp, "%.17g %.17g\n", xy[2 * i], xy[2 * i + 1]);
    out.append(tmp, (size_t)k);
  }
  if (buf && cap >= (int64_t)out.size()) std::memcpy(buf, out.data(), out.size());
  return (int64_t)out.size();
}

int64_t hood_format_trace_round(const double* slots, int64_t n, int64_t d, char* buf, int64_t cap) {
  if (!slots || n < 1 || d < 1 || n % d != 0) return -1;
  std::string out = "d " + std::to_string(d) + "\n";
  char tmp[96];
  for (int64_t b = 0; b < n / d; ++b) {
    const double* blk = slots + 2 * b * d;
    int64_t k = 0;
    while (k < d && !(blk[2 * k] > 1.0)) ++k;  // block_corners: up to the first REMOTE (geom.hpp:18)
    out += std::to_string(k) + "\n";
    for (int64_t i = 0; i < k; ++i) {
      const int m = std::snprintf(tmp, sizeof tmp, "%.17g %.17g\n", blk[2 * i], blk[2 * i + 1]);
      out.append(tmp, (size_t)m);
    }
  }
  if (buf && cap >= (int64_t)out.size()) std::memcpy(buf, out.data(), out.size());
  return (int64_t)out.size();
}

int hood_validate_points(const double* xy, int64_t n, int64_t* ijk) {
  if (ijk) ijk[0] = ijk[1] = ijk[2] = 0;
  if (n < 2 || (n & (n - 1)) != 0) {
    if (ijk) ijk[0] = n;
    return HOOD_ERR_NOT_POWER_OF_TWO;
  }
  if (!xy) return HOOD_ERR_INVALID_ARG;
  for (int64_t i = 0; i < n; ++i) {
    const double x = xy[2 * i];
    if (!(x > 0.0 && x < 1.0)) {
      if (ijk) ijk[0] = i;
      return HOOD_ERR_X_OUT_OF_RANGE;
    }
    if (i > 0 && !(x > xy[2 * (i - 1)])) {
      if (ijk) ijk[0] = i;
      return HOOD_ERR_X_NOT_INCREASING;
    }
  }
  auto bad = [&](uint64_t i, uint64_t j, uint64_t k) {
    // orient(pts[k], pts[i], pts[j]) as the reference's check_triple
    return std::fabs(orient(xy + 2 * k, xy + 2 * i, xy + 2 * j)) < kCollinearMargin;
  };
  auto report = [&](uint64_t i, uint64_t j, uint64_t k) {
    if (ijk) {
      ijk[0] = (int64_t)i;
      ijk[1] = (int64_t)j;
      ijk[2] = (int64_t)k;
    }
    return HOOD_ERR_DEGENERATE_TRIPLE;
  };
  const uint64_t un = (uint64_t)n;
  if (un <= 64) {
    for (uint64_t i = 0; i + 2 < un; ++i)
      for (uint64_t j = i + 1; j + 1 < un; ++j)
        for (uint64_t k = j + 1; k < un; ++k)
          if (bad(i, j, k)) return report(i, j, k);
  } else {
    for (uint64_t i = 0; i + 2 < un; ++i)
      if (bad(i, i + 1, i + 2)) return report(i, i + 1, i + 2);
    // the reference's deterministic sample: mt19937_64 seeded with the
    // golden-ratio constant xor n, three uniform picks per triple
    std::mt19937_64 rng(0x9e3779b97f4a7c15ull ^ un);
    std::uniform_int_distribution<std::size_t> pick(0, un - 1);
    for (uint64_t s = 0; s < 10 * un; ++s) {
      const uint64_t a = pick(rng), b = pick(rng), c = pick(rng);
      if (a == b || b == c || a == c) continue;
      if (bad(a, b, c)) return report(a, b, c);
    }
  }
  return HOOD_OK;
}

}  // extern "C"
