// TEST / BASELINE INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference sources (compiled in place from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libhoodref.so).
// Nothing from the reference is copied here: this file only calls its public
// API (hood::oracle::upper_hull, hood::build_hood, the round-loop pieces and the
// test generators).  Loaded by tests/ (golden fixtures, oracle pinning) and by
// bench.py's reference arm / cpu_baseline.  Never linked into the product.
#include <cstdint>
#include <cstring>
#include <span>
#include <thread>
#include <vector>

#include <sstream>
#include <string>

#include "hood/cli.hpp"
#include "hood/driver.hpp"
#include "hood/hoodbuf.hpp"
#include "hood/kernel.hpp"
#include "hood/oracle.hpp"
#include "hood/psim.hpp"
#include "support/generators.hpp"

using hood::Point2;

namespace {

std::span<const Point2> as_points(const double* xy, int64_t n) {
  static_assert(sizeof(Point2) == 2 * sizeof(double));
  return {reinterpret_cast<const Point2*>(xy), static_cast<std::size_t>(n)};
}

int64_t emit(const std::vector<Point2>& h, double* out) {
  std::memcpy(out, h.data(), h.size() * sizeof(Point2));
  return static_cast<int64_t>(h.size());
}

}  // namespace

extern "C" {

// oracle.cpp:7-20 on one core.
int64_t ref_upper_hull(const double* xy, int64_t n, double* out) {
  return emit(hood::oracle::upper_hull(as_points(xy, n)), out);
}

// All-core variant built only from the reference's own function: T contiguous
// slabs on T threads, then upper_hull of the concatenated slab hulls
// (SURVEY.md A10 / BASELINE.md section 3 item 2).
int64_t ref_upper_hull_mt(const double* xy, int64_t n, int threads, double* out) {
  if (threads <= 1 || n < 4 * threads) return ref_upper_hull(xy, n, out);
  std::vector<std::vector<Point2>> parts(static_cast<std::size_t>(threads));
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      const int64_t lo = n * t / threads, hi = n * (t + 1) / threads;
      parts[static_cast<std::size_t>(t)] = hood::oracle::upper_hull(as_points(xy + 2 * lo, hi - lo));
    });
  }
  for (auto& th : pool) th.join();
  std::vector<Point2> cat;
  for (auto& p : parts) cat.insert(cat.end(), p.begin(), p.end());
  return emit(hood::oracle::upper_hull(cat), out);
}

// Batched: one upper_hull per `block` points, blocks spread over threads.
// Corners of block b land at out[2*b*block ...], counts[b] = corner count.
void ref_block_hulls_mt(const double* xy, int64_t n, int64_t block, int threads,
                        double* out, int32_t* counts) {
  const int64_t nb = (n + block - 1) / block;
  if (threads < 1) threads = 1;
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      for (int64_t b = t; b < nb; b += threads) {
        const int64_t s = b * block, len = std::min(block, n - s);
        counts[b] = static_cast<int32_t>(
            emit(hood::oracle::upper_hull(as_points(xy + 2 * s, len)), out + 2 * s));
      }
    });
  }
  for (auto& th : pool) th.join();
}

// tests/support/generators.hpp:32-43 (validated uniform points).
int ref_make_random_point_set(int n, uint64_t seed, double* out) {
  try {
    const hood::PointSet ps = hood::testsupport::make_random_point_set(n, seed);
    std::memcpy(out, ps.points().data(), static_cast<std::size_t>(n) * sizeof(Point2));
    return 0;
  } catch (...) {
    return -1;
  }
}

// hood::build_hood (driver.cpp:19-45) on a validated PointSet.  If
// `rounds_out` is non-null it receives the REMOTE-padded buffer after every
// round (n slots per round, on_round_end observer).  Returns the corner count,
// -1 on ValidationError, -2 on DegenerateTangent, -3 on other errors.
int64_t ref_build_hood(const double* xy, int64_t n, double* out, double* rounds_out,
                       int64_t* conflicts) {
  try {
    const hood::PointSet ps =
        hood::validate_points(std::vector<Point2>(as_points(xy, n).begin(), as_points(xy, n).end()));
    hood::BuildOptions opts;
    int64_t r = 0;
    if (rounds_out) {
      opts.on_round_end = [&](const hood::Round&, const hood::HoodBuffer& buf,
                              const hood::LaunchReport&) {
        std::memcpy(rounds_out + 2 * n * r, buf.slots().data(),
                    static_cast<std::size_t>(n) * sizeof(Point2));
        ++r;
      };
    }
    const hood::BuildReport rep = hood::build_hood(ps, opts);
    if (conflicts) *conflicts = static_cast<int64_t>(rep.conflicts);
    return emit(rep.hull, out);
  } catch (const hood::ValidationError&) {
    return -1;
  } catch (const hood::DegenerateTangent&) {
    return -2;
  } catch (...) {
    return -3;
  }
}

// The raw round loop of driver.cpp:20-43 driven through the reference's own
// HoodBuffer / MergeArrays / match_and_merge_kernel / launch, without
// validate_points (which rejects every random set with n >= 2^16).
int64_t ref_build_hood_raw(const double* xy, int64_t n, double* out) {
  try {
    hood::HoodBuffer buf(std::vector<Point2>(as_points(xy, n).begin(), as_points(xy, n).end()), 2);
    for (const hood::Round& round : hood::round_schedule(static_cast<int>(n))) {
      hood::MergeArrays arrays = hood::MergeArrays::for_round(std::move(buf).take_slots());
      const hood::PhaseKernel kernel =
          hood::match_and_merge_kernel(static_cast<int>(n), {round.d1, round.d2});
      const hood::LaunchReport rep = hood::launch(kernel, arrays);
      hood::require_tangents(rep, round.r);
      buf = hood::HoodBuffer(std::move(arrays.newhood), 2 * round.d);
    }
    return emit(buf.block_corners(0), out);
  } catch (const hood::DegenerateTangent&) {
    return -2;
  } catch (...) {
    return -3;
  }
}

// One match_and_merge block (kernel.cpp:177-187) on a 2d-slot window; writes
// newhood and scratch.  Returns 0, -2 on DegenerateTangent, -3 otherwise.
int ref_merge_block(const double* slots, int d1, int d2, double* newhood, int32_t* scratch) {
  try {
    const int n = 2 * d1 * d2;
    hood::MergeArrays m = hood::MergeArrays::for_round(
        std::vector<Point2>(as_points(slots, n).begin(), as_points(slots, n).end()));
    hood::match_and_merge_block(m, 0, {d1, d2});
    std::memcpy(newhood, m.newhood.data(), static_cast<std::size_t>(n) * sizeof(Point2));
    std::memcpy(scratch, m.scratch.data(), static_cast<std::size_t>(n) * sizeof(int32_t));
    return 0;
  } catch (const hood::DegenerateTangent&) {
    return -2;
  } catch (...) {
    return -3;
  }
}

// tests/support/generators.hpp:66-91: two padded hoods of interval length d.
int ref_make_random_hood_pair(int d, uint64_t seed, double* slots, int32_t* pq_counts) {
  try {
    const auto pair = hood::testsupport::make_random_hood_pair(d, seed);
    std::memcpy(slots, pair.arrays.hood.data(), static_cast<std::size_t>(2 * d) * sizeof(Point2));
    pq_counts[0] = static_cast<int32_t>(pair.p_corners.size());
    pq_counts[1] = static_cast<int32_t>(pair.q_corners.size());
    return 0;
  } catch (...) {
    return -1;
  }
}

// kernel.hpp:31-67 classifiers.
int ref_classify_g(const double* hood, int64_t len, int i, int j, int start, int d) {
  return static_cast<int>(hood::classify_g(as_points(hood, len), i, j, start, d));
}
int ref_classify_f(const double* hood, int64_t len, int i, int j, int start, int d) {
  return static_cast<int>(hood::classify_f(as_points(hood, len), i, j, start, d));
}


// cli.cpp:62-99 parse_points (which validates, hoodbuf.cpp:30-70).
// Returns 0 ok, 1 ParseError (line in *line), 2 ValidationError (code in
// *line: 0 not_power_of_two, 1 x_out_of_range, 2 x_not_increasing,
// 3 degenerate_triple; indices in ijk), 3 out of capacity.
int ref_parse_points(const char* text, int64_t len, double* xy, int64_t cap, int64_t* count, int64_t* line,
                     int64_t* ijk) {
  std::istringstream in(std::string(text, static_cast<std::size_t>(len)));
  try {
    const hood::PointSet ps = hood::cli::parse_points(in, "<text>");
    *count = ps.size();
    if (ps.size() > cap) return 3;
    std::memcpy(xy, ps.points().data(), static_cast<std::size_t>(ps.size()) * sizeof(Point2));
    return 0;
  } catch (const hood::cli::ParseError& e) {
    *line = e.line;
    return 1;
  } catch (const hood::ValidationError& e) {
    *line = static_cast<int64_t>(e.code);
    ijk[0] = static_cast<int64_t>(e.i);
    ijk[1] = static_cast<int64_t>(e.j);
    ijk[2] = static_cast<int64_t>(e.k);
    return 2;
  }
}

// hoodbuf.cpp:30-70 validate_points: -1 ok, else the ValidationError code.
int ref_validate_points(const double* xy, int64_t n, int64_t* ijk) {
  std::vector<Point2> v(as_points(xy, n).begin(), as_points(xy, n).end());
  try {
    hood::validate_points(std::move(v));
    return -1;
  } catch (const hood::ValidationError& e) {
    ijk[0] = static_cast<int64_t>(e.i);
    ijk[1] = static_cast<int64_t>(e.j);
    ijk[2] = static_cast<int64_t>(e.k);
    return static_cast<int>(e.code);
  }
}

// cli.cpp:96-100 format_coord (write_point_set prints "<n>\n" then
// "<format_coord(x)> <format_coord(y)>\n" per point, cli.cpp:101-106).  The
// stream-based writer itself is not called: libstdc++'s formatted output
// crashes inside a ctypes-loaded library on this image.
int ref_format_coord(double v, char* buf, int cap) {
  const std::string s = hood::cli::format_coord(v);
  if (static_cast<int>(s.size()) >= cap) return -1;
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return static_cast<int>(s.size());
}

}  // extern "C"
