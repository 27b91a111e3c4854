// hood_b200.hpp -- header-only C++ face of the C-ABI in hood_b200.h, shaped
// like the reference entry point it replaces:
//
//     hood::build_hood(const PointSet&, const BuildOptions&) -> BuildReport
//         (/root/reference/proj/include/hood/driver.hpp:27-45)
//     hood::oracle::upper_hull(std::span<const Point2>) -> std::vector<Point2>
//         (/root/reference/proj/include/hood/oracle.hpp:23)
//
// A caller holding the reference's points (any standard-layout {double x, y}
// struct, e.g. hood::Point2 from geom.hpp:7-12, or a {float x, y} pair for the
// float2 storage) swaps the call for hood::b200::build_hood(points) and gets
// the same corners, left to right, bit-identical to input points.  Errors are
// C++ exceptions like the reference's: ValidationError for x not strictly
// increasing / out of (0, 1) (hoodbuf.hpp:18-32), CudaError for device
// failures.  Not thread-safe per context; each thread gets its own
// (thread_local) context per device, matching the reference's reentrancy.
#pragma once

#include <cstddef>
#include <cstdint>
#include <fstream>
#include <iterator>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "hood_b200.h"

namespace hood::b200 {

struct ValidationError : std::runtime_error {
  // The subset of hood::ValidationError::Code (hoodbuf.hpp:19-24) the device
  // build checks; not_power_of_two and degenerate_triple are host-side
  // validate_points concerns the build does not need.
  enum class Code { x_out_of_range, x_not_increasing };
  ValidationError(Code c, std::size_t index, std::string msg)
      : std::runtime_error(std::move(msg)), code(c), i(index) {}
  Code code;
  std::size_t i;
};

struct ParseError : std::runtime_error {  // cli.hpp:23-28
  ParseError(const std::string& where, long long line)
      : std::runtime_error(where + ":" + std::to_string(line) + ": parse error"), line(line) {}
  long long line;
};

struct CudaError : std::runtime_error {
  CudaError(int status, int cuda_error, std::string msg)
      : std::runtime_error(std::move(msg)), status(status), cuda_error(cuda_error) {}
  int status;
  int cuda_error;
};

struct BuildOptions {
  int device = 0;
  // 0: one instance over all points.  Otherwise a power of two dividing n:
  // n / block_len independent instances (batched build; the reference's
  // round blocks of length d).
  std::int64_t block_len = 0;
  // validate_points' x in (0, 1) (hoodbuf.cpp:30-70); x strictly increasing
  // is always checked.
  bool check_range = false;
};

template <class P>
struct BuildReport {
  std::vector<P> hull;                   // instance 0 (the whole set when block_len == 0)
  std::vector<std::vector<P>> instances;  // every instance, when block_len splits the input
};

namespace detail {

template <class P>
using scalar_t = std::remove_cv_t<decltype(P::x)>;

template <class P>
constexpr void check_layout() {
  using S = scalar_t<P>;
  static_assert(std::is_same_v<S, double> || std::is_same_v<S, float>, "points must be {double x, y} or {float x, y}");
  static_assert(std::is_same_v<std::remove_cv_t<decltype(P::y)>, S>, "x and y must share a type");
  static_assert(std::is_standard_layout_v<P> && sizeof(P) == 2 * sizeof(S), "points must be packed {x, y} pairs");
}

inline void throw_status(hood_ctx* ctx, int rc) {
  hood_error e{rc, 0, -1};
  if (rc == HOOD_ERR_X_NOT_INCREASING || rc == HOOD_ERR_X_OUT_OF_RANGE || rc == HOOD_ERR_CUDA) hood_last_error(ctx, &e);
  if (e.code == HOOD_OK) e.code = rc;
  switch (e.code) {
    case HOOD_ERR_X_NOT_INCREASING:
      throw ValidationError(ValidationError::Code::x_not_increasing, static_cast<std::size_t>(e.index),
                            "x not strictly increasing at point " + std::to_string(e.index));
    case HOOD_ERR_X_OUT_OF_RANGE:
      throw ValidationError(ValidationError::Code::x_out_of_range, static_cast<std::size_t>(e.index),
                            "x outside (0, 1) at point " + std::to_string(e.index));
    default:
      throw CudaError(e.code, e.cuda_error, std::string("hood_b200: ") + hood_status_string(e.code));
  }
}

// One context per device per host thread.
inline hood_ctx* context(int device) {
  struct Holder {
    std::vector<hood_ctx*> ctx;
    ~Holder() {
      for (hood_ctx* c : ctx)
        if (c) hood_destroy(c);
    }
  };
  thread_local Holder h;
  if (device < 0) throw std::invalid_argument("hood_b200: negative device");
  if (h.ctx.size() <= static_cast<std::size_t>(device)) h.ctx.resize(static_cast<std::size_t>(device) + 1, nullptr);
  hood_ctx*& c = h.ctx[static_cast<std::size_t>(device)];
  if (!c) {
    const int rc = hood_create(&c, device);
    if (rc != HOOD_OK) {
      c = nullptr;
      throw CudaError(rc, 0, std::string("hood_b200: hood_create failed: ") + hood_status_string(rc));
    }
  }
  return c;
}

}  // namespace detail

// Upper hood of x-sorted points: the drop-in for hood::build_hood's hull
// (driver.hpp:43-45) and hood::oracle::upper_hull (oracle.hpp:23).
template <class P>
BuildReport<P> build_hood(std::span<const P> points, const BuildOptions& opt = {}) {
  detail::check_layout<P>();
  using S = detail::scalar_t<P>;
  BuildReport<P> rep;
  const std::int64_t n = static_cast<std::int64_t>(points.size());
  if (n == 0) return rep;
  const std::int64_t L = (opt.block_len <= 0 || opt.block_len == n) ? n : opt.block_len;
  if (n % L != 0) throw std::invalid_argument("hood_b200: block_len must divide the point count");
  const std::int64_t inst = n / L;
  hood_ctx* ctx = detail::context(opt.device);
  std::vector<P> corners(static_cast<std::size_t>(n));
  std::vector<std::int32_t> counts(static_cast<std::size_t>(inst));
  const std::uint32_t flags = opt.check_range ? HOOD_FLAG_CHECK_RANGE : 0u;
  int rc;
  if constexpr (std::is_same_v<S, double>)
    rc = hood_build_host_f64(ctx, reinterpret_cast<const double*>(points.data()), n, L == n ? 0 : L,
                             reinterpret_cast<double*>(corners.data()), counts.data(), flags);
  else
    rc = hood_build_host_f32(ctx, reinterpret_cast<const float*>(points.data()), n, L == n ? 0 : L,
                             reinterpret_cast<float*>(corners.data()), counts.data(), flags);
  if (rc != HOOD_OK) detail::throw_status(ctx, rc);
  hood_error e{};
  if (hood_last_error(ctx, &e) != HOOD_OK) detail::throw_status(ctx, e.code);
  if (inst == 1) {
    corners.resize(static_cast<std::size_t>(counts[0]));
    rep.hull = std::move(corners);
    return rep;
  }
  rep.instances.resize(static_cast<std::size_t>(inst));
  for (std::int64_t i = 0; i < inst; ++i) {
    const auto* b = corners.data() + i * L;
    rep.instances[static_cast<std::size_t>(i)].assign(b, b + counts[static_cast<std::size_t>(i)]);
  }
  rep.hull = rep.instances[0];
  return rep;
}

template <class P>
BuildReport<P> build_hood(const std::vector<P>& points, const BuildOptions& opt = {}) {
  return build_hood(std::span<const P>(points), opt);
}

// hood::oracle::upper_hull's signature (oracle.hpp:23).
template <class P>
std::vector<P> upper_hull(std::span<const P> points, int device = 0) {
  BuildOptions o;
  o.device = device;
  return build_hood(points, o).hull;
}

// ---- point files (cli.cpp:56-106) and validate_points (hoodbuf.cpp:30-70) ----

struct Point2d {
  double x = 0.0, y = 0.0;
  friend bool operator==(const Point2d&, const Point2d&) = default;
};

// validate_points: throws ValidationError (x_out_of_range / x_not_increasing
// carry the index; not_power_of_two and degenerate_triple are reported through
// std::invalid_argument with the reference's wording).
template <class P>
void validate_points(std::span<const P> pts) {
  detail::check_layout<P>();
  static_assert(std::is_same_v<detail::scalar_t<P>, double>, "validate_points takes {double x, y}");
  std::int64_t ijk[3];
  const int rc = hood_validate_points(reinterpret_cast<const double*>(pts.data()), (std::int64_t)pts.size(), ijk);
  if (rc == HOOD_OK) return;
  if (rc == HOOD_ERR_X_OUT_OF_RANGE)
    throw ValidationError(ValidationError::Code::x_out_of_range, (std::size_t)ijk[0],
                          "point " + std::to_string(ijk[0]) + " has x outside (0, 1)");
  if (rc == HOOD_ERR_X_NOT_INCREASING)
    throw ValidationError(ValidationError::Code::x_not_increasing, (std::size_t)ijk[0],
                          "point " + std::to_string(ijk[0]) + " does not increase in x over its predecessor");
  if (rc == HOOD_ERR_NOT_POWER_OF_TWO)
    throw std::invalid_argument("point count " + std::to_string(ijk[0]) + " is not a power of 2 (or is < 2)");
  throw std::invalid_argument("points " + std::to_string(ijk[0]) + ", " + std::to_string(ijk[1]) + ", " +
                              std::to_string(ijk[2]) + " are collinear within margin");
}

// parse_points (no validation): the point count, then x y pairs.
inline std::vector<Point2d> parse_points(const std::string& text, const std::string& where = "<stream>") {
  std::int64_t n = 0, line = 0;
  int rc = hood_parse_points(text.data(), (std::int64_t)text.size(), nullptr, 0, &n, &line);
  if (rc == HOOD_ERR_PARSE) throw ParseError(where, line);
  std::vector<Point2d> pts((std::size_t)n);
  rc = hood_parse_points(text.data(), (std::int64_t)text.size(), reinterpret_cast<double*>(pts.data()), n, &n,
                         &line);
  if (rc == HOOD_ERR_PARSE) throw ParseError(where, line);
  if (rc != HOOD_OK) throw std::runtime_error(std::string("hood_b200: ") + hood_status_string(rc));
  return pts;
}

// read_points = parse + validate (cli.cpp:56-60).
inline std::vector<Point2d> read_points(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("can't open " + path);
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  auto pts = parse_points(text, path);
  validate_points(std::span<const Point2d>(pts));
  return pts;
}

// write_point_set's text (cli.cpp:101-106, "%.17g").
template <class P>
std::string format_points(std::span<const P> pts) {
  detail::check_layout<P>();
  static_assert(std::is_same_v<detail::scalar_t<P>, double>, "format_points takes {double x, y}");
  const auto* xy = reinterpret_cast<const double*>(pts.data());
  const std::int64_t len = hood_format_points(xy, (std::int64_t)pts.size(), nullptr, 0);
  std::string s((std::size_t)len, '\0');
  hood_format_points(xy, (std::int64_t)pts.size(), s.data(), len);
  return s;
}

// write_section / write_trace_round (cli.cpp:47-52, 108-118).
template <class P>
std::string format_section(const std::string& label, std::span<const P> pts) {
  detail::check_layout<P>();
  static_assert(std::is_same_v<detail::scalar_t<P>, double>, "format_section takes {double x, y}");
  const auto* xy = reinterpret_cast<const double*>(pts.data());
  const std::int64_t len = hood_format_section(label.c_str(), xy, (std::int64_t)pts.size(), nullptr, 0);
  std::string s((std::size_t)len, '\0');
  hood_format_section(label.c_str(), xy, (std::int64_t)pts.size(), s.data(), len);
  return s;
}

// The trace file of build_hood under the CLI's on_round_begin observer
// (cli.cpp:163-169), the round loop run on the GPU.
template <class P>
void write_trace(const std::string& path, std::span<const P> pts, int device = 0) {
  detail::check_layout<P>();
  static_assert(std::is_same_v<detail::scalar_t<P>, double>, "write_trace takes {double x, y}");
  hood_ctx* ctx = detail::context(device);
  const int rc = hood_write_trace_f64(ctx, reinterpret_cast<const double*>(pts.data()), (std::int64_t)pts.size(),
                                      path.c_str());
  if (rc != HOOD_OK) throw std::runtime_error(std::string("hood_b200: write_trace: ") + hood_status_string(rc));
}

}  // namespace hood::b200
