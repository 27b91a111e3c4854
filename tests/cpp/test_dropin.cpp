// Drop-in check of include/hood_b200.hpp from C++ (the reference's own
// language): the reference's Point2 layout in, hood::build_hood semantics out.
// Known answers are the reference's unit tests (file:line cited); random sets
// are checked against a local monotone chain with the reference predicate
// (oracle.cpp:7-20, geom.hpp:22-28).  Needs a GPU; run by tests/test_gpu_parity.py.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#include "hood_b200.hpp"

namespace {

struct Point2 {  // geom.hpp:7-12
  double x = 0.0, y = 0.0;
  friend bool operator==(const Point2&, const Point2&) = default;
};
struct Point2f {
  float x = 0.f, y = 0.f;
  friend bool operator==(const Point2f&, const Point2f&) = default;
};

template <class P>
bool left_of(P r, P p, P q) {  // geom.hpp:22-28, in double, no contraction
  const volatile double a = (double(q.x) - double(p.x)) * (double(r.y) - double(p.y));
  const volatile double b = (double(q.y) - double(p.y)) * (double(r.x) - double(p.x));
  return a - b > 0.0;
}

template <class P>
std::vector<P> chain(const std::vector<P>& pts) {  // oracle.cpp:7-20
  std::vector<P> h;
  for (const P& q : pts) {
    while (h.size() >= 2 && !left_of(h[h.size() - 1], h[h.size() - 2], q)) h.pop_back();
    h.push_back(q);
  }
  return h;
}

int failures = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);     \
      ++failures;                                                  \
    }                                                              \
  } while (0)

std::vector<Point2f> grid(std::int64_t n, std::uint64_t seed) {
  // x on the 2^-24 grid, strictly increasing; y on the same grid
  std::mt19937_64 g(seed);
  std::vector<Point2f> v(static_cast<std::size_t>(n));
  const std::int64_t step = (std::int64_t(1) << 24) / n;
  for (std::int64_t i = 0; i < n; ++i) {
    const std::int64_t r = step > 1 ? 1 + static_cast<std::int64_t>(g() % static_cast<std::uint64_t>(step - 1)) : 1;
    v[static_cast<std::size_t>(i)].x = static_cast<float>(std::ldexp(double(i * step + r), -24));
    v[static_cast<std::size_t>(i)].y = static_cast<float>(std::ldexp(double(1 + g() % ((1u << 24) - 1)), -24));
  }
  return v;
}

}  // namespace

int main() {
  using hood::b200::build_hood;
  // test_kernel.cpp:17-117 (E1): A, B, C, D -> all four corners
  {
    std::vector<Point2> e1{{0.1, 0.5}, {0.2, 0.6}, {0.6, 0.9}, {0.7, 0.2}};
    CHECK(build_hood(e1).hull == e1);
  }
  // test_kernel.cpp:127-132 / test_oracle.cpp:23-26: a cup keeps its endpoints
  {
    std::vector<Point2> cup{{0.1, 0.9}, {0.3, 0.3}, {0.6, 0.25}, {0.9, 0.8}};
    const auto h = build_hood(cup).hull;
    CHECK(h.size() == 2 && h[0] == cup[0] && h[1] == cup[3]);
  }
  // test_driver.cpp:36-42: two points are their own hood
  {
    std::vector<Point2> two{{0.25, 0.1}, {0.75, 0.9}};
    CHECK(build_hood(two).hull == two);
  }
  // test_driver.cpp:51-59: a concave parabola, every point a corner
  {
    std::vector<Point2> par;
    for (int k = 1; k <= 8; ++k) par.push_back({k / 9.0, (k / 9.0) * (1.0 - k / 9.0)});
    CHECK(build_hood(par).hull == par);
  }
  // random float-grid sets against the monotone chain, single and batched
  for (int lg = 4; lg <= 22; lg += 3) {
    const auto pts = grid(std::int64_t(1) << lg, 1000 + lg);
    CHECK(build_hood(pts).hull == chain(pts));
  }
  {
    const std::int64_t L = 1024, inst = 256;
    std::vector<Point2f> all;
    for (int i = 0; i < inst; ++i) {
      const auto g = grid(L, 77 + i);
      all.insert(all.end(), g.begin(), g.end());
    }
    hood::b200::BuildOptions o;
    o.block_len = L;
    const auto rep = build_hood(all, o);
    CHECK(static_cast<std::int64_t>(rep.instances.size()) == inst);
    for (int i = 0; i < inst; ++i) {
      std::vector<Point2f> one(all.begin() + i * L, all.begin() + (i + 1) * L);
      CHECK(rep.instances[static_cast<std::size_t>(i)] == chain(one));
    }
  }
  // double storage: an arc, every point a corner (config 3 shape)
  {
    std::vector<Point2> arc;
    const int n = 1 << 16;
    for (int i = 0; i < n; ++i) {
      const double x = (i + 0.5) / n;
      arc.push_back({x, 0.25 + x * (1 - x)});
    }
    CHECK(build_hood(arc).hull == chain(arc));
  }
  // validate_points' errors (hoodbuf.cpp:48-58) surface as ValidationError
  {
    auto pts = grid(4096, 5);
    pts[1234].x = pts[1233].x;
    bool thrown = false;
    try {
      build_hood(pts);
    } catch (const hood::b200::ValidationError& e) {
      thrown = e.code == hood::b200::ValidationError::Code::x_not_increasing && e.i == 1234;
    }
    CHECK(thrown);
    auto r = grid(64, 6);
    r[10].x = 1.5f;
    r[11].x = 1.6f;
    for (std::size_t i = 12; i < r.size(); ++i) r[i].x = 1.7f + 0.01f * float(i);
    hood::b200::BuildOptions o;
    o.check_range = true;
    thrown = false;
    try {
      build_hood(r, o);
    } catch (const hood::b200::ValidationError& e) {
      thrown = e.code == hood::b200::ValidationError::Code::x_out_of_range && e.i == 10;
    }
    CHECK(thrown);
  }
  // the reference's point-file front end (cli.cpp:62-106) feeding the build
  {
    const std::string text = "# E1\n4\n0.1 0.5\n0.2 0.6\n0.6 0.9\n0.7 0.2\n";
    const auto pts = hood::b200::parse_points(text);
    hood::b200::validate_points(std::span<const hood::b200::Point2d>(pts));
    CHECK(build_hood(pts).hull == pts);
    CHECK(hood::b200::parse_points(hood::b200::format_points(std::span<const hood::b200::Point2d>(pts))) == pts);
    bool thrown = false;
    try {
      hood::b200::parse_points("3\n0.1 0.2\n0.3");
    } catch (const hood::b200::ParseError& e) {
      thrown = e.line == 3;
    }
    CHECK(thrown);
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
