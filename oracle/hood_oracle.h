/*
 * TEST INFRASTRUCTURE ONLY -- parity oracle for the upper-hood hot path.
 *
 * A plain-C restatement of the reference CPU algorithm (arxiv/paper_1203_5004,
 * reference tree mounted at /root/reference/proj).  Only tests/, the smoke()
 * check in __graft_entry__.py and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  The product (libhood_b200.so) never links or
 * calls it.
 *
 * Parity is pinned two ways (see tests/test_oracle_golden.py):
 *   - the known-answer vectors of the reference's own tests
 *     (proj/tests/test_oracle.cpp, test_kernel.cpp, test_driver.cpp,
 *     acceptance.cpp, tests/data/sample8.txt), restated in pytest;
 *   - fixtures produced by the reference itself (tests/golden/ fixtures, generated
 *     by tests/golden/make_golden.py against oracle/_ref/libhoodref.so, which
 *     is compiled from the unmodified reference sources by oracle/Makefile).
 *
 * Every arithmetic step follows proj/include/hood/geom.hpp:22-28 exactly:
 * orient = (q.x-p.x)*(r.y-p.y) - (q.y-p.y)*(r.x-p.x) in IEEE double, each
 * operation separately rounded (this file is compiled with -ffp-contract=off).
 */
#ifndef HOOD_ORACLE_H
#define HOOD_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* REMOTE sentinel (geom.hpp:14): x = 10, y = 0; a slot is unused iff x > 1. */
#define ORACLE_REMOTE_X 10.0
#define ORACLE_REMOTE_Y 0.0

/* geom.hpp:22-24 -- det(q - p, r - p). Points are {x, y} pairs. */
double oracle_orient(const double* r, const double* p, const double* q);
/* geom.hpp:26-28 */
int oracle_left_of(const double* r, const double* p, const double* q);

/* oracle.cpp:7-20 -- Andrew monotone chain on x-sorted points; pops while the
 * last corner is not strictly left of (second-to-last -> p).  Output corners
 * are copies of input points (bit-identical).  Returns the corner count. */
int64_t oracle_upper_hull_f64(const double* xy, int64_t n, double* out_xy);
/* The same algorithm on float storage: coordinates promoted to double before
 * the predicate (the reference's Point2 is double; float inputs are exactly
 * representable).  Output corners are the original floats. */
int64_t oracle_upper_hull_f32(const float* xy, int64_t n, float* out_xy);

/* Independent hull of every consecutive block of `block` points (the last
 * block may be short when n % block != 0).  Block b's corners are written to
 * out_xy[b*block ...] and, if `pad_remote`, the rest of the block is filled
 * with the REMOTE sentinel -- the HoodBuffer layout of
 * hoodbuf.hpp:57-79 after the round with interval length `block`
 * (test_driver.cpp:72-94 pins round blocks == oracle(interval)). */
void oracle_block_hulls_f64(const double* xy, int64_t n, int64_t block,
                            double* out_xy, int32_t* counts, int pad_remote);
void oracle_block_hulls_f32(const float* xy, int64_t n, int64_t block,
                            float* out_xy, int32_t* counts, int pad_remote);

/* Slab-parallel hull: T contiguous slabs hulled on T pthreads, then the hull
 * of the concatenated slab hulls (identical to the monolithic
 * hull).  Used only as the all-core CPU baseline ("port" kind). */
int64_t oracle_upper_hull_mt_f64(const double* xy, int64_t n, int threads,
                                 double* out_xy);
int64_t oracle_upper_hull_mt_f32(const float* xy, int64_t n, int threads,
                                 float* out_xy);

/* oracle.cpp:22-43 -- index of the corner of `hull` supporting the tangent
 * from p, by exhaustion; -1 when not unique (NoUniqueTangent). */
int64_t oracle_brute_tangent_to_right(const double* p, const double* hull,
                                      int64_t k);
/* oracle.cpp:45-71 -- (a, b) corner indices of the common upper tangent;
 * returns 0 on success, -1 when not unique. */
int oracle_brute_common_tangent(const double* p, int64_t m, const double* q,
                                int64_t k, int64_t* a, int64_t* b);

/* kernel.hpp:31-47 / :51-67 -- the reference kernel's classifiers on a
 * REMOTE-padded hood window [start, start+2d): -1 LOW, 0 EQUAL, +1 HIGH. */
int oracle_classify_g(const double* hood, int i, int j, int start, int d);
int oracle_classify_f(const double* hood, int i, int j, int start, int d);

/* driver.cpp:5-17 -- fills up to `cap` rounds {r, d1, d2, d}; returns the
 * number of rounds (log2 n - 1 for a power of two n). */
int oracle_round_schedule(int n, int32_t* rounds4, int cap);

/* hoodbuf.cpp:30-70 minus the mt19937_64-sampled triples (those need
 * libstdc++'s distribution; the boundary precondition is not on the timed
 * path).  Returns 0 valid, 1 not_power_of_two, 2 x_out_of_range,
 * 3 x_not_increasing, 4 degenerate_triple; *bad = first offending index. */
int oracle_validate_points(const double* xy, int64_t n, int64_t* bad);

#ifdef __cplusplus
}
#endif

#endif /* HOOD_ORACLE_H */
