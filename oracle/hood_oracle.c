/*
 * TEST INFRASTRUCTURE ONLY -- see hood_oracle.h.  CPU restatement of the
 * reference algorithm; never linked into the product library.
 * Build: gcc -O2 -ffp-contract=off (oracle/Makefile).  No -march=native: the
 * reference is built for plain x86-64 with FMA disabled.
 */
#include "hood_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#if defined(__FP_FAST_FMA) && !defined(HOOD_ORACLE_ALLOW_FMA)
#error "oracle must be compiled without FMA contraction"
#endif

/* geom.hpp:22-24 */
double oracle_orient(const double* r, const double* p, const double* q) {
  return (q[0] - p[0]) * (r[1] - p[1]) - (q[1] - p[1]) * (r[0] - p[0]);
}

/* geom.hpp:26-28 */
int oracle_left_of(const double* r, const double* p, const double* q) {
  return oracle_orient(r, p, q) > 0.0;
}

static int is_remote(const double* p) { return p[0] > 1.0; } /* geom.hpp:18 */

/* oracle.cpp:7-20: the stack lives in out_xy. */
int64_t oracle_upper_hull_f64(const double* xy, int64_t n, double* out) {
  int64_t h = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double* p = xy + 2 * i;
    while (h >= 2 && !oracle_left_of(out + 2 * (h - 1), out + 2 * (h - 2), p)) --h;
    out[2 * h] = p[0];
    out[2 * h + 1] = p[1];
    ++h;
  }
  return h;
}

static int left_of_f32(const float* r, const float* p, const float* q) {
  const double rr[2] = {r[0], r[1]}, pp[2] = {p[0], p[1]}, qq[2] = {q[0], q[1]};
  return oracle_left_of(rr, pp, qq);
}

int64_t oracle_upper_hull_f32(const float* xy, int64_t n, float* out) {
  int64_t h = 0;
  for (int64_t i = 0; i < n; ++i) {
    const float* p = xy + 2 * i;
    while (h >= 2 && !left_of_f32(out + 2 * (h - 1), out + 2 * (h - 2), p)) --h;
    out[2 * h] = p[0];
    out[2 * h + 1] = p[1];
    ++h;
  }
  return h;
}

void oracle_block_hulls_f64(const double* xy, int64_t n, int64_t block,
                            double* out, int32_t* counts, int pad_remote) {
  for (int64_t b = 0; b * block < n; ++b) {
    const int64_t s = b * block;
    const int64_t len = (n - s < block) ? (n - s) : block;
    const int64_t h = oracle_upper_hull_f64(xy + 2 * s, len, out + 2 * s);
    counts[b] = (int32_t)h;
    if (pad_remote)
      for (int64_t k = h; k < len; ++k) {
        out[2 * (s + k)] = ORACLE_REMOTE_X;
        out[2 * (s + k) + 1] = ORACLE_REMOTE_Y;
      }
  }
}

void oracle_block_hulls_f32(const float* xy, int64_t n, int64_t block,
                            float* out, int32_t* counts, int pad_remote) {
  for (int64_t b = 0; b * block < n; ++b) {
    const int64_t s = b * block;
    const int64_t len = (n - s < block) ? (n - s) : block;
    const int64_t h = oracle_upper_hull_f32(xy + 2 * s, len, out + 2 * s);
    counts[b] = (int32_t)h;
    if (pad_remote)
      for (int64_t k = h; k < len; ++k) {
        out[2 * (s + k)] = (float)ORACLE_REMOTE_X;
        out[2 * (s + k) + 1] = (float)ORACLE_REMOTE_Y;
      }
  }
}

/* ---- slab-parallel all-core baseline --------------------------------- */

typedef struct {
  const void* xy;
  void* out;
  int64_t n;
  int64_t h;
  int f32;
} slab_job;

static void* slab_worker(void* arg) {
  slab_job* j = (slab_job*)arg;
  if (j->f32)
    j->h = oracle_upper_hull_f32((const float*)j->xy, j->n, (float*)j->out);
  else
    j->h = oracle_upper_hull_f64((const double*)j->xy, j->n, (double*)j->out);
  return NULL;
}

static int64_t hull_mt(const void* xy, int64_t n, int threads, void* out, int f32) {
  const size_t esz = f32 ? 2 * sizeof(float) : 2 * sizeof(double);
  if (threads < 1) threads = 1;
  if (threads > n / 2 + 1) threads = (int)(n / 2 + 1);
  if (threads <= 1)
    return f32 ? oracle_upper_hull_f32((const float*)xy, n, (float*)out)
               : oracle_upper_hull_f64((const double*)xy, n, (double*)out);
  slab_job* jobs = (slab_job*)calloc((size_t)threads, sizeof(slab_job));
  pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  void* tmp = malloc((size_t)n * esz);
  for (int t = 0; t < threads; ++t) {
    const int64_t lo = n * t / threads, hi = n * (t + 1) / threads;
    jobs[t].xy = (const char*)xy + lo * esz;
    jobs[t].out = (char*)tmp + lo * esz;
    jobs[t].n = hi - lo;
    jobs[t].f32 = f32;
    pthread_create(&tid[t], NULL, slab_worker, &jobs[t]);
  }
  int64_t total = 0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(tid[t], NULL);
    memmove((char*)tmp + total * esz, jobs[t].out, (size_t)jobs[t].h * esz);
    total += jobs[t].h;
  }
  const int64_t h = f32 ? oracle_upper_hull_f32((const float*)tmp, total, (float*)out)
                        : oracle_upper_hull_f64((const double*)tmp, total, (double*)out);
  free(tmp);
  free(tid);
  free(jobs);
  return h;
}

int64_t oracle_upper_hull_mt_f64(const double* xy, int64_t n, int threads, double* out) {
  return hull_mt(xy, n, threads, out, 0);
}

int64_t oracle_upper_hull_mt_f32(const float* xy, int64_t n, int threads, float* out) {
  return hull_mt(xy, n, threads, out, 1);
}

/* ---- brute tangents (oracle.cpp:22-71) -------------------------------- */

int64_t oracle_brute_tangent_to_right(const double* p, const double* hull, int64_t k) {
  int64_t found = k;
  int candidates = 0;
  for (int64_t t = 0; t < k; ++t) {
    int others_below = 1;
    for (int64_t o = 0; o < k; ++o)
      if (o != t && oracle_orient(hull + 2 * o, p, hull + 2 * t) >= 0.0) {
        others_below = 0;
        break;
      }
    if (others_below) {
      found = t;
      ++candidates;
    }
  }
  return candidates == 1 ? found : -1;
}

int oracle_brute_common_tangent(const double* p, int64_t m, const double* q, int64_t k,
                                int64_t* a_out, int64_t* b_out) {
  int64_t fa = m, fb = k;
  int candidates = 0;
  for (int64_t a = 0; a < m; ++a)
    for (int64_t b = 0; b < k; ++b) {
      int others_below = 1;
      for (int64_t o = 0; o < m && others_below; ++o)
        if (o != a && oracle_orient(p + 2 * o, p + 2 * a, q + 2 * b) >= 0.0) others_below = 0;
      for (int64_t o = 0; o < k && others_below; ++o)
        if (o != b && oracle_orient(q + 2 * o, p + 2 * a, q + 2 * b) >= 0.0) others_below = 0;
      if (others_below) {
        fa = a;
        fb = b;
        ++candidates;
      }
    }
  *a_out = fa;
  *b_out = fb;
  return candidates == 1 ? 0 : -1;
}

/* ---- classifiers (kernel.hpp:31-67) ----------------------------------- */

int oracle_classify_g(const double* hood, int i, int j, int start, int d) {
  if (is_remote(hood + 2 * j)) return 1;
  const double* p = hood + 2 * i;
  const double* q = hood + 2 * j;
  const int atend = (j == start + 2 * d - 1) || is_remote(hood + 2 * (j + 1));
  double qn[2] = {q[0], q[1]};
  if (atend) qn[1] -= 1.0;
  else { qn[0] = hood[2 * (j + 1)]; qn[1] = hood[2 * (j + 1) + 1]; }
  if (oracle_left_of(qn, p, q)) return -1;
  const int atstart = (j == start + d);
  double qp[2] = {q[0], q[1]};
  if (atstart) qp[1] -= 1.0;
  else { qp[0] = hood[2 * (j - 1)]; qp[1] = hood[2 * (j - 1) + 1]; }
  return oracle_left_of(qp, p, q) ? 1 : 0;
}

int oracle_classify_f(const double* hood, int i, int j, int start, int d) {
  if (is_remote(hood + 2 * i)) return 1;
  const double* p = hood + 2 * i;
  const double* q = hood + 2 * j;
  const int atend = (i == start + d - 1) || is_remote(hood + 2 * (i + 1));
  double pn[2] = {p[0], p[1]};
  if (atend) pn[1] -= 1.0;
  else { pn[0] = hood[2 * (i + 1)]; pn[1] = hood[2 * (i + 1) + 1]; }
  if (oracle_left_of(pn, p, q)) return -1;
  const int atstart = (i == start);
  double pp[2] = {p[0], p[1]};
  if (atstart) pp[1] -= 1.0;
  else { pp[0] = hood[2 * (i - 1)]; pp[1] = hood[2 * (i - 1) + 1]; }
  return oracle_left_of(pp, p, q) ? 1 : 0;
}

/* ---- driver.cpp:5-17 --------------------------------------------------- */

int oracle_round_schedule(int n, int32_t* rounds4, int cap) {
  int d1 = 2, d2 = 1, r = 1, count = 0;
  for (int d = d1 * d2; d < n; d = d1 * d2) {
    if (count < cap) {
      rounds4[4 * count + 0] = r;
      rounds4[4 * count + 1] = d1;
      rounds4[4 * count + 2] = d2;
      rounds4[4 * count + 3] = d;
    }
    ++count;
    if (d1 > d2) d2 *= 2;
    else d1 *= 2;
    ++r;
  }
  return count;
}

/* ---- hoodbuf.cpp:30-70 (without the sampled triples) ------------------- */

int oracle_validate_points(const double* xy, int64_t n, int64_t* bad) {
  *bad = 0;
  if (n < 2 || (n & (n - 1)) != 0) { *bad = n; return 1; }
  for (int64_t i = 0; i < n; ++i) {
    if (!(xy[2 * i] > 0.0 && xy[2 * i] < 1.0)) { *bad = i; return 2; }
    if (i > 0 && !(xy[2 * i] > xy[2 * (i - 1)])) { *bad = i; return 3; }
  }
  const double margin = 1e-9; /* kCollinearMargin, hoodbuf.hpp:16 */
  if (n <= 64) {
    for (int64_t i = 0; i + 2 < n; ++i)
      for (int64_t j = i + 1; j + 1 < n; ++j)
        for (int64_t k = j + 1; k < n; ++k)
          if (fabs(oracle_orient(xy + 2 * k, xy + 2 * i, xy + 2 * j)) < margin) {
            *bad = i; return 4;
          }
  } else {
    for (int64_t i = 0; i + 2 < n; ++i)
      if (fabs(oracle_orient(xy + 2 * (i + 2), xy + 2 * i, xy + 2 * (i + 1))) < margin) {
        *bad = i; return 4;
      }
  }
  return 0;
}
