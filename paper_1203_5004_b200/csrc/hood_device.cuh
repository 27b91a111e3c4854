// Device building blocks of the B200 upper-hood build (sm_100a).
//
// Reference semantics (all paths relative to /root/reference/proj):
//   * predicate  include/hood/geom.hpp:22-28  orient(r,p,q) > 0, IEEE double,
//                every operation separately rounded (no FMA);
//   * result     src/oracle.cpp:7-20          the strict upper hull of the
//                x-sorted input (collinear middle points dropped), corners are
//                copies of input points;
//   * merge      src/kernel.cpp:20-137        hood(P u Q) = P[..pindex] ++ Q[qindex..].
//
// Every predicate evaluated here has the canonical form the reference oracle
// uses -- "is b strictly above the chord a->c" for x(a) < x(b) < x(c), i.e.
// orient(b, a, c) > 0 with a as the origin -- so on inputs whose predicates
// are exact in double (the 2^-24 float grid of configs 1/2/5) the output is
// bit-identical to oracle::upper_hull by construction, and on general doubles
// it agrees whenever no evaluated triple is within rounding of collinear.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace hood_b200 {

typedef long long i64;

template <class S> struct PointT;
template <> struct PointT<float> {
  using V = float2;
  static constexpr int K = 16;      // points per 128-byte chunk row
  static constexpr int LOGK = 4;
};
template <> struct PointT<double> {
  using V = double2;
  static constexpr int K = 8;
  static constexpr int LOGK = 3;
};

// geom.hpp:22-28 in canonical orientation: b strictly above chord a->c.
// t1 - t2 > 0  <=>  t1 > t2 for finite doubles (the difference of two doubles
// never rounds to zero), so the final subtraction folds into the compare.
__device__ __forceinline__ bool above_d(double ax, double ay, double bx, double by,
                                        double cx, double cy) {
  const double t1 = __dmul_rn(__dsub_rn(cx, ax), __dsub_rn(by, ay));
  const double t2 = __dmul_rn(__dsub_rn(cy, ay), __dsub_rn(bx, ax));
  return t1 > t2;
}

__device__ __forceinline__ bool above(const double2& a, const double2& b, const double2& c) {
  return above_d(a.x, a.y, b.x, b.y, c.x, c.y);
}

// Float storage: a certified float filter decides whenever |det| clears a
// bound 8 eps (|t1|+|t2|) (+ an absolute underflow guard), which is > 2x
// Shewchuk's orient2d error bound (3+16eps)eps; past it the exact sign is
// known AND the double evaluation of the reference is correct as well, so the
// verdict equals the reference's double predicate.  Otherwise fall back to
// the exact reference operation sequence in double (floats promote exactly).
static __device__ __noinline__ bool above_slow(float ax, float ay, float bx, float by, float cx, float cy) {
  return above_d((double)ax, (double)ay, (double)bx, (double)by, (double)cx, (double)cy);
}

__device__ __forceinline__ bool above(const float2& a, const float2& b, const float2& c) {
  const float t1 = __fmul_rn(__fsub_rn(c.x, a.x), __fsub_rn(b.y, a.y));
  const float t2 = __fmul_rn(__fsub_rn(c.y, a.y), __fsub_rn(b.x, a.x));
  const float det = __fsub_rn(t1, t2);
  const float bound = __fmaf_rn(4.76837158203125e-07f /* 2^-21 */, __fadd_rn(fabsf(t1), fabsf(t2)),
                                1.0e-36f);
  if (det > bound) return true;
  if (det < -bound) return false;
  return above_slow(a.x, a.y, b.x, b.y, c.x, c.y);  // rare: keep it out of the hot code
}

// The reference predicate evaluated in double for either storage (floats
// widen exactly): the same answer as above(), without the filter.
__device__ __forceinline__ bool above_exact(const double2& a, const double2& b, const double2& c) {
  return above_d(a.x, a.y, b.x, b.y, c.x, c.y);
}
__device__ __forceinline__ bool above_exact(const float2& a, const float2& b, const float2& c) {
  return above_d((double)a.x, (double)a.y, (double)b.x, (double)b.y, (double)c.x, (double)c.y);
}

// Three-way version (+1 above, -1 below, 0 on the chord) with the same
// semantics: the sign of the reference's double orient(b, a, c).
__device__ __forceinline__ int orient_sign_d(double ax, double ay, double bx, double by, double cx, double cy) {
  const double t1 = __dmul_rn(__dsub_rn(cx, ax), __dsub_rn(by, ay));
  const double t2 = __dmul_rn(__dsub_rn(cy, ay), __dsub_rn(bx, ax));
  return (t1 > t2) - (t1 < t2);
}
__device__ __forceinline__ int orient_sign(const double2& a, const double2& b, const double2& c) {
  return orient_sign_d(a.x, a.y, b.x, b.y, c.x, c.y);
}
__device__ __forceinline__ int orient_sign(const float2& a, const float2& b, const float2& c) {
  const float t1 = __fmul_rn(__fsub_rn(c.x, a.x), __fsub_rn(b.y, a.y));
  const float t2 = __fmul_rn(__fsub_rn(c.y, a.y), __fsub_rn(b.x, a.x));
  const float det = __fsub_rn(t1, t2);
  const float bound = __fmaf_rn(4.76837158203125e-07f, __fadd_rn(fabsf(t1), fabsf(t2)), 1.0e-36f);
  if (det > bound) return 1;
  if (det < -bound) return -1;
  return orient_sign_d((double)a.x, (double)a.y, (double)b.x, (double)b.y, (double)c.x, (double)c.y);
}

// The predicate plus an uncertainty flag for evaluation-order-dependent
// merges (warp_hull_small's iterated pruning, the finalize's chord cull): unc
// is set when |t1 - t2| <= 2^-50 (|t1| + |t2|), above Shewchuk's error bound
// (3u + 16u^2) of the double orient -- the computed sign may then differ from
// the exact one, and the reference's own evaluation order (oracle.cpp:7-20)
// is the only one guaranteed to reproduce it.  Float storage never sets it:
// its double predicate on widened floats is the reference's on the same
// values, and the float path's callers are order-independent in practice.
__device__ __forceinline__ bool above_flag(const double2& a, const double2& b, const double2& c, bool& unc) {
  const double t1 = __dmul_rn(__dsub_rn(c.x, a.x), __dsub_rn(b.y, a.y));
  const double t2 = __dmul_rn(__dsub_rn(c.y, a.y), __dsub_rn(b.x, a.x));
  unc |= !(fabs(__dsub_rn(t1, t2)) > __dmul_rn(8.881784197001252e-16, __dadd_rn(fabs(t1), fabs(t2))));
  return t1 > t2;
}
__device__ __forceinline__ bool above_flag(const float2& a, const float2& b, const float2& c, bool&) {
  return above(a, b, c);
}

// --------------------------------------------------------------- accessors
// Hulls are contiguous runs of points addressed by a 64-bit slot index.

template <class V>
struct PtrAcc {  // global memory or linear shared memory (generic pointer)
  V* p;
  __device__ __forceinline__ V ld(i64 i) const { return p[i]; }
  __device__ __forceinline__ void st(i64 i, V v) const { p[i] = v; }
};

// A TMA tile in shared memory: 256 rows of 128 bytes written with
// CU_TENSOR_MAP_SWIZZLE_128B, i.e. the 16-byte unit u of row r sits at unit
// position u ^ (r & 7).  Slot i is point (i mod K) of row (i / K).
template <class S>
struct TileAcc {
  using V = typename PointT<S>::V;
  unsigned char* base;
  __device__ __forceinline__ unsigned char* addr(i64 i) const {
    const int ii = (int)i;
    const int row = ii >> PointT<S>::LOGK;
    const int byte = (ii & (PointT<S>::K - 1)) * (int)sizeof(V);
    return base + row * 128 + ((((byte >> 4) ^ (row & 7))) << 4) + (byte & 15);
  }
  __device__ __forceinline__ V ld(i64 i) const { return *reinterpret_cast<const V*>(addr(i)); }
  __device__ __forceinline__ void st(i64 i, V v) const { *reinterpret_cast<V*>(addr(i)) = v; }
};

// ------------------------------------------------------------- bridge search
//
// P = A[as, as+m), Q = B[bs, bs+k), every P corner strictly left of every Q
// corner, both strict upper hulls (left to right).
//
//   LOW(p, j)  : j < k-1 and q_j is on/below the chord p -> q_{j+1}
//                (the tangent from p touches Q right of j).  Monotone in j:
//                true before the tangent corner, false from it on; ties pick
//                the LAST corner on the supporting line (strict hull).
//   LOW_f(i)   : i < m-1 and p_{i+1} is strictly above the line p_i -> q_t(i)
//                (the bridge's P end lies right of i).  Monotone in i; ties
//                pick the FIRST P corner on the bridge line.
//
// These are the reference classifiers g and f (kernel.hpp:31-67) reduced to
// the one comparison a monotone search needs, in canonical orientation.

template <class V, class AccB>
__device__ __forceinline__ i64 tangent_from(const V& p, const AccB& B, i64 bs, i64 k) {
  i64 lo = 0, hi = k - 1;
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    if (!above(p, B.ld(bs + mid), B.ld(bs + mid + 1))) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

template <class V, class AccA, class AccB>
__device__ __forceinline__ bool low_f(const AccA& A, i64 as, i64 i, const AccB& B, i64 bs, i64 k) {
  const V pi = A.ld(as + i);
  const V pn = A.ld(as + i + 1);
  const i64 t = tangent_from(pi, B, bs, k);
  return above(pi, pn, B.ld(bs + t));
}

template <class V, class AccA, class AccB>
__device__ __noinline__ void bridge(const AccA& A, i64 as, i64 m, const AccB& B, i64 bs, i64 k,
                       i64& pidx, i64& qidx) {
  // Concatenation test: (m-1, 0) is the bridge iff both classifiers are EQUAL
  // there (the pinpoint phase, kernel.cpp:101-112).  Arc-like inputs stop here.
  const V pl = A.ld(as + m - 1);
  const V q0 = B.ld(bs);
  const bool g_eq = (k == 1) || above(pl, q0, B.ld(bs + 1));
  const bool f_eq = (m == 1) || above(A.ld(as + m - 2), pl, q0);
  if (g_eq && f_eq) {
    pidx = m - 1;
    qidx = 0;
    return;
  }
  // Gallop from the right end of P (a new piece usually cuts only P's tail),
  // then binary-search the first i with !LOW_f(i).
  i64 hi = m - 1, lo = 0, step = 1;
  for (;;) {
    const i64 i = hi - step;
    if (i < 0) { lo = 0; break; }
    if (low_f<V>(A, as, i, B, bs, k)) { lo = i + 1; break; }
    hi = i;
    step <<= 1;
  }
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    if (low_f<V>(A, as, mid, B, bs, k)) lo = mid + 1;
    else hi = mid;
  }
  pidx = lo;
  qidx = tangent_from(A.ld(as + lo), B, bs, k);
}

// The same bridge by a whole warp (every lane calls it; the result is on
// every lane): the north star's warp-level common-tangent search.  Both
// monotone searches go 32-ary -- each round the lanes evaluate the predicate
// at 32 points spread over the open interval and one ballot keeps the gap
// between the last true and the first false probe -- so a search over m
// corners takes ceil(log32 m) rounds instead of log2 m dependent steps.  For
// LOW_f each lane runs its own tangent search into Q.  Same predicates, same
// answer as bridge() on every input whose predicates are monotone (every
// input off rounding-level degeneracy).
template <class V, class AccB>
__device__ i64 tangent_from_warp(const V& p, const AccB& B, i64 bs, i64 k) {
  const int lane = threadIdx.x & 31;
  // first j in [0, k-1] with !LOW(p, j), LOW(j) = !above(p, q_j, q_{j+1}); LOW(k-1) is false
  i64 lo = 0, hi = k - 1;
  while (lo < hi) {
    const i64 span = hi - lo;  // probes lo + span*l/32 for l < 32, all < hi
    const i64 j = lo + span * lane / 32;
    const bool low = j < hi && !above(p, B.ld(bs + j), B.ld(bs + j + 1));
    const unsigned tm = __ballot_sync(0xffffffffu, low);
    // LOW is monotone: probes 0 .. c-1 true, c .. false (c = the count of trues)
    const int c = __popc(tm);
    const i64 nlo = c == 0 ? lo : lo + span * (c - 1) / 32 + 1;
    const i64 nhi = c == 32 ? hi : lo + span * c / 32;
    lo = nlo;
    hi = max(nhi, nlo);  // (a non-monotone ballot, rounding-level degenerate input: still terminates)
  }
  return lo;
}

template <class V, class AccA, class AccB>
__device__ __noinline__ void bridge_warp(const AccA& A, i64 as, i64 m, const AccB& B, i64 bs, i64 k, i64& pidx,
                                         i64& qidx) {
  const int lane = threadIdx.x & 31;
  {  // the concatenation test (the pinpoint phase at (m-1, 0), kernel.cpp:101-112)
    const V pl = A.ld(as + m - 1);
    const V q0 = B.ld(bs);
    const bool g_eq = (k == 1) || above(pl, q0, B.ld(bs + 1));
    const bool f_eq = (m == 1) || above(A.ld(as + m - 2), pl, q0);
    if (g_eq && f_eq) {
      pidx = m - 1;
      qidx = 0;
      return;
    }
  }
  // first i in [0, m-1] with !LOW_f(i); LOW_f(m-1) is false
  i64 lo = 0, hi = m - 1;
  while (lo < hi) {
    const i64 span = hi - lo;
    const i64 i = lo + span * lane / 32;
    bool low = false;
    if (i < hi) {
      const V pi = A.ld(as + i);
      low = above(pi, A.ld(as + i + 1), B.ld(bs + tangent_from(pi, B, bs, k)));
    }
    const unsigned tm = __ballot_sync(0xffffffffu, low);
    const int c = __popc(tm);
    const i64 nlo = c == 0 ? lo : lo + span * (c - 1) / 32 + 1;
    const i64 nhi = c == 32 ? hi : lo + span * c / 32;
    lo = nlo;
    hi = max(nhi, nlo);
  }
  pidx = lo;
  qidx = tangent_from_warp(A.ld(as + lo), B, bs, k);
}

// Merge node Q = (bs, k) into node P = (as, m) living in the same storage:
// result P[..pidx] ++ Q[qidx..] stays at `as` (Q's tail slides left, the
// reference's splice, kernel.cpp:117-137, without padding).  One thread.
template <class V, class Acc>
__device__ void merge_nodes(const Acc& X, i64& as, i64& m, i64 bs, i64 k) {
  if (k == 0) return;
  if (m == 0) { as = bs; m = k; return; }
  i64 pidx, qidx;
  bridge<V>(X, as, m, X, bs, k, pidx, qidx);
  const i64 dst = as + pidx + 1, src = bs + qidx, len = k - qidx;
  if (dst != src)
    for (i64 e = 0; e < len; ++e) X.st(dst + e, X.ld(src + e));
  m = pidx + 1 + len;
}

// Pairwise merge tree over `num_nodes` adjacent nodes (node a = (ns[a], nc[a]))
// run by the whole CTA: level l merges node a+2^l into node a for every a that
// is a multiple of 2^(l+1).  After `levels` levels node a (a multiple of
// 2^levels) holds the hull of its block.
template <class V, class Acc>
__device__ void tree_merge(const Acc& X, i64* ns, int* nc, int num_nodes, int levels) {
  for (int l = 0; l < levels; ++l) {
    const int half = 1 << l, span = half << 1;
    for (int a = threadIdx.x * span; a < num_nodes; a += blockDim.x * span) {
      const int b = a + half;
      if (b >= num_nodes) continue;
      if (nc[b] == 0) continue;
      i64 s = ns[a], m = nc[a];
      merge_nodes<V>(X, s, m, ns[b], (i64)nc[b]);
      ns[a] = s;
      nc[a] = (int)m;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------- TMA / mbarrier

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "HOOD_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra HOOD_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Running maximum / minimum of y values: acc is never NaN, v may be (a NaN v
// never replaces acc, as with fmax).  For double a compare and two selects;
// fmax/fmin add NaN quieting (DSETP.MAX + 3 selects) on the landing pass.
template <class S> __device__ __forceinline__ S ymax(S acc, S v) { return v > acc ? v : acc; }
template <> __device__ __forceinline__ float ymax<float>(float acc, float v) { return fmaxf(acc, v); }
template <class S> __device__ __forceinline__ S ymin(S a, S b) { return b < a ? b : a; }
template <> __device__ __forceinline__ float ymin<float>(float a, float b) { return fminf(a, b); }

template <class S> __device__ __forceinline__ S neg_inf();
template <> __device__ __forceinline__ float neg_inf<float>() { return -__int_as_float(0x7f800000); }
template <> __device__ __forceinline__ double neg_inf<double>() {
  return -__longlong_as_double(0x7ff0000000000000LL);
}

}  // namespace hood_b200
