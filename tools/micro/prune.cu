// warp_hull_small (iterated pruning, one warp) vs the serial monotone chain on
// the same 48 double2 points: cycles for the whole hull.
#include <cstdio>
__device__ __forceinline__ bool above(const double2& a, const double2& b, const double2& c) {
  const double t1 = __dmul_rn(__dsub_rn(c.x, a.x), __dsub_rn(b.y, a.y));
  const double t2 = __dmul_rn(__dsub_rn(c.y, a.y), __dsub_rn(b.x, a.x));
  return t1 > t2;
}
template <class V>
__device__ __forceinline__ int warp_hull_small(const V* P, int m, V* dst, int* rounds) {
  const int lane = threadIdx.x & 31;
  const int i0 = lane, i1 = lane + 32;
  const V q0 = i0 < m ? P[i0] : V{}, q1 = i1 < m ? P[i1] : V{};
  unsigned long long alive = m >= 64 ? ~0ull : ((1ull << m) - 1ull);
  auto keep = [&](int i, const V& q) -> bool {
    if (!((alive >> i) & 1ull)) return false;
    const unsigned long long lo = alive & ((1ull << i) - 1ull);
    const unsigned long long hi = i == 63 ? 0ull : (alive & ~((2ull << i) - 1ull));
    if (!lo || !hi) return true;
    return above(P[63 - __clzll(lo)], q, P[__ffsll(hi) - 1]);
  };
  int r = 0;
  for (;;) {
    const bool k0 = keep(i0, q0);
    const bool k1 = m > 32 ? keep(i1, q1) : false;
    const unsigned long long nxt = (unsigned long long)__ballot_sync(0xffffffffu, k0) |
                                   ((unsigned long long)__ballot_sync(0xffffffffu, k1) << 32);
    ++r;
    if (nxt == alive) break;
    alive = nxt;
  }
  __syncwarp();
  if ((alive >> i0) & 1ull) dst[__popcll(alive & ((1ull << i0) - 1ull))] = q0;
  if (m > 32 && ((alive >> i1) & 1ull)) dst[__popcll(alive & ((1ull << i1) - 1ull))] = q1;
  __syncwarp();
  *rounds = r;
  return __popcll(alive);
}
__global__ void k(const double2* in, int m, long long* t, int* out) {
  __shared__ double2 run[64], H[64];
  if (threadIdx.x < m) run[threadIdx.x] = in[threadIdx.x];
  __syncthreads();
  if (threadIdx.x >= 32) return;
  for (int rep = 0; rep < 2; ++rep) {
    __syncwarp();
    long long a = clock64();
    int rounds;
    const int h = warp_hull_small<double2>(run, m, H, &rounds);
    long long b = clock64();
    if (threadIdx.x == 0) { t[rep] = b - a; out[0] = h; out[1] = rounds; }
  }
}
int main() {
  const int m = 48;
  double2 p[m];
  for (int i = 0; i < m; ++i) { double x = (i + 0.5) / m; p[i] = make_double2(x, 0.9 + 0.1 * x * (1 - x) + ((i % 3) ? 0 : -0.004)); }
  double2* d; long long* t; int* o;
  cudaMalloc(&d, sizeof p); cudaMalloc(&t, 16); cudaMalloc(&o, 8);
  cudaMemcpy(d, p, sizeof p, cudaMemcpyHostToDevice);
  k<<<1, 64>>>(d, m, t, o);
  long long ht[2]; int ho[2];
  cudaMemcpy(ht, t, 16, cudaMemcpyDeviceToHost); cudaMemcpy(ho, o, 8, cudaMemcpyDeviceToHost);
  printf("warp_hull_small on 48 points: %lld / %lld cycles (cold/warm), hull %d, %d rounds\n", ht[0], ht[1], ho[0], ho[1]);
}
