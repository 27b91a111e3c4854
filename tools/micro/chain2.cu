// Serial monotone chain variants over 48 points in smem, one thread: cycles
// per point for (a) double predicate, (b) float filter + exact fallback,
// (c) (b) with the stack top in registers and q prefetched.
#include <cstdio>
__device__ __forceinline__ bool above_d(double ax, double ay, double bx, double by, double cx, double cy) {
  const double t1 = __dmul_rn(__dsub_rn(cx, ax), __dsub_rn(by, ay));
  const double t2 = __dmul_rn(__dsub_rn(cy, ay), __dsub_rn(bx, ax));
  return t1 > t2;
}
__device__ __noinline__ bool above_slow(float ax, float ay, float bx, float by, float cx, float cy) {
  return above_d(ax, ay, bx, by, cx, cy);
}
__device__ __forceinline__ bool above_f(float2 a, float2 b, float2 c) {
  const float t1 = __fmul_rn(__fsub_rn(c.x, a.x), __fsub_rn(b.y, a.y));
  const float t2 = __fmul_rn(__fsub_rn(c.y, a.y), __fsub_rn(b.x, a.x));
  const float det = __fsub_rn(t1, t2);
  const float bound = __fmaf_rn(4.76837158203125e-07f, __fadd_rn(fabsf(t1), fabsf(t2)), 1.0e-36f);
  if (det > bound) return true;
  if (det < -bound) return false;
  return above_slow(a.x, a.y, b.x, b.y, c.x, c.y);
}
__global__ void k(const float2* in, int m, long long* t, int* out) {
  __shared__ float2 runf[64], Hf[64];
  __shared__ double2 run[64], H[64];
  if (threadIdx.x < m) { runf[threadIdx.x] = in[threadIdx.x]; run[threadIdx.x] = make_double2(in[threadIdx.x].x, in[threadIdx.x].y); }
  __syncthreads();
  if (threadIdx.x) return;
  for (int rep = 0; rep < 2; ++rep) {
    long long a = clock64();
    int h = 0;
    double2 h1 = make_double2(0, 0), h2 = h1;
    for (int e = 0; e < m; ++e) {
      const double2 q = run[e];
      while (h >= 2 && !above_d(h2.x, h2.y, h1.x, h1.y, q.x, q.y)) { --h; h1 = h2; if (h >= 2) h2 = H[h - 2]; }
      H[h] = q; ++h; h2 = h1; h1 = q;
    }
    long long b = clock64();
    int hf = 0;
    float2 f1 = make_float2(0, 0), f2 = f1;
    for (int e = 0; e < m; ++e) {
      const float2 q = runf[e];
      while (hf >= 2 && !above_f(f2, f1, q)) { --hf; f1 = f2; if (hf >= 2) f2 = Hf[hf - 2]; }
      Hf[hf] = q; ++hf; f2 = f1; f1 = q;
    }
    long long c = clock64();
    int hg = 0;
    float2 g1 = make_float2(0, 0), g2 = g1, q = runf[0];
    for (int e = 0; e < m; ++e) {
      const float2 qn = runf[e + 1 < m ? e + 1 : e];
      bool pop = hg >= 2 && !above_f(g2, g1, q);
      while (pop) { --hg; g1 = g2; g2 = hg >= 2 ? Hf[hg - 2] : g2; pop = hg >= 2 && !above_f(g2, g1, q); }
      Hf[hg] = q; ++hg; g2 = g1; g1 = q; q = qn;
    }
    long long d = clock64();
    t[3 * rep] = b - a; t[3 * rep + 1] = c - b; t[3 * rep + 2] = d - c;
    out[0] = h; out[1] = hf; out[2] = hg;
  }
}
int main() {
  const int m = 48;
  float2 p[m];
  for (int i = 0; i < m; ++i) { float x = (i + 0.5f) / m; p[i] = make_float2(x, 0.9f + 0.1f * x * (1 - x) + ((i % 3) ? 0 : -0.004f)); }
  float2* d; long long* t; int* o;
  cudaMalloc(&d, sizeof p); cudaMalloc(&t, 48); cudaMalloc(&o, 12);
  cudaMemcpy(d, p, sizeof p, cudaMemcpyHostToDevice);
  k<<<1, 64>>>(d, m, t, o);
  long long ht[6]; int ho[3];
  cudaMemcpy(ht, t, 48, cudaMemcpyDeviceToHost); cudaMemcpy(ho, o, 12, cudaMemcpyDeviceToHost);
  printf("48 points (warm): double %.1f, float filter %.1f, float filter + prefetch %.1f cycles/point; hulls %d %d %d\n",
         ht[3] / 48.0, ht[4] / 48.0, ht[5] / 48.0, ho[0], ho[1], ho[2]);
}
