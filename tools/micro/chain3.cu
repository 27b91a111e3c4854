// Monotone chain with the stack top in registers (4-deep shift window; the
// smem stack only sees the window's bottom) vs the plain smem stack.
#include <cstdio>
__device__ __forceinline__ bool above_d(double2 a, double2 b, double2 c) {
  const double t1 = __dmul_rn(__dsub_rn(c.x, a.x), __dsub_rn(b.y, a.y));
  const double t2 = __dmul_rn(__dsub_rn(c.y, a.y), __dsub_rn(b.x, a.x));
  return t1 > t2;
}
__global__ void k(const double2* in, int m, long long* t, int* out) {
  __shared__ double2 run[64], H[64], H2[64];
  if (threadIdx.x < m) run[threadIdx.x] = in[threadIdx.x];
  __syncthreads();
  if (threadIdx.x) return;
  for (int rep = 0; rep < 2; ++rep) {
    long long a = clock64();
    int h = 0;
    double2 h1 = make_double2(0, 0), h2 = h1;
    for (int e = 0; e < m; ++e) {
      const double2 q = run[e];
      while (h >= 2 && !above_d(h2, h1, q)) { --h; h1 = h2; if (h >= 2) h2 = H[h - 2]; }
      H[h] = q; ++h; h2 = h1; h1 = q;
    }
    long long b = clock64();
    // window: w0 = top (index h-1), w1 = h-2, w2 = h-3, w3 = h-4; H2[0..h-5] below
    int g = 0;
    double2 w0 = make_double2(0, 0), w1 = w0, w2 = w0, w3 = w0;
    double2 q = run[0];
    for (int e = 0; e < m; ++e) {
      const double2 qn = run[e + 1 < m ? e + 1 : e];
      while (g >= 2 && !above_d(w1, w0, q)) {
        --g;
        w0 = w1; w1 = w2; w2 = w3;
        if (g >= 4) w3 = H2[g - 4];
      }
      if (g >= 4) H2[g - 4] = w3;
      w3 = w2; w2 = w1; w1 = w0; w0 = q; ++g;
      q = qn;
    }
    // flush the window
    long long c = clock64();
    t[2 * rep] = b - a; t[2 * rep + 1] = c - b;
    out[0] = h; out[1] = g;
  }
}
int main() {
  const int m = 48;
  double2 p[m];
  for (int i = 0; i < m; ++i) { double x = (i + 0.5) / m; p[i] = make_double2(x, 0.9 + 0.1 * x * (1 - x) + ((i % 3) ? 0 : -0.004)); }
  double2* d; long long* t; int* o;
  cudaMalloc(&d, sizeof p); cudaMalloc(&t, 32); cudaMalloc(&o, 8);
  cudaMemcpy(d, p, sizeof p, cudaMemcpyHostToDevice);
  k<<<1, 64>>>(d, m, t, o);
  long long ht[4]; int ho[2];
  cudaMemcpy(ht, t, 32, cudaMemcpyDeviceToHost); cudaMemcpy(ho, o, 8, cudaMemcpyDeviceToHost);
  printf("48 points (warm): smem stack %.1f, register window %.1f cycles/point; hulls %d %d\n", ht[2] / 48.0, ht[3] / 48.0, ho[0], ho[1]);
}
