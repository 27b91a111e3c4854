// Serial monotone chain over 48 double2 points in smem, one thread: cycles per
// point (the finalize chain's cost model).
#include <cstdio>
__device__ __forceinline__ bool above_d(double ax, double ay, double bx, double by, double cx, double cy) {
  const double t1 = __dmul_rn(__dsub_rn(cx, ax), __dsub_rn(by, ay));
  const double t2 = __dmul_rn(__dsub_rn(cy, ay), __dsub_rn(bx, ax));
  return t1 > t2;
}
__global__ void k(const double2* in, int m, long long* t, int* out) {
  __shared__ double2 run[64], H[64];
  if (threadIdx.x < m) run[threadIdx.x] = in[threadIdx.x];
  __syncthreads();
  if (threadIdx.x) return;
  for (int rep = 0; rep < 2; ++rep) {
    long long a = clock64();
    int h = 0, pred = 0;
    double2 h1 = make_double2(0, 0), h2 = h1;
    for (int e = 0; e < m; ++e) {
      const double2 q = run[e];
      while (h >= 2 && (++pred, !above_d(h2.x, h2.y, h1.x, h1.y, q.x, q.y))) {
        --h; h1 = h2; if (h >= 2) h2 = H[h - 2];
      }
      H[h] = q; ++h; h2 = h1; h1 = q;
    }
    long long b = clock64();
    t[rep] = b - a; out[0] = h; out[1] = pred;
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
  printf("chain of %d points: %lld / %lld cycles (cold/warm), hull %d, predicates %d -> %.1f cycles/point\n", m, ht[0], ht[1], ho[0], ho[1], (double)ht[1] / m);
}
