// Dependent-chain latencies on this GPU: FADD, DADD, DMUL, F2F.F64.F32, LDS.
#include <cstdio>
__global__ void k(double* out, long long* t, float fin, double din) {
  __shared__ double sh[64];
  sh[threadIdx.x] = din;
  __syncthreads();
  float f = fin; double d = din; double e = din;
  long long a = clock64();
#pragma unroll 1
  for (int i = 0; i < 125; ++i) { f = __fadd_rn(f, 1e-7f); f = __fadd_rn(f, 1e-7f); f = __fadd_rn(f, 1e-7f); f = __fadd_rn(f, 1e-7f); f = __fadd_rn(f, 1e-7f); f = __fadd_rn(f, 1e-7f); f = __fadd_rn(f, 1e-7f); f = __fadd_rn(f, 1e-7f); }
  long long b = clock64();
#pragma unroll 1
  for (int i = 0; i < 125; ++i) { d = __dadd_rn(d, 1e-9); d = __dadd_rn(d, 1e-9); d = __dadd_rn(d, 1e-9); d = __dadd_rn(d, 1e-9); d = __dadd_rn(d, 1e-9); d = __dadd_rn(d, 1e-9); d = __dadd_rn(d, 1e-9); d = __dadd_rn(d, 1e-9); }
  long long c = clock64();
#pragma unroll 1
  for (int i = 0; i < 125; ++i) { e = __dmul_rn(e, 1.0000001); e = __dmul_rn(e, 1.0000001); e = __dmul_rn(e, 1.0000001); e = __dmul_rn(e, 1.0000001); e = __dmul_rn(e, 1.0000001); e = __dmul_rn(e, 1.0000001); e = __dmul_rn(e, 1.0000001); e = __dmul_rn(e, 1.0000001); }
  long long g = clock64();
  double h = 0; float ff = fin;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { h = (double)ff; ff = (float)h + 1e-7f; }
  long long m = clock64();
  int idx = 0;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) idx = (int)sh[idx & 63] & 63;
  long long z = clock64();
  out[0] = f + d + e + h + idx;
  t[0] = (b - a); t[1] = (c - b); t[2] = (g - c); t[3] = m - g; t[4] = z - m;
}
int main() {
  double* o; long long* t; cudaMalloc(&o, 8); cudaMalloc(&t, 64);
  k<<<1, 32>>>(o, t, 1.0f, 1.0);
  long long h[5]; cudaMemcpy(h, t, 40, cudaMemcpyDeviceToHost);
  printf("per-iteration cycles: FADD %.1f  DADD %.1f  DMUL %.1f  F2F+FADD %.1f  LDS-chase %.1f\n",
         h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0, h[3] / 1000.0, h[4] / 1000.0);
}
