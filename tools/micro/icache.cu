// Cold instruction fetch: one warp runs 4096 straight-line independent FADDs
// twice; the first pass fetches the code, the second runs it from the I-cache.
#include <cstdio>
template <int N>
__device__ __forceinline__ float body(float a, float b) {
  float acc[8] = {a, a, a, a, a, a, a, a};
#pragma unroll
  for (int i = 0; i < N; ++i) acc[i & 7] = __fadd_rn(acc[i & 7], b);
  return acc[0] + acc[1] + acc[2] + acc[3] + acc[4] + acc[5] + acc[6] + acc[7];
}
__global__ void k(float a, float b, long long* t, float* out) {
  float r = 0;
  long long c[3];
  c[0] = clock64();
#pragma unroll 1
  for (int rep = 0; rep < 2; ++rep) {
    r += body<4096>(a + rep, b);
    c[rep + 1] = clock64();
  }
  if (threadIdx.x == 0) { t[0] = c[1] - c[0]; t[1] = c[2] - c[1]; out[0] = r; }
}
int main() {
  long long* t; float* o;
  cudaMalloc(&t, 16); cudaMalloc(&o, 4);
  k<<<1, 32>>>(1.0f, 1e-7f, t, o);
  long long h[2];
  cudaMemcpy(h, t, 16, cudaMemcpyDeviceToHost);
  printf("4096 straight-line FADD: cold %lld cycles (%.2f/instr), warm %lld cycles (%.2f/instr)\n",
         h[0], h[0] / 4096.0, h[1], h[1] / 4096.0);
}
