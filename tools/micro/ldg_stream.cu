// Microbenchmark: LDG.128 register streaming (per-warp contiguous ranges,
// software-pipelined) vs. size -- the alternative to the TMA ring.  Not part of
// the library.
#include <cuda_runtime.h>
#include <cstdio>

template <int U, int NB>
__global__ void __launch_bounds__(256) ldg_stream(const float4* __restrict__ in, long long n16, float* sink) {
  const int lane = threadIdx.x & 31;
  const long long gw = (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const long long nw = (long long)gridDim.x * (blockDim.x / 32);
  const long long blk = 32LL * U;                 // float4 per warp-block
  const long long nblk = n16 / blk;
  const long long per = (nblk + nw - 1) / nw;
  const long long b0 = gw * per, b1 = min(nblk, b0 + per);
  float acc = 0.f;
  float4 buf[NB][U];
#pragma unroll
  for (int s = 0; s < NB - 1; ++s)
    if (b0 + s < b1)
#pragma unroll
      for (int j = 0; j < U; ++j) buf[s][j] = __ldcs(in + (b0 + s) * blk + j * 32 + lane);
  for (long long b = b0; b < b1; b += NB) {
#pragma unroll
    for (int s = 0; s < NB; ++s) {
      const long long nb = b + s + NB - 1;
      if (nb < b1)
#pragma unroll
        for (int j = 0; j < U; ++j) buf[(s + NB - 1) % NB][j] = __ldcs(in + nb * blk + j * 32 + lane);
      if (b + s < b1)
#pragma unroll
        for (int j = 0; j < U; ++j) acc = fmaxf(acc, fmaxf(buf[s][j].y, buf[s][j].w));
    }
  }
  if (acc == 12345.f) sink[0] = acc;
}

template <int U, int NB>
void run(const float4* buf, size_t bytes, int blocks_per_sm, int sms) {
  float* sink; cudaMalloc(&sink, 4);
  void* fl; cudaMalloc(&fl, 256 << 20);
  float best = 1e9;
  for (int it = 0; it < 6; ++it) {
    cudaMemset(fl, it, 256 << 20);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    ldg_stream<U, NB><<<sms * blocks_per_sm, 256>>>(buf, bytes / 16, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (it > 0 && ms < best) best = ms;
  }
  printf("LDG U=%d NB=%d blocks/sm=%d %5zu MB: %.1f us  %.0f GB/s  %s\n", U, NB, blocks_per_sm, bytes >> 20,
         best * 1e3, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(sink); cudaFree(fl);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t big = 1ull << 31; float4* b2; cudaMalloc(&b2, big); cudaMemset(b2, 1, big);
  for (size_t mb : {32, 64, 128, 256, 1024}) {
    run<4, 3>(b2, mb << 20, 2, sms);
    run<4, 3>(b2, mb << 20, 4, sms);
    run<8, 2>(b2, mb << 20, 3, sms);
    run<4, 4>(b2, mb << 20, 3, sms);
  }
  return 0;
}
