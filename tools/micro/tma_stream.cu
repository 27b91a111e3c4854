// Microbenchmark: raw TMA 2D streaming throughput with the slab kernel's box
// shape (rows x 128 B, SWIZZLE_128B) vs. ring depth.  Not part of the library.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include "../../paper_1203_5004_b200/csrc/hood_device.cuh"
using namespace hood_b200;

template <int ROWS, int NS>
__global__ void stream_kernel(const __grid_constant__ CUtensorMap tmap, long long tiles, int* sink) {
  extern __shared__ unsigned char raw[];
  unsigned char* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[NS];
  constexpr int TB = ROWS * 128;
  if (threadIdx.x == 0) { for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1); fence_barrier_init(); }
  __syncthreads();
  const long long per = (tiles + gridDim.x - 1) / gridDim.x;
  const long long t0 = blockIdx.x * per, t1 = min(tiles, t0 + per);
  int acc = 0;
  if (threadIdx.x == 0) {
    long long issue = t0;
    for (int s = 0; s < NS && issue < t1; ++s, ++issue) {
      mbar_expect_tx(&full[s], TB);
      tma_load_2d(sm + s * TB, &tmap, 0, (int)(issue * ROWS), &full[s]);
    }
    for (long long t = t0, k = 0; t < t1; ++t, ++k) {
      const int s = k % NS;
      mbar_wait(&full[s], (k / NS) & 1);
      acc += sm[s * TB + (k & 127)];
      if (issue < t1) {
        fence_proxy_async();
        mbar_expect_tx(&full[s], TB);
        tma_load_2d(sm + s * TB, &tmap, 0, (int)(issue * ROWS), &full[s]);
        ++issue;
      }
    }
    sink[blockIdx.x] = acc;
  }
}

template <int ROWS, int NS>
void run(PFN_cuTensorMapEncodeTiled_v12000 enc, void* buf, size_t bytes, int sms, int ctas_per_sm) {
  CUtensorMap m;
  const cuuint64_t rows = bytes / 128;
  const cuuint64_t gdim[2] = {128, rows};
  const cuuint64_t gstride[1] = {128};
  const cuuint32_t box[2] = {128, ROWS};
  const cuuint32_t es[2] = {1, 1};
  enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, gdim, gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const size_t smem = (size_t)NS * ROWS * 128 + 1024;
  cudaFuncSetAttribute(stream_kernel<ROWS, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int* sink; cudaMalloc(&sink, 4096 * sizeof(int));
  void* fl; cudaMalloc(&fl, 256 << 20);
  const long long tiles = rows / ROWS;
  float best = 1e9;
  for (int it = 0; it < 6; ++it) {
    cudaMemset(fl, it, 256 << 20);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    stream_kernel<ROWS, NS><<<sms * ctas_per_sm, 32, smem>>>(m, tiles, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (it > 0 && ms < best) best = ms;
  }
  printf("rows %3d (%5d B) stages %2d ctas/sm %d : %.1f us  %.0f GB/s  err=%s\n", ROWS, ROWS * 128, NS, ctas_per_sm,
         best * 1e3, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(sink); cudaFree(fl);
}

int main() {
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = 128ull << 20;
  void* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 1, bytes);
  const size_t big = 1ull << 31; void* b2; cudaMalloc(&b2, big); cudaMemset(b2, 1, big);
  for (size_t mb : {16, 32, 64, 128, 256, 512, 1024, 2048}) run<128, 6>(enc, b2, mb << 20, sms, 2);
  for (size_t mb : {32, 128, 512}) run<128, 6>(enc, b2, mb << 20, sms, 1);
  return 0;
}
