// C-ABI of the B200 upper-hood build (include/hood_b200.h).
//
// Host-side mirror of the reference driver (driver.cpp:19-45): where the
// reference loops over log2(n)-1 rounds on the host, this layer plans ONE
// slab launch (+ one finalize launch when an instance spans several slabs)
// and never synchronizes inside a build, so builds can be captured into CUDA
// graphs and the reference's per-round host<->device traffic
// disappears.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>
#include <cstdio>
#include <cstdlib>

#include "../../include/hood_b200.h"
#include "hood_device.cuh"
#include "hood_kernels.cuh"

using namespace hood_b200;

namespace {
struct Stager;
}

struct hood_ctx {
  int device = 0;
  int sms = 148;
  // device workspace
  int* seg_cnt = nullptr;
  void* seg_apt = nullptr;  // double2-sized slots (fits float2 too)
  long long* seg_base = nullptr;
  long long seg_cap = 0;
  unsigned long long* steal_w = nullptr;  // per unit claim word (0xff.. = not stealable)
  int* steal_done = nullptr;              // per unit parts done (0 between builds)
  int* part_cnt = nullptr;                // per part (2 per unit)
  long long* part_base = nullptr;
  unsigned steal_epoch = 0;
  DevError* err = nullptr;
  unsigned* arrive = nullptr;  // finished-unit counter (ring kernel -> finalize), zero between builds
  void* warm = nullptr;        // the finalize's warm-up instance (kWarmBytes)
  int* done = nullptr;      // merge_records: result already written by the gather kernel
  double* rec = nullptr;    // build_multi: this context's exchange record (cap+1 double2)
  long long rec_cap = 0;
  double* gathered = nullptr;  // build_multi (first context): G records
  long long gathered_elems = 0;
  // host-path buffers
  void* d_in = nullptr;
  size_t d_in_bytes = 0;
  void* d_out = nullptr;
  size_t d_out_bytes = 0;
  int* d_counts = nullptr;
  long long d_counts_cap = 0;
  cudaStream_t s_copy = nullptr, s_comp = nullptr;
  static constexpr int kChunks = 8;
  cudaEvent_t ev[kChunks] = {};
  // bookkeeping
  cudaStream_t last_stream = nullptr;
  bool have_last = false;
  int last_launches = 0;
  int sticky_cuda = 0;
  cudaEvent_t prof_before = nullptr, prof_after = nullptr;
  cudaEvent_t order_ev = nullptr;  // orders a build on a new stream after the last one
  Stager* stager = nullptr;        // host path: pinned bounce buffers for pageable input
  void* round_tmp = nullptr;       // merge_round in place: a copy of the input
  size_t round_tmp_bytes = 0;
  int dbg = 0;
  long long* trace = nullptr;
};

namespace {

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode;
}

struct Plan {
  bool hmode = true;
  bool lean = false;
  long long n = 0, L = 0, instances = 1, tiles = 0, tpi = 0;
  int spi = 1;
  long long units = 0, tpu = 1;
  int grid = 0;
  int seg_chunks = 256;
  int rows = 256;       // chunk rows per tile (TMA box height)
  long long T = 0;      // points per tile
};

template <class S>
int make_plan(hood_ctx* ctx, long long n, long long block_len, Plan& pl) {
  constexpr int K = PointT<S>::K;
  if (n < 1) return HOOD_ERR_INVALID_ARG;
  pl.n = n;
  pl.L = (block_len <= 0 || block_len == n) ? n : block_len;
  if (pl.L != n) {
    if ((pl.L & (pl.L - 1)) != 0 || n % pl.L != 0 || pl.L < K) return HOOD_ERR_INVALID_ARG;
  }
  pl.instances = n / pl.L;
  const long long Th = (long long)slab_tile_rows<S>(true) * K;
  pl.hmode = (pl.L == n || pl.L >= Th);
  pl.rows = slab_tile_rows<S>(pl.hmode);
  const long long T = (long long)pl.rows * K;
  pl.T = T;
  pl.tiles = (n + T - 1) / T;
  if (pl.hmode) {
    // one unit (contiguous x-range) per warp of the slab kernel
    const long long nw = slab_warps_per_cta<S>();
    const long long ctas = (long long)slab_kernel_occupancy<S>() * ctx->sms;
    pl.seg_chunks = 32;
    pl.tpi = (pl.L + T - 1) / T;
    long long spi = ctas * nw / pl.instances;
    // units of at least kMinUnitBlocks blocks (1: small inputs spread over
    // as many warps as they have blocks) keep the per-unit overhead
    // (edge anchors, hood write-out, finalize candidates) small
    spi = std::min(spi, std::max(1LL, pl.tpi / kMinUnitBlocks));
    spi = std::max(1LL, std::min(spi, std::min(pl.tpi, (long long)kMaxSlabsPerInstance)));
    pl.spi = (int)spi;
    pl.units = pl.instances * pl.spi;
    if (pl.tpi >= (1LL << 31) || pl.units >= (1LL << 31)) return HOOD_ERR_CAPACITY;
    // batched builds (every unit a whole instance, more instances than warps)
    // run the register-light ring variant at higher occupancy
    pl.lean = pl.spi == 1 && pl.instances > 1 && ring_lean_available<S>();
    if (pl.lean && slab_tile_rows<S>(true, true) != pl.rows) {  // the LEAN variant's own block size
      pl.rows = slab_tile_rows<S>(true, true);
      pl.T = (long long)pl.rows * K;
      pl.tiles = (n + pl.T - 1) / pl.T;
      pl.tpi = (pl.L + pl.T - 1) / pl.T;
    }
    const long long ctas_run = pl.lean ? (long long)slab_kernel_occupancy<S>(true) * ctx->sms : ctas;
    pl.grid = (int)std::min((pl.units + nw - 1) / nw, ctas_run);
  } else {
    const long long resident = (long long)instance_kernel_occupancy<S>() * ctx->sms;
    pl.seg_chunks = (int)(pl.L / K);
    pl.tpu = std::max(1LL, (pl.tiles + resident - 1) / resident);
    pl.units = (pl.tiles + pl.tpu - 1) / pl.tpu;
    pl.grid = (int)std::min(pl.units, resident);
  }
  return HOOD_OK;
}

int ensure_ws(hood_ctx* ctx, long long slabs) {
  if (!ctx->err) {
    if (cudaMalloc(&ctx->err, sizeof(DevError)) != cudaSuccess) return HOOD_ERR_CUDA;
    if (cudaMalloc(&ctx->done, sizeof(int)) != cudaSuccess) return HOOD_ERR_CUDA;
    if (cudaMemset(ctx->err, 0xff, sizeof(DevError)) != cudaSuccess) return HOOD_ERR_CUDA;
    // [0] finished units, [1] full units (both zeroed by the finalize that
    // reads them), [2] steals so far (hood_internal_steals reads and zeroes it)
    if (cudaMalloc(&ctx->arrive, 4 * sizeof(unsigned)) != cudaSuccess) return HOOD_ERR_CUDA;
    if (cudaMemset(ctx->arrive, 0, 4 * sizeof(unsigned)) != cudaSuccess) return HOOD_ERR_CUDA;
    if (cudaMalloc(&ctx->warm, kWarmBytes) != cudaSuccess) return HOOD_ERR_CUDA;
    // zero counts until the first reset kernel writes the instance (same
    // bytes every build, so a finalize never reads a torn one)
    if (cudaMemset(ctx->warm, 0, kWarmBytes) != cudaSuccess) return HOOD_ERR_CUDA;
  }
  if (slabs > ctx->seg_cap) {
    cudaFree(ctx->seg_cnt);
    cudaFree(ctx->seg_apt);
    cudaFree(ctx->seg_base);
    cudaFree(ctx->steal_w);
    cudaFree(ctx->steal_done);
    cudaFree(ctx->part_cnt);
    cudaFree(ctx->part_base);
    const long long cap = std::max(slabs, 4096LL);
    if (cudaMalloc(&ctx->seg_cnt, cap * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&ctx->seg_apt, cap * 2 * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&ctx->seg_base, cap * sizeof(long long)) != cudaSuccess ||
        cudaMalloc(&ctx->steal_w, cap * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc(&ctx->steal_done, cap * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&ctx->part_cnt, kStealParts * cap * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&ctx->part_base, kStealParts * cap * sizeof(long long)) != cudaSuccess)
      return HOOD_ERR_CUDA;
    // claim words start "not stealable" (a stolen count != 0); every owner
    // resets its own word at the start of each build, and every build leaves
    // every word in a state no thief takes (fully claimed); part counts
    // start (and are left by every merge) at -1 = no such part
    if (cudaMemset(ctx->steal_w, 0xff, cap * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMemset(ctx->steal_done, 0, cap * sizeof(int)) != cudaSuccess ||
        cudaMemset(ctx->part_cnt, 0xff, kStealParts * cap * sizeof(int)) != cudaSuccess)
      return HOOD_ERR_CUDA;
    ctx->seg_cap = cap;
  }
  return HOOD_OK;
}

template <class S>
int encode_map(const void* pts, long long n, int box_rows, CUtensorMap* map, long long* full_rows) {
  constexpr int K = PointT<S>::K;
  *full_rows = n / K;
  std::memset(map, 0, sizeof(*map));
  if (*full_rows == 0) return HOOD_OK;
  auto enc = encoder();
  if (!enc) return HOOD_ERR_CUDA;
  const cuuint64_t gdim[2] = {128, (cuuint64_t)*full_rows};
  const cuuint64_t gstride[1] = {128};
  const cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(pts), gdim, gstride, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? HOOD_OK : HOOD_ERR_CUDA;
}

bool steal_enabled();
constexpr long long kStealMinUnitBlocks = 64;

template <class S>
SlabParams<S> slab_params(hood_ctx* ctx, const Plan& pl, const void* pts, void* corners, int* counts,
                          long long full_rows, uint32_t flags) {
  SlabParams<S> p{};
  p.pts = pts;
  p.n = pl.n;
  p.L = pl.L;
  p.log2L = 0;
  while ((1LL << p.log2L) < pl.L) ++p.log2L;
  p.hmode = pl.hmode ? 1 : 0;
  p.lean = pl.lean ? 1 : 0;
  p.seg_chunks = pl.seg_chunks;
  p.tiles_per_inst = pl.tpi;
  p.slabs_per_inst = pl.spi;
  p.num_units = pl.units;
  p.tiles_per_unit = pl.tpu;
  p.num_tiles = pl.tiles;
  p.unit_lo = 0;
  p.unit_hi = pl.units;
  p.full_rows = full_rows;
  p.out = corners;
  p.out_counts = counts;
  p.seg_cnt = ctx->seg_cnt;
  p.seg_apt = ctx->seg_apt;
  p.seg_base = ctx->seg_base;
  // tail stealing pays only on long units (config 4: ~590 blocks per unit;
  // on 9-18-block units it costs ~10%: profiles/r02/ab_steal.md)
  const bool long_units = pl.spi > 1 && pl.tpi / pl.spi >= kStealMinUnitBlocks;
  if (pl.hmode && long_units && !pl.lean && !(flags & HOOD_FLAG_CHECK_TRIPLES) && steal_enabled()) {
    ctx->steal_epoch = (ctx->steal_epoch + 1) % 0xffffu;  // 0xffff: the memset state, never an epoch
    p.steal_epoch = ctx->steal_epoch;
    p.steal_w = ctx->steal_w;
    p.steal_count = ctx->arrive + 2;
    p.steal_done = ctx->steal_done;
    p.part_cnt = ctx->part_cnt;
    p.part_base = ctx->part_base;
  }
  p.err = ctx->err;
  p.check_range = (flags & HOOD_FLAG_CHECK_RANGE) ? 1 : 0;
  p.check_triples = (flags & HOOD_FLAG_CHECK_TRIPLES) ? 1 : 0;
  p.dbg = ctx->dbg;
  p.trace = ctx->trace;
  p.read_lim = pl.n;
  return p;
}

template <class S>
FinalizeParams<S> finalize_params(hood_ctx* ctx, const Plan& pl, void* corners, int* counts) {
  using V = typename PointT<S>::V;
  FinalizeParams<S> f{};
  f.out = corners;
  f.out_counts = counts;
  f.seg_cnt = ctx->seg_cnt;
  f.seg_apt = ctx->seg_apt;
  f.seg_base = ctx->seg_base;
  f.seg_stride = 0;
  f.slabs_per_inst = pl.spi;
  f.L = pl.L;
  f.fcap = (int)(32768 / sizeof(V));  // 64 KB of survivor stack, as double2
  f.trace = ctx->trace ? ctx->trace + 7 * 64 : nullptr;
  return f;
}

// HOOD_DEBUG_SYNC=1: synchronize after every launch and name the failing one.
void debug_check(const char* what, cudaStream_t st) {
  static const bool on = [] {
    const char* e = std::getenv("HOOD_DEBUG_SYNC");
    return e && e[0] == '1';
  }();
  if (!on) return;
  const cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) std::fprintf(stderr, "[hood_b200] %s failed: %s\n", what, cudaGetErrorString(e));
}

// Event record that also works inside CUDA-graph capture (an external event
// node, so the replay timestamps it).
void record_event(cudaEvent_t ev, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal);
  else cudaEventRecord(ev, st);
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// HOOD_STEAL=0 turns tail stealing off (A/B and diagnosis only).
bool steal_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HOOD_STEAL");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  return cs != cudaStreamCaptureStatusNone;
}

// A context's workspace (unit summaries, error record, finished-unit counter)
// is reused by every build, so a build on another stream than the context's
// last one is ordered after it (an event edge).  Inside a graph capture the
// caller orders the replay; a capture-time edge to an uncaptured stream would
// invalidate the capture, so none is added there.
void order_after_last(hood_ctx* ctx, cudaStream_t st) {
  if (!ctx->have_last || ctx->last_stream == st) return;
  if (capturing(st) || capturing(ctx->last_stream)) return;
  if (!ctx->order_ev && cudaEventCreateWithFlags(&ctx->order_ev, cudaEventDisableTiming) != cudaSuccess) return;
  cudaEventRecord(ctx->order_ev, ctx->last_stream);
  cudaStreamWaitEvent(st, ctx->order_ev, 0);
}

template <class S>
int build_device(hood_ctx* ctx, const S* pts, long long n, long long block_len, S* corners, int* counts,
                 S* padded, uint32_t flags, cudaStream_t st) {
  if (!ctx || !pts || !corners || !counts) return HOOD_ERR_INVALID_ARG;
  if (!aligned16(pts) || !aligned16(corners)) return HOOD_ERR_INVALID_ARG;
  cudaSetDevice(ctx->device);
  Plan pl;
  int rc = make_plan<S>(ctx, n, block_len, pl);
  if (rc) return rc;
  if ((rc = ensure_ws(ctx, pl.units))) return rc;
  order_after_last(ctx, st);
  CUtensorMap map;
  long long full_rows = 0;
  std::memset(&map, 0, sizeof(map));  // the ring kernel (hmode) fills with cp.async, no tensor map
  if (!pl.hmode && (rc = encode_map<S>(pts, n, pl.rows, &map, &full_rows))) return rc;
  // the ring path resets the error record in-stream (launch_slab_kernel),
  // except under profile events, which bracket the ring kernel alone
  const bool reset_in_stream = pl.hmode && !ctx->prof_before;
  if (!reset_in_stream && cudaMemsetAsync(ctx->err, 0xff, sizeof(DevError), st) != cudaSuccess)
    return HOOD_ERR_CUDA;
  SlabParams<S> p = slab_params<S>(ctx, pl, pts, corners, counts, full_rows, flags);
  // single instance, PDL finalize: it starts on the finished-unit count
  const bool early = pl.hmode && pl.spi > 1 && pl.instances == 1 && !ctx->prof_after;
  p.arrive = early ? ctx->arrive : nullptr;
  p.full_units = (pl.hmode && pl.spi > 1 && pl.instances == 1) ? ctx->arrive + 1 : nullptr;
  if (ctx->prof_before) record_event(ctx->prof_before, st);
  // the finalize's warm-up merge pays only when its CTA is resident early,
  // i.e. when the ring grid leaves SMs free (small inputs: config 1 -10%);
  // on a full GPU it would run past the last unit and delay the real merge
  const bool warm_ok = (long long)pl.grid * 2 <= (long long)ctx->sms * slab_kernel_occupancy<S>(false);
  void* warm = (early && reset_in_stream && warm_ok) ? ctx->warm : nullptr;
  launch_slab_kernel<S>(p, &map, pl.grid, st, reset_in_stream, warm);
  debug_check("slab kernel", st);
  if (ctx->prof_after) record_event(ctx->prof_after, st);
  int launches = reset_in_stream ? 2 : 1;  // + the error-reset kernel
  if (pl.hmode && pl.spi > 1) {
    FinalizeParams<S> f = finalize_params<S>(ctx, pl, corners, counts);
    if (early) {
      f.arrive = ctx->arrive;
      f.arrive_target = (unsigned)pl.units;
      f.warm = warm;
    }
    if (pl.instances == 1) f.full_units = ctx->arrive + 1;
    launch_finalize<S>(f, (int)pl.instances, st, /*pdl=*/!ctx->prof_after);
    debug_check("finalize", st);
    ++launches;
  }
  if (padded) {
    launch_pad_fill<S>(padded, corners, counts, n, pl.L, st);
    debug_check("pad fill", st);
    ++launches;
  }
  const cudaError_t e = cudaGetLastError();
  ctx->last_stream = st;
  ctx->have_last = true;
  ctx->last_launches = launches;
  if (e != cudaSuccess) {
    ctx->sticky_cuda = (int)e;
    return HOOD_ERR_CUDA;
  }
  return HOOD_OK;
}

int decode_error(hood_ctx* ctx, hood_error* out) {
  hood_error e{HOOD_OK, 0, -1};
  if (ctx->sticky_cuda) {
    e.code = HOOD_ERR_CUDA;
    e.cuda_error = ctx->sticky_cuda;
    ctx->sticky_cuda = 0;
  } else if (ctx->have_last && ctx->err) {
    cudaError_t ce = cudaStreamSynchronize(ctx->last_stream);
    DevError de{~0ULL, -1, ~0ULL};
    if (ce == cudaSuccess) ce = cudaMemcpy(&de, ctx->err, sizeof(de), cudaMemcpyDeviceToHost);
    if (ce != cudaSuccess) {
      e.code = HOOD_ERR_CUDA;
      e.cuda_error = (int)ce;
    } else if (de.key != ~0ULL && de.key >= kTripleKey) {
      e.code = HOOD_ERR_DEGENERATE_TRIPLE;  // points (index, index+1, index+2)
      e.index = (int64_t)(de.key - kTripleKey);
    } else if (de.key != ~0ULL) {
      e.code = (de.key & 1ULL) ? HOOD_ERR_X_NOT_INCREASING : HOOD_ERR_X_OUT_OF_RANGE;
      e.index = (int64_t)(de.key >> 1);
    } else if (de.need >= 0) {
      e.code = HOOD_ERR_CAPACITY;  // an exchange record needed `need` corners
      e.index = (int64_t)de.need;
    } else if (de.degen != ~0ULL) {
      e.code = HOOD_ERR_DEGENERATE;  // hood_merge_round: block (pair) index
      e.index = (int64_t)de.degen;
    }
  }
  if (out) *out = e;
  return e.code;
}

template <class S>
int ensure_host_bufs(hood_ctx* ctx, long long n, long long instances) {
  const size_t bytes = (size_t)n * 2 * sizeof(S);
  if (bytes > ctx->d_in_bytes) {
    cudaFree(ctx->d_in);
    cudaFree(ctx->d_out);
    ctx->d_in = ctx->d_out = nullptr;
    if (cudaMalloc(&ctx->d_in, bytes) != cudaSuccess || cudaMalloc(&ctx->d_out, bytes) != cudaSuccess)
      return HOOD_ERR_CUDA;
    ctx->d_in_bytes = ctx->d_out_bytes = bytes;
  }
  if (instances > ctx->d_counts_cap) {
    cudaFree(ctx->d_counts);
    if (cudaMalloc(&ctx->d_counts, instances * sizeof(int)) != cudaSuccess) return HOOD_ERR_CUDA;
    ctx->d_counts_cap = instances;
  }
  if (!ctx->s_copy) {
    cudaStreamCreateWithFlags(&ctx->s_copy, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&ctx->s_comp, cudaStreamNonBlocking);
    for (auto& e : ctx->ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  }
  return HOOD_OK;
}

// Pageable host input (a std::vector): host threads copy it, chunk by chunk,
// into pinned bounce buffers owned by the context (two per thread, reused
// once the DMA that read them has finished) and each chunk goes to the device
// by DMA on the thread's own stream the moment it is staged; the build's
// kernels wait on the events of the chunks they read.  The copies from
// pageable memory -- the step the driver would otherwise do page by page
// through its own small staging buffer -- run at the host threads' aggregate
// memcpy bandwidth, overlapped with the PCIe transfer.
struct Stager {
  size_t chunk = 8u << 20;  // bytes per staged chunk (8 MiB measured best of 4-64 on B200 boxes)
  int threads = 0;
  std::vector<void*> bufs;              // 2 per thread, pinned (cudaHostAlloc), allocated on first use
  std::vector<cudaEvent_t> buf_ev;      // per buffer: the last DMA that read it
  std::vector<cudaStream_t> streams;    // per thread
  std::vector<cudaEvent_t> chunk_ev;    // per chunk of the current input: its DMA
};

bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();  // pageable memory on older runtimes: clear the error
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

int ensure_stager(hood_ctx* ctx, long long nchunks) {
  if (!ctx->stager) {
    ctx->stager = new Stager();
    const unsigned hw = std::thread::hardware_concurrency();
    int t = (int)std::max(1u, std::min(8u, hw ? hw / 2 : 4u));
    if (const char* e = std::getenv("HOOD_STAGE_THREADS")) t = std::max(1, std::min(64, std::atoi(e)));
    ctx->stager->threads = t;
    if (const char* e = std::getenv("HOOD_STAGE_CHUNK_MB")) ctx->stager->chunk = (size_t)std::max(1, std::atoi(e)) << 20;
  }
  Stager& sg = *ctx->stager;
  if (sg.streams.empty()) {
    sg.streams.resize(sg.threads);
    sg.bufs.assign(2 * sg.threads, nullptr);
    sg.buf_ev.resize(2 * sg.threads);
    for (auto& st : sg.streams)
      if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return HOOD_ERR_CUDA;
    for (auto& e : sg.buf_ev)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return HOOD_ERR_CUDA;
  }
  while ((long long)sg.chunk_ev.size() < nchunks) {
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return HOOD_ERR_CUDA;
    sg.chunk_ev.push_back(e);
  }
  return HOOD_OK;
}

void destroy_stager(Stager* sg) {
  if (!sg) return;
  for (void* b : sg->bufs)
    if (b) cudaFreeHost(b);
  for (auto e : sg->buf_ev) cudaEventDestroy(e);
  for (auto e : sg->chunk_ev) cudaEventDestroy(e);
  for (auto st : sg->streams) cudaStreamDestroy(st);
  delete sg;
}

// Staged upload of `bytes` from pageable `src` to `dst`.  `ready(k)` is called
// on the calling thread (in order, k = 1 .. nchunks) once chunks [0, k) have
// their DMA enqueued; it may make the build stream wait on their events.
template <class F>
int staged_upload(hood_ctx* ctx, const void* src, void* dst, size_t bytes, F&& ready) {
  int rc;
  if ((rc = ensure_stager(ctx, 0))) return rc;
  const size_t CH = ctx->stager->chunk;
  const long long nch = (long long)((bytes + CH - 1) / CH);
  if ((rc = ensure_stager(ctx, nch))) return rc;
  Stager& sg = *ctx->stager;
  const int T = (int)std::min<long long>(sg.threads, nch);
  std::atomic<long long> next{0};
  std::atomic<int> failed{0};
  std::mutex mu;
  std::condition_variable cv;
  std::vector<char> done((size_t)nch, 0);
  auto worker = [&](int t) {
    cudaSetDevice(ctx->device);
    int use = 0;
    for (;;) {
      const long long j = next.fetch_add(1);
      if (j >= nch || failed.load()) break;
      const int b = 2 * t + (use++ & 1);
      if (!sg.bufs[b] && cudaHostAlloc(&sg.bufs[b], CH, cudaHostAllocDefault) != cudaSuccess) {
        sg.bufs[b] = nullptr;
        failed = 1;
      }
      const size_t off = (size_t)j * CH, len = std::min(CH, bytes - off);
      if (!failed.load()) {
        cudaEventSynchronize(sg.buf_ev[b]);  // the buffer's previous DMA has read it
        std::memcpy(sg.bufs[b], static_cast<const char*>(src) + off, len);
        if (cudaMemcpyAsync(static_cast<char*>(dst) + off, sg.bufs[b], len, cudaMemcpyHostToDevice, sg.streams[t]) !=
                cudaSuccess ||
            cudaEventRecord(sg.buf_ev[b], sg.streams[t]) != cudaSuccess ||
            cudaEventRecord(sg.chunk_ev[j], sg.streams[t]) != cudaSuccess)
          failed = 1;
      }
      {
        std::lock_guard<std::mutex> lk(mu);
        done[(size_t)j] = 1;
      }
      cv.notify_all();
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t) pool.emplace_back(worker, t);
  long long prefix = 0;
  while (prefix < nch) {
    {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] { return done[(size_t)prefix] != 0 || failed.load(); });
      while (prefix < nch && done[(size_t)prefix]) ++prefix;
    }
    if (failed.load()) break;
    ready(prefix);
  }
  for (auto& th : pool) th.join();
  if (failed.load()) {
    // wake-up order: drain whatever was enqueued before reporting
    for (auto st : sg.streams) cudaStreamSynchronize(st);
    return HOOD_ERR_CUDA;
  }
  return HOOD_OK;
}

// Reference-facing host call: H2D in chunks, each chunk's units launched as
// soon as its bytes land, then finalize and D2H of the compact corners only.
// Pinned input is copied by one DMA per unit range on the copy stream;
// pageable input goes through staged_upload.
template <class S>
int build_host(hood_ctx* ctx, const S* h_pts, long long n, long long block_len, S* h_corners, int* h_counts,
               uint32_t flags) {
  using V = typename PointT<S>::V;
  if (!ctx || !h_pts || !h_corners || !h_counts) return HOOD_ERR_INVALID_ARG;
  cudaSetDevice(ctx->device);
  Plan pl;
  int rc = make_plan<S>(ctx, n, block_len, pl);
  if (rc) return rc;
  if ((rc = ensure_ws(ctx, pl.units))) return rc;
  if ((rc = ensure_host_bufs<S>(ctx, n, pl.instances))) return rc;
  S* d_in = reinterpret_cast<S*>(ctx->d_in);
  S* d_out = reinterpret_cast<S*>(ctx->d_out);
  CUtensorMap map;
  long long full_rows = 0;
  std::memset(&map, 0, sizeof(map));
  if (!pl.hmode && (rc = encode_map<S>(d_in, n, pl.rows, &map, &full_rows))) return rc;
  cudaStream_t sc = ctx->s_copy, sk = ctx->s_comp;
  order_after_last(ctx, sk);
  cudaMemsetAsync(ctx->err, 0xff, sizeof(DevError), sk);
  SlabParams<S> p = slab_params<S>(ctx, pl, d_in, d_out, ctx->d_counts, full_rows, flags);
  const bool full_ok = pl.hmode && pl.spi > 1 && pl.instances == 1;
  p.full_units = full_ok ? ctx->arrive + 1 : nullptr;
  const int chunks = (pl.hmode && pl.instances == 1 && pl.units >= hood_ctx::kChunks) ? hood_ctx::kChunks : 1;
  auto range_of = [&](int c, long long& u0, long long& u1, long long& p0, long long& p1) {
    u0 = pl.units * c / chunks;
    u1 = pl.units * (c + 1) / chunks;
    if (chunks == 1) {
      p0 = 0;
      p1 = n;
    } else {
      p0 = (u0 * pl.tpi / pl.spi) * pl.T;
      p1 = (u1 == pl.units) ? n : std::min(n, (u1 * pl.tpi / pl.spi) * pl.T);
    }
  };
  auto launch_range = [&](int c) {
    long long u0, u1, p0, p1;
    range_of(c, u0, u1, p0, p1);
    p.unit_lo = u0;
    p.unit_hi = u1;
    p.read_lim = p1;
    const long long units_c = u1 - u0;
    const long long per_cta = pl.hmode ? slab_warps_per_cta<S>() : 1;
    launch_slab_kernel<S>(p, &map, (int)std::min<long long>((units_c + per_cta - 1) / per_cta, pl.grid), sk);
  };
  const size_t bytes = (size_t)n * sizeof(V);
  // small pageable inputs (at most two staging chunks) go through the
  // driver's own staging: spawning the copy threads would cost more
  const bool small = bytes <= 2 * (ctx->stager ? ctx->stager->chunk : (size_t)(8u << 20));
  if (small || is_pinned(h_pts)) {
    for (int c = 0; c < chunks; ++c) {
      long long u0, u1, p0, p1;
      range_of(c, u0, u1, p0, p1);
      cudaMemcpyAsync(d_in + 2 * p0, h_pts + 2 * p0, (size_t)(p1 - p0) * sizeof(V), cudaMemcpyHostToDevice, sc);
      cudaEventRecord(ctx->ev[c], sc);
      cudaStreamWaitEvent(sk, ctx->ev[c], 0);
      launch_range(c);
    }
  } else {
    int next_c = 0;
    long long waited = 0;
    rc = staged_upload(ctx, h_pts, d_in, bytes, [&](long long prefix) {
      const size_t landed = std::min(bytes, (size_t)prefix * ctx->stager->chunk);
      // every unit range whose points [.., p1) have been staged
      while (next_c < chunks) {
        long long u0, u1, p0, p1;
        range_of(next_c, u0, u1, p0, p1);
        if ((size_t)p1 * sizeof(V) > landed) break;
        for (; waited < prefix; ++waited) cudaStreamWaitEvent(sk, ctx->stager->chunk_ev[waited], 0);
        launch_range(next_c++);
      }
    });
    if (rc) return rc;
  }
  if (pl.hmode && pl.spi > 1) {
    FinalizeParams<S> f = finalize_params<S>(ctx, pl, d_out, ctx->d_counts);
    f.full_units = full_ok ? ctx->arrive + 1 : nullptr;
    launch_finalize<S>(f, (int)pl.instances, sk);
  }
  cudaMemcpyAsync(h_counts, ctx->d_counts, pl.instances * sizeof(int), cudaMemcpyDeviceToHost, sk);
  if (cudaStreamSynchronize(sk) != cudaSuccess) return HOOD_ERR_CUDA;
  ctx->last_stream = sk;
  ctx->have_last = true;
  ctx->last_launches = chunks + ((pl.hmode && pl.spi > 1) ? 1 : 0);
  hood_error err;
  if ((rc = decode_error(ctx, &err))) return rc;
  if (pl.instances == 1) {
    cudaMemcpy(h_corners, d_out, (size_t)h_counts[0] * sizeof(V), cudaMemcpyDeviceToHost);
  } else {
    // every instance's corners in one strided copy: rows of L slots, the
    // widest instance's count of columns
    int widest = 0;
    for (long long i = 0; i < pl.instances; ++i) widest = std::max(widest, h_counts[i]);
    if (widest > 0) {
      const size_t pitch = (size_t)pl.L * sizeof(V);
      cudaMemcpy2DAsync(h_corners, pitch, d_out, pitch, (size_t)widest * sizeof(V), (size_t)pl.instances,
                        cudaMemcpyDeviceToHost, sk);
    }
    cudaStreamSynchronize(sk);
  }
  return cudaGetLastError() == cudaSuccess ? HOOD_OK : HOOD_ERR_CUDA;
}

template <class S>
int merge_segments(hood_ctx* ctx, const S* seg_pts, const int* counts, long long G, long long stride,
                   S* corners, int* count, cudaStream_t st) {
  using V = typename PointT<S>::V;
  if (!ctx || !seg_pts || !counts || !corners || !count) return HOOD_ERR_INVALID_ARG;
  if (G < 1 || G > kMaxSlabsPerInstance || stride < 1) return HOOD_ERR_INVALID_ARG;
  cudaSetDevice(ctx->device);
  int rc;
  if ((rc = ensure_ws(ctx, G))) return rc;
  order_after_last(ctx, st);
  if (seg_pts != corners &&
      cudaMemcpyAsync(corners, seg_pts, (size_t)G * stride * sizeof(V), cudaMemcpyDeviceToDevice, st) !=
          cudaSuccess)
    return HOOD_ERR_CUDA;
  cudaMemcpyAsync(ctx->seg_cnt, counts, G * sizeof(int), cudaMemcpyDeviceToDevice, st);
  cudaMemsetAsync(ctx->err, 0xff, sizeof(DevError), st);
  FinalizeParams<S> f{};
  f.out = corners;
  f.out_counts = count;
  f.seg_cnt = ctx->seg_cnt;
  f.seg_apt = nullptr;
  f.seg_base = nullptr;
  f.seg_stride = stride;
  f.slabs_per_inst = (int)G;
  f.L = G * stride;
  f.fcap = (int)(32768 / sizeof(V));  // 64 KB of survivor stack, as double2
  launch_finalize<S>(f, 1, st);
  ctx->last_stream = st;
  ctx->have_last = true;
  ctx->last_launches = 1;
  return cudaGetLastError() == cudaSuccess ? HOOD_OK : HOOD_ERR_CUDA;
}

// One round of the reference loop on the GPU: REMOTE-padded blocks of d in,
// blocks of 2d out (driver.cpp:20-43 with launch(match_and_merge_kernel),
// kernel.cpp:155-161): the corner count of every block (the non-REMOTE
// prefix, hoodbuf.cpp:87-92), the common tangent of every pair (optionally
// left in scratch as the pinpoint phase does), the splice with REMOTE padding.
// d_in == d_out merges through a copy of the input in the context workspace.
template <class S>
int merge_round(hood_ctx* ctx, const S* in, long long n, long long d, S* out, int* scratch, cudaStream_t st) {
  using V = typename PointT<S>::V;
  if (!ctx || !in || !out) return HOOD_ERR_INVALID_ARG;
  if (d < 1 || (d & (d - 1)) != 0 || n < 2 * d || n % (2 * d) != 0) return HOOD_ERR_INVALID_ARG;
  cudaSetDevice(ctx->device);
  int rc;
  if ((rc = ensure_ws(ctx, n / d))) return rc;
  order_after_last(ctx, st);
  const size_t bytes = (size_t)n * sizeof(V);
  if (in == out) {
    if (bytes > ctx->round_tmp_bytes) {
      cudaFree(ctx->round_tmp);
      ctx->round_tmp = nullptr;
      if (cudaMalloc(&ctx->round_tmp, bytes) != cudaSuccess) return HOOD_ERR_CUDA;
      ctx->round_tmp_bytes = bytes;
    }
    if (cudaMemcpyAsync(ctx->round_tmp, in, bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess) return HOOD_ERR_CUDA;
    in = reinterpret_cast<const S*>(ctx->round_tmp);
  }
  if (cudaMemsetAsync(ctx->err, 0xff, sizeof(DevError), st) != cudaSuccess) return HOOD_ERR_CUDA;
  // workspace: block counts (n/d ints) and per-pair (pindex, qindex) (n/(2d) int2)
  int* pq = reinterpret_cast<int*>(ctx->seg_base);
  launch_block_count<S>(in, n, d, ctx->seg_cnt, st);
  launch_round_merge<S>(in, n, d, ctx->seg_cnt, pq, scratch, out, ctx->err, st);
  ctx->last_stream = st;
  ctx->have_last = true;
  ctx->last_launches = 3;
  return cudaGetLastError() == cudaSuccess ? HOOD_OK : HOOD_ERR_CUDA;
}

// Multi-GPU exchange: pack this rank's slab hood into a
// record; merge the G gathered records into the global hood.
template <class S>
int pack_record(hood_ctx* ctx, const S* corners, const int* count, long long cap, double x_offset, double* rec,
                cudaStream_t st) {
  if (!ctx || !corners || !count || !rec || cap < 1) return HOOD_ERR_INVALID_ARG;
  cudaSetDevice(ctx->device);
  int rc;
  if ((rc = ensure_ws(ctx, 1))) return rc;
  order_after_last(ctx, st);
  launch_pack_record<S>(corners, count, cap, x_offset, rec, ctx->err, st);
  ctx->last_stream = st;
  ctx->have_last = true;
  ctx->last_launches = 1;
  return cudaGetLastError() == cudaSuccess ? HOOD_OK : HOOD_ERR_CUDA;
}

int merge_records(hood_ctx* ctx, const double* recs, long long G, long long cap, double* out, int* count,
                  cudaStream_t st) {
  if (!ctx || !recs || !out || !count || cap < 1) return HOOD_ERR_INVALID_ARG;
  if (G < 1 || G > kMaxSlabsPerInstance) return HOOD_ERR_INVALID_ARG;
  cudaSetDevice(ctx->device);
  int rc;
  if ((rc = ensure_ws(ctx, G))) return rc;
  order_after_last(ctx, st);
  launch_gather_records(recs, G, cap, out, ctx->seg_cnt, count, ctx->done, ctx->err, st);
  FinalizeParams<double> f{};
  f.out = out;
  f.out_counts = count;
  f.seg_cnt = ctx->seg_cnt;
  f.seg_apt = nullptr;
  f.seg_base = nullptr;
  f.seg_stride = cap;
  f.slabs_per_inst = (int)G;
  f.L = G * cap;
  f.fcap = (int)(32768 / sizeof(double2));
  f.done = ctx->done;
  launch_finalize<double>(f, 1, st, /*pdl=*/true);  // returns at once when the gather kernel merged
  ctx->last_stream = st;
  ctx->have_last = true;
  ctx->last_launches = 2;
  return cudaGetLastError() == cudaSuccess ? HOOD_OK : HOOD_ERR_CUDA;
}

// Single-process multi-GPU build (SURVEY.md 8(b) hood_build_multi, the P2P
// variant of 8(e)): every context builds its slab's hood on its own device,
// the slab hood sizes are read back, the records (sized to the largest slab
// hood when one exceeds cap -- the count-sized exchange distributed.py does
// for the NCCL path; nothing is ever truncated) are packed and copied
// peer-to-peer (NVLink) to the first context's device, which merges them.
// Synchronous.  HOOD_ERR_CAPACITY (hood_last_error(ctxs[0]).index = the
// needed slots) only when the merged hood itself exceeds G*cap.
template <class S>
int build_multi(hood_ctx* const* ctxs, int G, const S* const* slabs, const int64_t* n_per, const double* x_off,
                double* d_out, int* d_count, long long cap) {
  if (!ctxs || G < 1 || !slabs || !n_per || !d_out || !d_count || cap < 1) return HOOD_ERR_INVALID_ARG;
  if (G > kMaxSlabsPerInstance) return HOOD_ERR_INVALID_ARG;
  hood_ctx* c0 = ctxs[0];
  int rc;
  // 1. every slab: build on its own device and stream
  for (int g = 0; g < G; ++g) {
    hood_ctx* c = ctxs[g];
    if (!c || !slabs[g] || n_per[g] < 1) return HOOD_ERR_INVALID_ARG;
    cudaSetDevice(c->device);
    if ((rc = ensure_host_bufs<S>(c, n_per[g], 1))) return rc;
    S* corners = reinterpret_cast<S*>(c->d_out);
    if ((rc = build_device<S>(c, slabs[g], n_per[g], 0, corners, c->d_counts, nullptr, 0, c->s_comp))) return rc;
  }
  // 2. the slab hood sizes (and every slab's validation errors)
  long long rcap = cap;
  for (int g = 0; g < G; ++g) {
    hood_error e;
    if ((rc = decode_error(ctxs[g], &e))) return rc;
    int k = 0;
    cudaSetDevice(ctxs[g]->device);
    if (cudaMemcpy(&k, ctxs[g]->d_counts, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return HOOD_ERR_CUDA;
    rcap = std::max(rcap, (long long)k);
  }
  // 3. records of rcap corners, peer-to-peer to the first device
  for (int g = 0; g < G; ++g) {
    hood_ctx* c = ctxs[g];
    cudaSetDevice(c->device);
    if (c->rec_cap < rcap) {
      cudaFree(c->rec);
      c->rec = nullptr;
      if (cudaMalloc(&c->rec, (size_t)(rcap + 1) * 2 * sizeof(double)) != cudaSuccess) return HOOD_ERR_CUDA;
      c->rec_cap = rcap;
    }
    launch_pack_record<S>(c->d_out, c->d_counts, rcap, x_off ? x_off[g] : 0.0, c->rec, c->err, c->s_comp);
  }
  cudaSetDevice(c0->device);
  // G records, then (when rcap > cap) G*rcap double2 of merge output
  const long long need = (long long)G * (rcap + 1) * 2 + (rcap > cap ? (long long)G * rcap * 2 : 0);
  if (c0->gathered_elems < need) {
    cudaFree(c0->gathered);
    c0->gathered = nullptr;
    if (cudaMalloc(&c0->gathered, (size_t)need * sizeof(double)) != cudaSuccess) return HOOD_ERR_CUDA;
    c0->gathered_elems = need;
  }
  for (int g = 0; g < G; ++g) {
    hood_ctx* c = ctxs[g];
    cudaSetDevice(c->device);
    cudaEventRecord(c->ev[0], c->s_comp);
    cudaSetDevice(c0->device);
    cudaStreamWaitEvent(c0->s_comp, c->ev[0], 0);
    cudaMemcpyPeerAsync(c0->gathered + (size_t)g * (rcap + 1) * 2, c0->device, c->rec, c->device,
                        (size_t)(rcap + 1) * 2 * sizeof(double), c0->s_comp);
  }
  // 4. merge on the first device; into the caller's buffer when the records
  // fit its G*cap slots, else into a scratch buffer checked below
  double* out = rcap > cap ? c0->gathered + (size_t)G * (rcap + 1) * 2 : d_out;
  if ((rc = merge_records(c0, c0->gathered, G, rcap, out, d_count, c0->s_comp))) return rc;
  if (cudaStreamSynchronize(c0->s_comp) != cudaSuccess) return HOOD_ERR_CUDA;
  if (out != d_out) {
    int h = 0;
    if (cudaMemcpy(&h, d_count, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return HOOD_ERR_CUDA;
    if (h > (long long)G * cap) {
      DevError de{~0ULL, (long long)h, ~0ULL};
      cudaMemcpy(c0->err, &de, sizeof(de), cudaMemcpyHostToDevice);
      c0->have_last = true;
      return HOOD_ERR_CAPACITY;
    }
    if (cudaMemcpy(d_out, out, (size_t)h * 2 * sizeof(double), cudaMemcpyDeviceToDevice) != cudaSuccess)
      return HOOD_ERR_CUDA;
  }
  hood_error e;
  return decode_error(c0, &e);
}

}  // namespace

extern "C" {

int hood_build_multi_f32(hood_ctx* const* ctxs, int G, const float* const* d_slabs, const int64_t* n_per,
                         const double* x_offsets, double* d_out, int32_t* d_count, int64_t cap) {
  return build_multi<float>(ctxs, G, d_slabs, n_per, x_offsets, d_out, d_count, cap);
}
int hood_build_multi_f64(hood_ctx* const* ctxs, int G, const double* const* d_slabs, const int64_t* n_per,
                         const double* x_offsets, double* d_out, int32_t* d_count, int64_t cap) {
  return build_multi<double>(ctxs, G, d_slabs, n_per, x_offsets, d_out, d_count, cap);
}

int hood_pack_record_f32(hood_ctx* ctx, const float* d_corners, const int32_t* d_count, int64_t cap,
                         double x_offset, double* d_rec, void* stream) {
  return pack_record<float>(ctx, d_corners, d_count, cap, x_offset, d_rec, reinterpret_cast<cudaStream_t>(stream));
}
int hood_pack_record_f64(hood_ctx* ctx, const double* d_corners, const int32_t* d_count, int64_t cap,
                         double x_offset, double* d_rec, void* stream) {
  return pack_record<double>(ctx, d_corners, d_count, cap, x_offset, d_rec, reinterpret_cast<cudaStream_t>(stream));
}
int hood_merge_records(hood_ctx* ctx, const double* d_recs, int64_t G, int64_t cap, double* d_out, int32_t* d_count,
                       void* stream) {
  return merge_records(ctx, d_recs, G, cap, d_out, d_count, reinterpret_cast<cudaStream_t>(stream));
}

int hood_merge_round_f32(hood_ctx* ctx, const float* d_in, int64_t n, int64_t d, float* d_out, void* stream) {
  return merge_round<float>(ctx, d_in, n, d, d_out, nullptr, reinterpret_cast<cudaStream_t>(stream));
}
int hood_merge_round_f64(hood_ctx* ctx, const double* d_in, int64_t n, int64_t d, double* d_out, void* stream) {
  return merge_round<double>(ctx, d_in, n, d, d_out, nullptr, reinterpret_cast<cudaStream_t>(stream));
}
int hood_merge_round_scratch_f32(hood_ctx* ctx, const float* d_in, int64_t n, int64_t d, float* d_out,
                                 int32_t* d_scratch, void* stream) {
  return merge_round<float>(ctx, d_in, n, d, d_out, d_scratch, reinterpret_cast<cudaStream_t>(stream));
}
int hood_merge_round_scratch_f64(hood_ctx* ctx, const double* d_in, int64_t n, int64_t d, double* d_out,
                                 int32_t* d_scratch, void* stream) {
  return merge_round<double>(ctx, d_in, n, d, d_out, d_scratch, reinterpret_cast<cudaStream_t>(stream));
}

// One reference round from host buffers (the observer mode of the drop-in
// build_hood): H2D, hood_merge_round, D2H,
// synchronous; a degenerate tangent comes back as HOOD_ERR_DEGENERATE with
// hood_last_error().index = the block.
int merge_round_host(hood_ctx* ctx, const double* h_in, long long n, long long d, double* h_out) {
  if (!ctx || !h_in || !h_out) return HOOD_ERR_INVALID_ARG;
  if (d < 1 || (d & (d - 1)) != 0 || n < 2 * d || n % (2 * d) != 0) return HOOD_ERR_INVALID_ARG;
  cudaSetDevice(ctx->device);
  int rc;
  if ((rc = ensure_host_bufs<double>(ctx, n, 1))) return rc;
  const size_t bytes = (size_t)n * 2 * sizeof(double);
  cudaStream_t sk = ctx->s_comp;
  order_after_last(ctx, sk);
  if (cudaMemcpyAsync(ctx->d_in, h_in, bytes, cudaMemcpyHostToDevice, sk) != cudaSuccess) return HOOD_ERR_CUDA;
  if ((rc = merge_round<double>(ctx, reinterpret_cast<const double*>(ctx->d_in), n, d,
                                reinterpret_cast<double*>(ctx->d_out), nullptr, sk)))
    return rc;
  if (cudaMemcpyAsync(h_out, ctx->d_out, bytes, cudaMemcpyDeviceToHost, sk) != cudaSuccess) return HOOD_ERR_CUDA;
  hood_error e;
  return decode_error(ctx, &e);
}

// The round trace of build_hood (cli.cpp:163-166 observer + write_trace_round,
// cli.cpp:108-118): the input is the HoodBuffer at d = 2 (init_hood,
// hoodbuf.cpp:88-92); each round is formatted, then merged on the GPU.
int hood_write_trace_f64(hood_ctx* ctx, const double* h_pts, int64_t n, const char* path) {
  if (!ctx || !h_pts || !path || n < 2 || (n & (n - 1)) != 0) return HOOD_ERR_INVALID_ARG;
  cudaSetDevice(ctx->device);
  FILE* f = std::fopen(path, "wb");
  if (!f) return HOOD_ERR_INVALID_ARG;
  const size_t bytes = (size_t)n * 2 * sizeof(double);
  double *d_a = nullptr, *d_b = nullptr;
  std::vector<double> h((size_t)n * 2);
  std::vector<char> text;
  int rc = HOOD_OK;
  if (cudaMalloc(&d_a, bytes) != cudaSuccess || cudaMalloc(&d_b, bytes) != cudaSuccess ||
      cudaMemcpy(d_a, h_pts, bytes, cudaMemcpyHostToDevice) != cudaSuccess)
    rc = HOOD_ERR_CUDA;
  std::memcpy(h.data(), h_pts, bytes);
  // driver.cpp:5-17: rounds while d = d1 * d2 < n, d doubling
  for (long long d = 2; rc == HOOD_OK && d < n; d *= 2) {
    const int64_t len = hood_format_trace_round(h.data(), n, d, nullptr, 0);
    text.resize((size_t)len);
    hood_format_trace_round(h.data(), n, d, text.data(), len);
    if (std::fwrite(text.data(), 1, text.size(), f) != text.size()) rc = HOOD_ERR_INVALID_ARG;
    if (rc == HOOD_OK) rc = merge_round<double>(ctx, d_a, n, d, d_b, nullptr, 0);
    if (rc == HOOD_OK && cudaMemcpy(h.data(), d_b, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) rc = HOOD_ERR_CUDA;
    std::swap(d_a, d_b);
  }
  if (rc == HOOD_OK && std::fputs("0\n", f) < 0) rc = HOOD_ERR_INVALID_ARG;  // write_trace_end
  if (std::fclose(f) != 0 && rc == HOOD_OK) rc = HOOD_ERR_INVALID_ARG;
  cudaFree(d_a);
  cudaFree(d_b);
  return rc;
}

int hood_merge_round_host_f64(hood_ctx* ctx, const double* h_in, int64_t n, int64_t d, double* h_out) {
  return merge_round_host(ctx, h_in, n, d, h_out);
}

int hood_create(hood_ctx** out, int device) {
  if (!out) return HOOD_ERR_INVALID_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return HOOD_ERR_CUDA;
  if (cudaSetDevice(device) != cudaSuccess) return HOOD_ERR_CUDA;
  hood_ctx* c = new hood_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  if (!encoder()) {
    delete c;
    return HOOD_ERR_CUDA;
  }
  *out = c;
  return HOOD_OK;
}

int hood_destroy(hood_ctx* c) {
  if (!c) return HOOD_OK;
  cudaSetDevice(c->device);
  cudaFree(c->seg_cnt);
  cudaFree(c->seg_apt);
  cudaFree(c->seg_base);
  cudaFree(c->steal_w);
  cudaFree(c->steal_done);
  cudaFree(c->part_cnt);
  cudaFree(c->part_base);
  cudaFree(c->err);
  cudaFree(c->done);
  cudaFree(c->arrive);
  cudaFree(c->warm);
  cudaFree(c->rec);
  cudaFree(c->gathered);
  cudaFree(c->d_in);
  cudaFree(c->d_out);
  cudaFree(c->d_counts);
  cudaFree(c->round_tmp);
  destroy_stager(c->stager);
  if (c->order_ev) cudaEventDestroy(c->order_ev);
  if (c->s_copy) {
    for (auto& e : c->ev) cudaEventDestroy(e);
    cudaStreamDestroy(c->s_copy);
    cudaStreamDestroy(c->s_comp);
  }
  delete c;
  return HOOD_OK;
}

int hood_reserve(hood_ctx* ctx, int64_t n, int64_t block_len, int f64) {
  if (!ctx) return HOOD_ERR_INVALID_ARG;
  cudaSetDevice(ctx->device);
  Plan pl;
  const int rc = f64 ? make_plan<double>(ctx, n, block_len, pl) : make_plan<float>(ctx, n, block_len, pl);
  if (rc) return rc;
  return ensure_ws(ctx, std::max(pl.units, (long long)kMaxSlabsPerInstance));
}

int hood_build_f32(hood_ctx* ctx, const float* d_pts, int64_t n, int64_t block_len, float* d_corners,
                   int32_t* d_counts, float* d_padded, uint32_t flags, void* stream) {
  return build_device<float>(ctx, d_pts, n, block_len, d_corners, d_counts, d_padded, flags,
                             reinterpret_cast<cudaStream_t>(stream));
}

int hood_build_f64(hood_ctx* ctx, const double* d_pts, int64_t n, int64_t block_len, double* d_corners,
                   int32_t* d_counts, double* d_padded, uint32_t flags, void* stream) {
  return build_device<double>(ctx, d_pts, n, block_len, d_corners, d_counts, d_padded, flags,
                              reinterpret_cast<cudaStream_t>(stream));
}

int hood_build_host_f32(hood_ctx* ctx, const float* h_pts, int64_t n, int64_t block_len, float* h_corners,
                        int32_t* h_counts, uint32_t flags) {
  return build_host<float>(ctx, h_pts, n, block_len, h_corners, h_counts, flags);
}

int hood_build_host_f64(hood_ctx* ctx, const double* h_pts, int64_t n, int64_t block_len,
                        double* h_corners, int32_t* h_counts, uint32_t flags) {
  return build_host<double>(ctx, h_pts, n, block_len, h_corners, h_counts, flags);
}

int hood_merge_segments_f32(hood_ctx* ctx, const float* d_seg_pts, const int32_t* d_counts, int64_t G,
                            int64_t seg_stride, float* d_corners, int32_t* d_count, void* stream) {
  return merge_segments<float>(ctx, d_seg_pts, d_counts, G, seg_stride, d_corners, d_count,
                               reinterpret_cast<cudaStream_t>(stream));
}

int hood_merge_segments_f64(hood_ctx* ctx, const double* d_seg_pts, const int32_t* d_counts, int64_t G,
                            int64_t seg_stride, double* d_corners, int32_t* d_count, void* stream) {
  return merge_segments<double>(ctx, d_seg_pts, d_counts, G, seg_stride, d_corners, d_count,
                                reinterpret_cast<cudaStream_t>(stream));
}

int hood_last_error(hood_ctx* ctx, hood_error* out) {
  if (!ctx) return HOOD_ERR_INVALID_ARG;
  return decode_error(ctx, out);
}

int hood_last_launch_count(hood_ctx* ctx) { return ctx ? ctx->last_launches : 0; }

// Internal profiling hooks (not part of the public header): kernel debug
// mode (4: every odd ring warp held back 300 us, so the others steal) and,
// for the -DHOOD_TRACE build only, a device buffer of 1024 + 16 * 8192 int64
// for the kernels' stamps (tools/trace_ring.py, tools/trace_finalize.py).
extern "C" int hood_internal_set_debug(hood_ctx* ctx, int mode, void* trace) {
  if (!ctx) return HOOD_ERR_INVALID_ARG;
  ctx->dbg = mode;
  ctx->trace = reinterpret_cast<long long*>(trace);
  return HOOD_OK;
}

// Tests / diagnosis: the number of tail steals since the last call (synchronizes).
extern "C" long long hood_internal_steals(hood_ctx* ctx) {
  if (!ctx || !ctx->arrive) return -1;
  cudaSetDevice(ctx->device);
  if (ctx->have_last) cudaStreamSynchronize(ctx->last_stream);
  unsigned v = 0;
  if (cudaMemcpy(&v, ctx->arrive + 2, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  cudaMemset(ctx->arrive + 2, 0, sizeof(unsigned));
  return v;
}

// Measurement only: one bare read of [p, p + bytes) (bench.py's attainable
// read time for the same bytes, same flush); async on `stream`.
extern "C" int hood_internal_stream_read(hood_ctx* ctx, const void* p, long long bytes, void* stream) {
  if (!ctx || !p || bytes < 16) return HOOD_ERR_INVALID_ARG;
  cudaSetDevice(ctx->device);
  if (ensure_ws(ctx, 1)) return HOOD_ERR_CUDA;
  launch_stream_read(p, bytes, reinterpret_cast<float*>(ctx->done), ctx->sms, reinterpret_cast<cudaStream_t>(stream));
  return cudaGetLastError() == cudaSuccess ? HOOD_OK : HOOD_ERR_CUDA;
}

int hood_set_profile_events(hood_ctx* ctx, void* before, void* after) {
  if (!ctx) return HOOD_ERR_INVALID_ARG;
  ctx->prof_before = reinterpret_cast<cudaEvent_t>(before);
  ctx->prof_after = reinterpret_cast<cudaEvent_t>(after);
  return HOOD_OK;
}

const char* hood_status_string(int s) {
  switch (s) {
    case HOOD_OK: return "ok";
    case HOOD_ERR_INVALID_ARG: return "invalid argument";
    case HOOD_ERR_X_NOT_INCREASING: return "x not strictly increasing";
    case HOOD_ERR_X_OUT_OF_RANGE: return "x outside (0, 1)";
    case HOOD_ERR_DEGENERATE: return "degenerate tangent";
    case HOOD_ERR_CUDA: return "CUDA error";
    case HOOD_ERR_CAPACITY: return "capacity exceeded";
    case HOOD_ERR_NOT_POWER_OF_TWO: return "point count is not a power of 2 (or is < 2)";
    case HOOD_ERR_PARSE: return "parse error";
    case HOOD_ERR_DEGENERATE_TRIPLE: return "points collinear within margin";
  }
  return "unknown";
}

int hood_abi_version(void) { return HOOD_B200_ABI_VERSION; }

}  // extern "C"
