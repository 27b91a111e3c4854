// B200 (sm_100a) kernels of the upper-hood build.
//
// The reference round loop (driver.cpp:19-45) launches log2(n)-1 merge rounds
// over REMOTE-padded blocks, each round touching all 36n bytes of hood /
// newhood / scratch (psim.cpp:40-47).  Here one HBM pass does the work:
//
//   slab_hull_kernel  (the hot kernel, HBM-bound: reads 8n / 16n bytes once)
//     persistent CTAs, each owning a contiguous slab of 32 KB tiles streamed
//     through a 3-stage TMA (cp.async.bulk.tensor, 128B swizzle) + mbarrier
//     ring.  Per tile: each of 256 threads owns one 128-byte chunk row
//     (16 float2 / 8 double2 points) and
//       1. finds its chunk's max y, checks x strictly increasing (fused
//          validate_points, hoodbuf.cpp:48-58);
//       2. block scans give every chunk an anchor height
//          tau = min(max y of all points to its left in the slab,
//                    max y of all points to its right up to the end of the
//                    NEXT tile).  A point with y < tau lies strictly below the
//          chord of two input points that straddle it, so it is not a corner
//          of the final hood and is dropped with ONE compare (the
//          reference's low stages do ~2 predicate calls per point per round);
//       3. runs the monotone chain (oracle.cpp:7-20) over the survivors of its
//          chunk, the stack living in its own swizzled smem row;
//       4. merges the 256 chunk hoods with a CTA merge tree (bridge = the
//          reference's g/f classifiers as monotone searches, splice =
//          kernel.cpp:117-137 without padding);
//       5. merges the tile hood into the slab's running hood (smem, spilling
//          to the output slots in HBM when it outgrows kHCap -- the arc).
//   finalize_kernel   one CTA per instance: cull slab hoods against the slab
//     maxima on both sides, then merge the survivors (smem fast path, or in
//     place in HBM for huge hoods) -- the paper's high stages on compacted
//     hoods only.
//   pad_fill_kernel   optional REMOTE-padded n-slot output (HoodBuffer layout,
//     hoodbuf.cpp:72-92) for drop-in callers that want the padded form.
#include "hood_device.cuh"
#include "hood_kernels.cuh"

#include <cstdio>

namespace hood_b200 {

template <class S> struct HCap { static constexpr int value = 8192 / (int)(2 * sizeof(S)); };

__device__ __forceinline__ unsigned char* align1024(unsigned char* p) {
  const unsigned a = smem_u32(p);
  return p + ((1024u - (a & 1023u)) & 1023u);
}

template <class S>
constexpr size_t slab_smem_bytes() {
  using V = typename PointT<S>::V;
  return 1024 + (size_t)kStages * kTileBytes + (size_t)HCap<S>::value * sizeof(V) +
         kThreads * sizeof(long long) + kThreads * sizeof(int) + 64 * sizeof(S) +
         kStages * sizeof(uint64_t) + 16 * sizeof(long long) + 64;
}

template <class S>
__device__ __forceinline__ void load_row(const unsigned char* row_base, int t, typename PointT<S>::V* v);

template <>
__device__ __forceinline__ void load_row<float>(const unsigned char* stage, int t, float2* v) {
  const unsigned char* row = stage + t * 128;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const float4 q = *reinterpret_cast<const float4*>(row + ((u ^ (t & 7)) << 4));
    v[2 * u] = make_float2(q.x, q.y);
    v[2 * u + 1] = make_float2(q.z, q.w);
  }
}

template <>
__device__ __forceinline__ void load_row<double>(const unsigned char* stage, int t, double2* v) {
  const unsigned char* row = stage + t * 128;
#pragma unroll
  for (int u = 0; u < 8; ++u) v[u] = *reinterpret_cast<const double2*>(row + ((u ^ (t & 7)) << 4));
}

template <class S>
__device__ __forceinline__ S row_ymax(const unsigned char* stage, int t) {
  using V = typename PointT<S>::V;
  V v[PointT<S>::K];
  load_row<S>(stage, t, v);
  S m = v[0].y;
#pragma unroll
  for (int i = 1; i < PointT<S>::K; ++i) m = fmax(m, v[i].y);
  return m;
}

// ------------------------------------------------------------------ slab kernel

template <class S>
__global__ void __launch_bounds__(kThreads, 2)
slab_hull_kernel(const __grid_constant__ CUtensorMap tmap, const SlabParams<S> p) {
  using V = typename PointT<S>::V;
  constexpr int K = PointT<S>::K;
  constexpr int T = kThreads * K;
  constexpr int HC = HCap<S>::value;

  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = align1024(smem_raw);
  unsigned char* stages = smem;
  V* Hs = reinterpret_cast<V*>(smem + (size_t)kStages * kTileBytes);
  long long* ns = reinterpret_cast<long long*>(Hs + HC);
  int* nc = reinterpret_cast<int*>(ns + kThreads);
  S* red = reinterpret_cast<S*>(nc + kThreads);  // [0,8) seg warp totals, [8,16) next totals
  uint64_t* bar = reinterpret_cast<uint64_t*>(red + 64);
  long long* shv = reinterpret_cast<long long*>(bar + kStages);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const V* gpts = reinterpret_cast<const V*>(p.pts);
  V* gout = reinterpret_cast<V*>(p.out);
  const S NEG = neg_inf<S>();

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
  }
  __syncthreads();

  auto unit_range = [&](long long u, long long& t0, long long& t1) {
    if (p.hmode) {
      const long long inst = u / p.slabs_per_inst, j = u % p.slabs_per_inst;
      t0 = inst * p.tiles_per_inst + (j * p.tiles_per_inst) / p.slabs_per_inst;
      t1 = inst * p.tiles_per_inst + ((j + 1) * p.tiles_per_inst) / p.slabs_per_inst;
    } else {
      t0 = u * p.tiles_per_unit;
      t1 = min(t0 + p.tiles_per_unit, p.num_tiles);
    }
  };

  // Producer cursor (thread 0 only) -- issues tiles in consumption order.
  long long pu = p.unit_lo + blockIdx.x, pt = 0, pt_end = 0;
  int k_issued = 0;
  if (pu < p.unit_hi) unit_range(pu, pt, pt_end);
  auto produce = [&]() {
    if (pu >= p.unit_hi) return;
    const int st = k_issued % kStages;
    if (p.full_rows > 0) {
      mbar_expect_tx(&bar[st], kTileBytes);
      tma_load_2d(stages + (size_t)st * kTileBytes, &tmap, 0, (int)(pt * kThreads), &bar[st]);
    } else {
      mbar_expect_tx(&bar[st], 0);
    }
    ++k_issued;
    if (++pt >= pt_end) {
      pu += gridDim.x;
      if (pu < p.unit_hi) unit_range(pu, pt, pt_end);
    }
  };
  if (tid == 0)
    for (int s = 0; s < kStages; ++s) produce();

  // Running slab hood state (block-uniform).
  long long hN = 0;
  int hsm = 1;
  S runmax = NEG;

  const int seg = p.seg_chunks;
  const int W = seg < 32 ? seg : 32;
  int levels = 0;
  while ((1 << levels) < seg) ++levels;

  int k = 0;
  for (long long u = p.unit_lo + blockIdx.x; u < p.unit_hi; u += gridDim.x) {
    long long t0, t1;
    unit_range(u, t0, t1);
    const long long slab_base = t0 * T;
    const long long inst_u = p.hmode ? u / p.slabs_per_inst : 0;
    const long long lim_h = p.hmode ? min(p.n, (inst_u + 1) * p.L) : p.n;

    for (long long g = t0; g < t1; ++g, ++k) {
      const int st = k % kStages;
      unsigned char* tile = stages + (size_t)st * kTileBytes;
      const TileAcc<S> X{tile};
      const bool has_next = p.hmode && (g + 1 < t1);
      mbar_wait(&bar[st], (unsigned)((k / kStages) & 1));

      // ---- 1. own chunk: load, max y, x order (+ range) check
      const long long base_pt = g * T + (long long)tid * K;
      const long long lim = p.hmode ? lim_h : p.n;
      const int nv = (int)max(0LL, min((long long)K, lim - base_pt));
      V v[K];
      if (nv == K) {
        load_row<S>(tile, tid, v);
      } else {
#pragma unroll
        for (int i = 0; i < K; ++i) v[i] = (i < nv) ? gpts[base_pt + i] : V{};
      }
      S cm = NEG;
#pragma unroll
      for (int i = 0; i < K; ++i)
        if (i < nv) cm = fmax(cm, v[i].y);
      if (nv > 0) {
        unsigned long long bad = ~0ULL;
        const bool inst_start = (base_pt % p.L) == 0;
        if (!inst_start) {
          const V prev = (tid > 0) ? X.ld((long long)tid * K - 1) : gpts[base_pt - 1];
          if (!(v[0].x > prev.x)) bad = (unsigned long long)base_pt * 2 + 1;
        }
#pragma unroll
        for (int i = K - 1; i >= 1; --i)
          if (i < nv && !(v[i].x > v[i - 1].x)) bad = min(bad, (unsigned long long)(base_pt + i) * 2 + 1);
        if (p.check_range) {
#pragma unroll
          for (int i = K - 1; i >= 0; --i)
            if (i < nv && !(v[i].x > (S)0 && v[i].x < (S)1))
              bad = min(bad, (unsigned long long)(base_pt + i) * 2);
        }
        if (bad != ~0ULL) atomicMin(&p.err->key, bad);
      }
      S nx = NEG;
      if (has_next) {
        const int st2 = (k + 1) % kStages;
        mbar_wait(&bar[st2], (unsigned)(((k + 1) / kStages) & 1));
        const long long nbase = (g + 1) * T + (long long)tid * K;
        if (nbase + K <= lim) nx = row_ymax<S>(stages + (size_t)st2 * kTileBytes, tid);
      }

      // ---- 2. anchor heights: segmented exclusive prefix / suffix max
      const int gl = lane & (W - 1);
      S pin = cm, sin = cm;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        if (o < W) {
          const S a = __shfl_up_sync(0xffffffffu, pin, o, W);
          const S b = __shfl_down_sync(0xffffffffu, sin, o, W);
          if (gl >= o) pin = fmax(pin, a);
          if (gl + o < W) sin = fmax(sin, b);
        }
      }
      S pex = __shfl_up_sync(0xffffffffu, pin, 1, W);
      S sex = __shfl_down_sync(0xffffffffu, sin, 1, W);
      if (gl == 0) pex = NEG;
      if (gl == W - 1) sex = NEG;
      S segmax = __shfl_sync(0xffffffffu, pin, (lane & ~(W - 1)) + W - 1);
      S nred = nx;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) nred = fmax(nred, __shfl_xor_sync(0xffffffffu, nred, o));
      if (lane == 31) red[warp] = pin;
      if (lane == 0) red[8 + warp] = nred;
      __syncthreads();
      S nextmax = NEG;
      if (p.hmode) {
#pragma unroll
        for (int w = 0; w < 8; ++w) nextmax = fmax(nextmax, red[8 + w]);
      }
      if (seg > 32) {
        const int nsw = seg >> 5;
        const int sw0 = (warp / nsw) * nsw;
        S wp = NEG, ws = NEG, wt = NEG;
        for (int w = sw0; w < sw0 + nsw; ++w) {
          const S r = red[w];
          if (w < warp) wp = fmax(wp, r);
          if (w > warp) ws = fmax(ws, r);
          wt = fmax(wt, r);
        }
        pex = fmax(pex, wp);
        sex = fmax(sex, ws);
        segmax = wt;
      }
      if (p.hmode) {
        pex = fmax(pex, runmax);
        sex = fmax(sex, nextmax);
      }
      const S tau = fmin(pex, sex);

      // ---- 3. monotone chain over the survivors (oracle.cpp:7-20)
      const long long rb = (long long)tid * K;
      int sp = 0;
      V s1 = V{}, s2 = V{};
#pragma unroll
      for (int i = 0; i < K; ++i) {
        if (i < nv && !(v[i].y < tau)) {
          const V q = v[i];
          while (sp >= 2 && !above(s2, s1, q)) {
            --sp;
            s1 = s2;
            if (sp >= 2) s2 = X.ld(rb + sp - 2);
          }
          X.st(rb + sp, q);
          ++sp;
          s2 = s1;
          s1 = q;
        }
      }
      ns[tid] = rb;
      nc[tid] = sp;
      __syncthreads();

      // ---- 4. CTA merge tree over the chunk hoods of each segment
      tree_merge<V>(X, ns, nc, kThreads, levels);

      if (p.hmode) {
        // ---- 5. merge the tile hood into the running slab hood
        if (tid == 0) {
          const long long qs = ns[0], kq = nc[0];
          long long pidx = -1, qidx = 0, newN = hN;
          if (kq > 0) {
            if (hN > 0) {
              if (hsm) bridge<V>(PtrAcc<V>{Hs}, 0, hN, X, qs, kq, pidx, qidx);
              else bridge<V>(PtrAcc<V>{gout + slab_base}, 0, hN, X, qs, kq, pidx, qidx);
            }
            newN = pidx + 1 + kq - qidx;
          } else {
            pidx = hN - 1;
            qidx = 0;
          }
          shv[0] = pidx;
          shv[1] = qidx;
          shv[2] = newN;
          shv[3] = qs;
          shv[4] = kq;
        }
        __syncthreads();
        const long long pidx = shv[0], qidx = shv[1], newN = shv[2], qs = shv[3], kq = shv[4];
        if (kq > 0) {
          if (hsm && newN > HC) {  // spill the kept prefix to the output slots
            for (long long e = tid; e <= pidx; e += kThreads) gout[slab_base + e] = Hs[e];
            hsm = 0;
          }
          V* dstp = hsm ? Hs : gout + slab_base;
          for (long long e = tid; e < kq - qidx; e += kThreads) dstp[pidx + 1 + e] = X.ld(qs + qidx + e);
          hN = newN;
        }
        runmax = fmax(runmax, segmax);
      } else {
        // instance mode: every segment root is a finished instance hood
        const int s0 = (tid / seg) * seg;
        const long long inst_pt = g * T + (long long)s0 * K;
        if (inst_pt < p.n) {
          const long long start = ns[s0];
          const int cnt = nc[s0];
          for (int e = tid - s0; e < cnt; e += seg) gout[inst_pt + e] = X.ld(start + e);
          if (tid == s0) p.out_counts[inst_pt / p.L] = cnt;
        }
      }
      __syncthreads();
      if (tid == 0) {
        fence_proxy_async();
        produce();
      }
    }

    if (p.hmode) {
      if (hsm)
        for (long long e = tid; e < hN; e += kThreads) gout[slab_base + e] = Hs[e];
      if (tid == 0) {
        if (p.slabs_per_inst == 1) {
          p.out_counts[inst_u] = (int)hN;
        } else {
          p.seg_cnt[u] = (int)hN;
          p.seg_ymax[u] = runmax;
          p.seg_base[u] = slab_base;
        }
      }
      hN = 0;
      hsm = 1;
      runmax = NEG;
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------------ finalize

template <class S>
__global__ void __launch_bounds__(256) finalize_kernel(const FinalizeParams<S> p) {
  using V = typename PointT<S>::V;
  extern __shared__ unsigned char smem_raw[];
  const int M = p.slabs_per_inst;
  const long long s0 = (long long)blockIdx.x * M;
  const long long ibase = (long long)blockIdx.x * p.L;
  V* gout = reinterpret_cast<V*>(p.out);
  const S NEG = neg_inf<S>();

  long long* base = reinterpret_cast<long long*>(smem_raw);
  long long* nsd = base + M;
  S* pre = reinterpret_cast<S*>(nsd + M);
  S* suf = pre + M;
  int* cnt = reinterpret_cast<int*>(suf + M);
  int* lo = cnt + M;
  int* ncd = lo + M;
  int* scal = ncd + M;  // [0] total alive
  V* F = reinterpret_cast<V*>(smem_raw + (((size_t)(reinterpret_cast<unsigned char*>(scal + 8) - smem_raw) + 15) & ~(size_t)15));

  const int tid = threadIdx.x;
  if (tid == 0) scal[0] = 0;
  for (int s = tid; s < M; s += blockDim.x) {
    base[s] = p.seg_base ? p.seg_base[s0 + s] : ibase + (long long)s * p.seg_stride;
    cnt[s] = p.seg_cnt[s0 + s];
    S y = NEG;
    if (p.seg_ymax) y = p.seg_ymax[s0 + s];
    else
      for (int e = 0; e < cnt[s]; ++e) y = fmax(y, gout[base[s] + e].y);
    pre[s] = y;
    suf[s] = y;
  }
  __syncthreads();
  // inclusive prefix / suffix max (Hillis-Steele; M <= kMaxSlabsPerInstance)
  for (int o = 1; o < M; o <<= 1) {
    S a[4], b[4];
    int c = 0;
    for (int s = tid; s < M; s += blockDim.x, ++c) {
      a[c] = (s >= o) ? fmax(pre[s], pre[s - o]) : pre[s];
      b[c] = (s + o < M) ? fmax(suf[s], suf[s + o]) : suf[s];
    }
    __syncthreads();
    c = 0;
    for (int s = tid; s < M; s += blockDim.x, ++c) {
      pre[s] = a[c];
      suf[s] = b[c];
    }
    __syncthreads();
  }
  // alive range of every slab hood: corners with y >= tau form one run
  // (y is unimodal along an upper hull).
  for (int s = tid; s < M; s += blockDim.x) {
    const S tau = fmin(s > 0 ? pre[s - 1] : NEG, s + 1 < M ? suf[s + 1] : NEG);
    const int c = cnt[s];
    const V* h = gout + base[s];
    int l = 0, r = c;  // alive [l, r)
    if (c > 0 && !(h[0].y >= tau && h[c - 1].y >= tau)) {
      // peak: first i with !(y[i+1] > y[i])
      int a = 0, b = c - 1;
      while (a < b) {
        const int mid = (a + b) >> 1;
        if (h[mid + 1].y > h[mid].y) a = mid + 1;
        else b = mid;
      }
      const int pk = a;
      if (!(h[pk].y >= tau)) {
        l = r = 0;
      } else {
        int x0 = 0, x1 = pk;  // first index in [0,pk] with y >= tau
        while (x0 < x1) {
          const int mid = (x0 + x1) >> 1;
          if (h[mid].y >= tau) x1 = mid;
          else x0 = mid + 1;
        }
        l = x0;
        int y0 = pk, y1 = c - 1;  // last index in [pk, c) with y >= tau
        while (y0 < y1) {
          const int mid = (y0 + y1 + 1) >> 1;
          if (h[mid].y >= tau) y0 = mid;
          else y1 = mid - 1;
        }
        r = y0 + 1;
      }
    }
    lo[s] = l;
    ncd[s] = r - l;
    atomicAdd(&scal[0], r - l);
  }
  __syncthreads();
  const int total = scal[0];
  int levels = 0;
  while ((1 << levels) < M) ++levels;
  if (total <= p.fcap) {
    // fast path: compact the survivors into smem (exclusive scan, thread 0;
    // M is at most a few thousand)
    if (tid == 0) {
      long long off = 0;
      for (int s = 0; s < M; ++s) {
        nsd[s] = off;
        off += ncd[s];
      }
    }
    __syncthreads();
    for (int s = tid; s < M; s += blockDim.x)
      for (int e = 0; e < ncd[s]; ++e) F[nsd[s] + e] = gout[base[s] + lo[s] + e];
    __syncthreads();
    tree_merge<V>(PtrAcc<V>{F}, nsd, ncd, M, levels);
    const long long st = nsd[0];
    const int hc = ncd[0];
    for (int e = tid; e < hc; e += blockDim.x) gout[ibase + e] = F[st + e];
    if (tid == 0) p.out_counts[blockIdx.x] = hc;
  } else {
    for (int s = tid; s < M; s += blockDim.x) nsd[s] = base[s] + lo[s];
    __syncthreads();
    tree_merge<V>(PtrAcc<V>{gout}, nsd, ncd, M, levels);
    if (tid == 0) {
      const long long st = nsd[0];
      const int hc = ncd[0];
      if (st != ibase)
        for (int e = 0; e < hc; ++e) gout[ibase + e] = gout[st + e];
      p.out_counts[blockIdx.x] = hc;
    }
  }
}

// ------------------------------------------------------------------ padding

template <class S>
__global__ void pad_fill_kernel(typename PointT<S>::V* padded, const typename PointT<S>::V* corners,
                                const int* counts, long long n, long long L) {
  using V = typename PointT<S>::V;
  const V remote{(S)10, (S)0};  // geom.hpp:14
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long inst = i / L, off = i - inst * L;
    padded[i] = (off < counts[inst]) ? corners[i] : remote;
  }
}

// ------------------------------------------------------------------ host side

template <class S>
size_t slab_kernel_smem() {
  return slab_smem_bytes<S>();
}

template <class S>
int slab_kernel_occupancy() {
  static int occ = -1;
  if (occ < 0) {
    cudaFuncSetAttribute(slab_hull_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)slab_smem_bytes<S>());
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, slab_hull_kernel<S>, kThreads, slab_smem_bytes<S>());
    occ = o > 0 ? o : 1;
  }
  return occ;
}

template <class S>
void launch_slab_kernel(const SlabParams<S>& p, const CUtensorMap* tmap, int grid, cudaStream_t st) {
  slab_kernel_occupancy<S>();
  slab_hull_kernel<S><<<grid, kThreads, slab_smem_bytes<S>(), st>>>(*tmap, p);
}

size_t finalize_smem(int fcap_bytes, int slabs) {
  return (size_t)slabs * (2 * sizeof(long long) + 2 * sizeof(double) + 3 * sizeof(int)) + 64 + 16 +
         (size_t)fcap_bytes;
}

template <class S>
void launch_finalize(const FinalizeParams<S>& p, int instances, cudaStream_t st) {
  using V = typename PointT<S>::V;
  const size_t bytes = finalize_smem(p.fcap * (int)sizeof(V), p.slabs_per_inst);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(finalize_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  finalize_kernel<S><<<instances, 256, bytes, st>>>(p);
}

template <class S>
void launch_pad_fill(void* padded, const void* corners, const int* counts, long long n, long long L,
                     cudaStream_t st) {
  using V = typename PointT<S>::V;
  const long long blocks = min((n + 255) / 256, 148LL * 16);
  pad_fill_kernel<S><<<(int)blocks, 256, 0, st>>>(reinterpret_cast<V*>(padded),
                                                   reinterpret_cast<const V*>(corners), counts, n, L);
}

template void launch_slab_kernel<float>(const SlabParams<float>&, const CUtensorMap*, int, cudaStream_t);
template void launch_slab_kernel<double>(const SlabParams<double>&, const CUtensorMap*, int, cudaStream_t);
template void launch_finalize<float>(const FinalizeParams<float>&, int, cudaStream_t);
template void launch_finalize<double>(const FinalizeParams<double>&, int, cudaStream_t);
template void launch_pad_fill<float>(void*, const void*, const int*, long long, long long, cudaStream_t);
template void launch_pad_fill<double>(void*, const void*, const int*, long long, long long, cudaStream_t);
template int slab_kernel_occupancy<float>();
template int slab_kernel_occupancy<double>();
template size_t slab_kernel_smem<float>();
template size_t slab_kernel_smem<double>();

}  // namespace hood_b200
