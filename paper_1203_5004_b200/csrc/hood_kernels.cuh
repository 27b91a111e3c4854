// Kernel parameter blocks and host launch entry points (internal to the
// library; the public surface is the C-ABI in include/hood_b200.h).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace hood_b200 {

constexpr int kThreads = 256;       // one 128-byte chunk row per thread
constexpr int kStages = 3;          // TMA pipeline depth per CTA
constexpr int kTileBytes = kThreads * 128;
constexpr int kHCap = 1024;         // running slab hull kept in smem up to this many corners
#ifndef HOOD_MAX_SLABS
#define HOOD_MAX_SLABS 2048
#endif
constexpr int kMaxSlabsPerInstance = HOOD_MAX_SLABS;
#ifndef HOOD_MIN_UNIT_BLOCKS
#define HOOD_MIN_UNIT_BLOCKS 1
#endif
constexpr int kMinUnitBlocks = HOOD_MIN_UNIT_BLOCKS;  // ring kernel: blocks per unit at least

// First error of a build, encoded as key = index*2 + (x_not_increasing ? 1 : 0)
// so one atomicMin keeps validate_points' order (hoodbuf.cpp:48-58: at the
// same index the range check fires before the order check); consecutive-triple
// margin errors (hoodbuf.cpp:53-60, checked only after every x check) take
// key = kTripleKey + i, above every x key.  `need` (max, -1 = none) is the
// record capacity a multi-GPU exchange needed when a slab hood did not fit.
// Reset: all bytes 0xff.
struct DevError {
  unsigned long long key;
  long long need;
  unsigned long long degen;  // hood_merge_round: first block with a degenerate tangent (min, ~0 = none)
};
constexpr unsigned long long kTripleKey = 1ULL << 62;

// parts of a unit under tail stealing: the owner's and up to 3 stolen tails
#ifndef HOOD_STEAL_PARTS
#define HOOD_STEAL_PARTS 4
#endif
constexpr int kStealParts = HOOD_STEAL_PARTS;

template <class S>
struct SlabParams {
  const void* pts;          // n points, {x, y} interleaved, 16-byte aligned
  long long n;
  long long L;              // instance length (== n for a single instance)
  int log2L;                // instance mode: L == 1 << log2L
  int hmode;                // 1: slabs with a running hull; 0: whole instances per tile (L < T)
  int seg_chunks;           // chunks per culling segment: 256 (hmode) or L/K
  long long tiles_per_inst; // hmode: ceil(L / T)
  int slabs_per_inst;       // hmode
  long long num_units;      // hmode: slabs; else groups of tiles
  long long tiles_per_unit; // !hmode
  long long num_tiles;
  long long unit_lo, unit_hi;  // units processed by this launch
  long long full_rows;      // rows of the TMA tensor (n*sizeof(V)/128)
  void* out;                // corner slots (n), instance i at [i*L, i*L+count)
  int* out_counts;          // per instance
  int* seg_cnt;             // per slab (hmode)
  void* seg_apt;            // per slab: its highest hood corner (anchor point for finalize)
  long long* seg_base;
  DevError* err;
  int check_range;          // also flag x outside (0,1) (validate_points)
  int check_triples;        // also flag consecutive triples within the collinearity margin
  int dbg;                  // tests only: 4 = odd warps start 300 us late (forces steals)
  long long* trace;         // optional per-tile clock64 trace (profiling)
  long long read_lim;       // points at or past this index may not be read yet (host-path chunks)
  int lean;                 // ring kernel: the register-light variant (batched builds)
  unsigned* arrive;         // optional: +1 per finished unit (release), read by the finalize
  // optional (single instance): +1 per unit whose hood is ALL its points and
  // whose left seam continues the unit before it concavely (arc-like input);
  // when every unit counts, the finalize's answer is the input itself
  unsigned* full_units;
  // tail stealing (multi-unit instances, the STEAL kernel): per unit a claim
  // word (blocks the owner has claimed from the front, blocks stolen from the
  // end, steals so far), a parts-done counter, and per part (kStealParts u:
  // the owner's, kStealParts u + k: steal k's) its hood's corner count (-1:
  // no such part) and base slot
  unsigned long long* steal_w;  // [63:48] build epoch, [47:44] steals, [43:32] stolen blocks, [31:0] claimed blocks
  unsigned steal_epoch;         // this build's epoch (a word of another build is never stolen from)
  unsigned* steal_count;        // +1 per steal (tests / diagnosis)
  int* steal_done;
  int* part_cnt;
  long long* part_base;
};

template <class S>
struct FinalizeParams {
  void* out;
  int* out_counts;
  const int* seg_cnt;
  const void* seg_apt;      // per segment anchor point (its highest corner); nullptr: scan the corners
  const long long* seg_base; // nullptr: segment s starts at s * seg_stride
  long long seg_stride;
  int slabs_per_inst;
  long long L;
  int fcap;                 // smem corner capacity of the fast path
  long long* trace;         // optional phase clock64 stamps (profiling)
  const int* done;          // optional: nonzero = the result is already written (skip)
  // optional (single instance, PDL launch): start when *arrive reaches
  // arrive_target -- the ring kernel counts finished units -- instead of at the
  // ring grid's completion; the finalize zeroes it for the next build
  unsigned* arrive;
  unsigned arrive_target;
  unsigned* full_units;     // optional (single instance): see SlabParams; zeroed here for the next build
  // optional: a tiny resident dummy instance (kWarmBytes, written by the
  // error-reset kernel) the finalize merges first, while it waits for the
  // unit counter -- its code is then in the caches for the real merge
  void* warm;
  int dry;                  // internal: this is the dummy run (no waits)
};
constexpr int kWarmBytes = 256;

template <class S>
// reset_err (ring path only): reset the error record in a kernel the ring
// kernel follows programmatically, instead of a memset node
void launch_slab_kernel(const SlabParams<S>& p, const CUtensorMap* tmap, int grid, cudaStream_t st,
                        bool reset_err = false, void* warm = nullptr);
void launch_stream_read(const void* p, long long bytes, float* sink, int sms, cudaStream_t st);
template <class S>
void launch_finalize(const FinalizeParams<S>& p, int instances, cudaStream_t st, bool pdl = false);
template <class S>
void launch_pad_fill(void* padded, const void* corners, const int* counts, long long n, long long L,
                     cudaStream_t st);
template <class S>
void launch_block_count(const void* slots, long long n, long long d, int* counts, cudaStream_t st);
// One reference round on REMOTE-padded blocks (kernel.cpp:20-137): per pair
// of blocks the common tangent (pindex, qindex) by bridge() -- optionally left
// in scratch[start], scratch[start+1] as the pinpoint phase does -- with a
// degenerate tangent (another corner on the bridge line) reported in
// err->degen; then the splice into out (out != in).
template <class S>
void launch_round_merge(const void* in, long long n, long long d, const int* counts, int* pq, int* scratch,
                        void* out, DevError* err, cudaStream_t st);
// Multi-GPU exchange records: [count, 0 | corners (double, x + x_offset)], cap corners each.
// A slab hood of more than cap corners is reported in err->need (the record
// then holds its first cap corners and the true count in its header).
template <class S>
void launch_pack_record(const void* corners, const int* count, long long cap, double x_offset, double* rec,
                        DevError* err, cudaStream_t st);
// G records -> segments of stride cap in out (double2) + seg counts; hulls them directly
// (done = 1) when at most 64 corners arrived in total.
// A record whose header count exceeds cap is reported in err->need.
void launch_gather_records(const double* recs, long long G, long long cap, double* out, int* seg_cnt,
                           int* out_count, int* done, DevError* err, cudaStream_t st);
template <class S>
int slab_kernel_occupancy(bool lean = false);  // ring-kernel CTAs per SM
template <class S>
bool ring_lean_available();     // the register-light ring variant (batched builds) can run
template <class S>
int instance_kernel_occupancy();  // instance-kernel CTAs per SM
template <class S>
int slab_warps_per_cta();      // units (warps) per slab-kernel CTA
template <class S>
int slab_tile_rows(bool hmode, bool lean = false);  // chunk rows (= threads) per tile
size_t finalize_smem(int fcap_bytes, int slabs);

}  // namespace hood_b200
