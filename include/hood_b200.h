/*
 * hood_b200.h -- C-ABI of the B200-native upper-hood (upper convex hull)
 * build.  Drop-in replacement for the reference's hot path
 *
 *     hood::build_hood(const PointSet&, const BuildOptions&) -> BuildReport
 *         /root/reference/proj/include/hood/driver.hpp:43-45, src/driver.cpp:19-45
 *
 * and for its serial twin hood::oracle::upper_hull (oracle.hpp:23,
 * oracle.cpp:7-20), whose result the reference's build must reproduce
 * exactly (acceptance.cpp criterion 1).
 *
 * Plain pointers and sizes only.  Points are {x, y} pairs interleaved
 * (the reference's Point2 layout, geom.hpp:7-12), x strictly increasing
 * inside every instance.  Corners are returned left to right and are
 * bit-identical copies of input points.
 *
 * Every entry point returns a hood_status; device-side failures
 * (x not increasing, x out of range) are reported by hood_last_error(),
 * which synchronizes the stream of the last build.
 */
#ifndef HOOD_B200_H
#define HOOD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HOOD_B200_ABI_VERSION 1

typedef struct hood_ctx hood_ctx;

typedef enum hood_status {
  HOOD_OK = 0,
  HOOD_ERR_INVALID_ARG = 1,      /* bad size / alignment / block_len     */
  HOOD_ERR_X_NOT_INCREASING = 2, /* ValidationError::x_not_increasing    */
  HOOD_ERR_X_OUT_OF_RANGE = 3,   /* ValidationError::x_out_of_range      */
  HOOD_ERR_DEGENERATE = 4,       /* DegenerateTangent (hood_merge_round)  */
  HOOD_ERR_CUDA = 5,             /* a CUDA runtime call failed           */
  HOOD_ERR_CAPACITY = 6,         /* workspace / record capacity exceeded */
  HOOD_ERR_NOT_POWER_OF_TWO = 7, /* ValidationError::not_power_of_two    */
  HOOD_ERR_PARSE = 8,            /* cli.hpp ParseError (line in err_line) */
  HOOD_ERR_DEGENERATE_TRIPLE = 9 /* ValidationError::degenerate_triple   */
} hood_status;

/* hoodbuf.hpp:18-32 ValidationError / kernel.hpp:98-102 DegenerateTangent. */
typedef struct hood_error {
  int32_t code;       /* hood_status                                    */
  int32_t cuda_error; /* cudaError_t when code == HOOD_ERR_CUDA          */
  int64_t index;      /* first offending point index (validation)       */
} hood_error;

/* Build flags. */
#define HOOD_FLAG_CHECK_RANGE 0x1u   /* also reject x outside (0, 1) (validate_points) */
#define HOOD_FLAG_CHECK_TRIPLES 0x2u /* also reject consecutive triples (i, i+1, i+2) with
                                        |orient| < 1e-9 (validate_points' margin check,
                                        hoodbuf.cpp:53-60; HOOD_ERR_DEGENERATE_TRIPLE,
                                        index = i), after every x check as the reference
                                        orders them */

/* One context per device and host thread (the reference build is reentrant,
 * SPEC.md:423; contexts share nothing).  A context owns one device workspace
 * (unit summaries, error record, finished-unit counter): its builds must be
 * ordered on one stream (or synchronized); concurrent builds take one context
 * each. */
int hood_create(hood_ctx** ctx, int device);
int hood_destroy(hood_ctx* ctx);

/* Pre-size the device workspace so later builds of at most n points never
 * allocate (required before CUDA-graph capture). */
int hood_reserve(hood_ctx* ctx, int64_t n, int64_t block_len, int f64);

/* Device-pointer build, asynchronous on `stream` (a cudaStream_t, NULL = the
 * legacy default stream).
 *   d_pts      n points (2n scalars), 16-byte aligned.
 *   block_len  0 or n: one instance (any n >= 1).  Otherwise a power of two
 *              dividing n: n/block_len independent instances (the batched
 *              config; also the reference's per-round blocks of length d).
 *   d_corners  n slots; instance i's corners land at [i*block_len, ...).
 *   d_counts   one int32 per instance.
 *   d_padded   optional (NULL to skip): n slots in the reference HoodBuffer
 *              layout after the last round -- corners then REMOTE = (10, 0)
 *              (geom.hpp:14, hoodbuf.hpp:57-79).
 */
int hood_build_f32(hood_ctx* ctx, const float* d_pts, int64_t n, int64_t block_len, float* d_corners,
                   int32_t* d_counts, float* d_padded, uint32_t flags, void* stream);
int hood_build_f64(hood_ctx* ctx, const double* d_pts, int64_t n, int64_t block_len, double* d_corners,
                   int32_t* d_counts, double* d_padded, uint32_t flags, void* stream);

/* Host-pointer build (the reference-facing call: points in host memory,
 * compact corners back in host memory).  Synchronous.  h_corners needs n
 * slots; returns the per-instance counts in h_counts.  The input goes to the
 * device in chunks, each chunk's units launched as soon as its bytes land:
 * pinned (page-locked) input is copied by DMA directly; pageable input (a
 * std::vector) is staged by host threads through pinned bounce buffers
 * owned by the context, overlapped with the DMA. */
int hood_build_host_f32(hood_ctx* ctx, const float* h_pts, int64_t n, int64_t block_len, float* h_corners,
                        int32_t* h_counts, uint32_t flags);
int hood_build_host_f64(hood_ctx* ctx, const double* h_pts, int64_t n, int64_t block_len,
                        double* h_corners, int32_t* h_counts, uint32_t flags);

/* Final merge of G adjacent x-slab hoods (the multi-GPU exchange step):
 * segment g holds d_counts[g] corners at d_seg_pts + 2*g*seg_stride, slabs
 * left to right.  Writes the hood of the union to d_corners (capacity
 * G*seg_stride slots) and its size to d_count.  Asynchronous on `stream`. */
int hood_merge_segments_f32(hood_ctx* ctx, const float* d_seg_pts, const int32_t* d_counts, int64_t G,
                            int64_t seg_stride, float* d_corners, int32_t* d_count, void* stream);
int hood_merge_segments_f64(hood_ctx* ctx, const double* d_seg_pts, const int32_t* d_counts, int64_t G,
                            int64_t seg_stride, double* d_corners, int32_t* d_count, void* stream);

/* Multi-GPU exchange (the one collective of the x-slab sharding): each rank
 * packs its slab hood into a record of cap+1 double2 -- header (count, 0),
 * then the corners widened to double with x + x_offset -- the records are
 * all-gathered (NCCL), and every rank merges the G records (rank order = x
 * order) into the global hood: d_out (G*cap double2 slots) and d_count.
 * Asynchronous, graph-capturable.  A slab hood of more than cap corners is
 * never merged silently: the record keeps the true count in its header, and
 * hood_last_error() then reports HOOD_ERR_CAPACITY with index = the record
 * capacity needed (exchange again with records that large; the d_out/d_count
 * of that merge are not the global hood).  x + x_offset is exact for float2
 * slabs (float x widened to double plus a small integer offset); double2 slabs
 * should carry global x already (x_offset 0). */
int hood_pack_record_f32(hood_ctx* ctx, const float* d_corners, const int32_t* d_count, int64_t cap,
                         double x_offset, double* d_rec, void* stream);
int hood_pack_record_f64(hood_ctx* ctx, const double* d_corners, const int32_t* d_count, int64_t cap,
                         double x_offset, double* d_rec, void* stream);
int hood_merge_records(hood_ctx* ctx, const double* d_recs, int64_t G, int64_t cap, double* d_out,
                       int32_t* d_count, void* stream);

/* Single-process multi-GPU build (one context per device; the P2P form of
 * the exchange): context g builds the hood of slab g (d_slabs[g], n_per[g]
 * points on its own device, x in slab g's range, slabs left to right, x
 * shifted by x_offsets[g] when given), packs it, the records go peer-to-peer
 * to ctxs[0]'s device, which merges them into d_out (G*cap double2, on
 * ctxs[0]'s device) and d_count.  Synchronous.  Records are sized to the
 * largest slab hood when one exceeds cap (never truncated); HOOD_ERR_CAPACITY
 * (hood_last_error(ctxs[0]).index = slots needed) only when the global hood
 * itself has more than G*cap corners. */
int hood_build_multi_f32(hood_ctx* const* ctxs, int G, const float* const* d_slabs, const int64_t* n_per,
                         const double* x_offsets, double* d_out, int32_t* d_count, int64_t cap);
int hood_build_multi_f64(hood_ctx* const* ctxs, int G, const double* const* d_slabs, const int64_t* n_per,
                         const double* x_offsets, double* d_out, int32_t* d_count, int64_t cap);

/* One round of the reference round loop (driver.cpp:20-43, the per-round
 * operator launch(match_and_merge_kernel), kernel.cpp:155-161): d_in holds n
 * slots in HoodBuffer layout with blocks of d (each block: its hood's corners
 * left-packed, then REMOTE = (10, 0)); d_out receives the buffer with blocks of
 * 2d -- each the hood of two adjacent input blocks, REMOTE-padded.  d a power
 * of two, n a multiple of 2d; d_in == d_out allowed.  Asynchronous on
 * `stream`.  The per-round parity seam. */
int hood_merge_round_f32(hood_ctx* ctx, const float* d_in, int64_t n, int64_t d, float* d_out, void* stream);
int hood_merge_round_f64(hood_ctx* ctx, const double* d_in, int64_t n, int64_t d, double* d_out, void* stream);
/* The same round, also leaving the pinpoint phase's result in d_scratch
 * (n int32, kernel.cpp:101-112): for the pair window starting at slot
 * start = 2*b*d, d_scratch[start] = pindex and d_scratch[start+1] = qindex,
 * absolute slot indices of the common tangent's corners (the other entries
 * are not written).  A pair whose common tangent is not unique -- a corner
 * next to either end lies exactly on the bridge line, where the reference
 * throws DegenerateTangent(round, block) or reports the pinpoint's write-write
 * conflict (kernel.cpp:163-187, test_kernel.cpp:330-350) -- is reported by
 * hood_last_error() as HOOD_ERR_DEGENERATE with index = the first such block
 * (all four merge_round entry points check it). */
int hood_merge_round_scratch_f32(hood_ctx* ctx, const float* d_in, int64_t n, int64_t d, float* d_out,
                                 int32_t* d_scratch, void* stream);
int hood_merge_round_scratch_f64(hood_ctx* ctx, const double* d_in, int64_t n, int64_t d, double* d_out,
                                 int32_t* d_scratch, void* stream);

/* The same round from host buffers (n double2 slots in, n out), synchronous:
 * the drop-in build_hood's observer mode runs the reference round loop this
 * way.  Returns HOOD_ERR_DEGENERATE (index via
 * hood_last_error = the block) where the reference throws DegenerateTangent. */
int hood_merge_round_host_f64(hood_ctx* ctx, const double* h_in, int64_t n, int64_t d, double* h_out);

/* Synchronizes the stream of the last build and reports its first error:
 * validation (x range / order, then the consecutive-triple margin) before a
 * record capacity shortfall (HOOD_ERR_CAPACITY, index = capacity needed). */
int hood_last_error(hood_ctx* ctx, hood_error* out);

/* Number of kernels the last build enqueued (bench bookkeeping). */
int hood_last_launch_count(hood_ctx* ctx);

/* Optional: record two cudaEvent_t around the slab kernel of every later
 * device build on its stream (roofline timing of the dominant kernel).
 * Pass NULLs to stop. */
int hood_set_profile_events(hood_ctx* ctx, void* ev_before_slab, void* ev_after_slab);

/* Host front end (no GPU needed).  The reference's point files and input
 * checks, so files feed the build directly:
 *   hood_parse_points     cli.cpp:62-99 parse_points: the point count, then
 *                         x y pairs, '#' comments, count <= 2^26.  Writes
 *                         *count; HOOD_ERR_CAPACITY when cap < *count (retry
 *                         with a larger buffer); HOOD_ERR_PARSE with the line
 *                         in *err_line.  Does not validate (read_points =
 *                         parse + hood_validate_points, cli.cpp:56-60).
 *   hood_format_points    cli.cpp:101-106 write_point_set ("%.17g"); returns
 *                         the byte length, writes only when cap suffices.
 *   hood_validate_points  hoodbuf.cpp:30-70 validate_points: power of two,
 *                         x in (0, 1) strictly increasing, no triple within
 *                         the 1e-9 collinearity margin (all triples for n <= 64,
 *                         else consecutive + the reference's 10n sample);
 *                         ijk receives the offending indices. */
int hood_parse_points(const char* text, int64_t len, double* xy, int64_t cap, int64_t* count, int64_t* err_line);
int64_t hood_format_points(const double* xy, int64_t n, char* buf, int64_t cap);
int hood_validate_points(const double* xy, int64_t n, int64_t* ijk);

/* The reference's run output and round trace (cli.cpp:47-52, 108-118):
 *   hood_format_section      "<label> <n>" then one "%.17g %.17g" line per
 *                            point (write_section: label "points" / "hood").
 *   hood_format_trace_round  one round of the trace from a HoodBuffer layout
 *                            (hoodbuf.hpp:57-79): "d <d>", then per block of d
 *                            slots its corner count and corners (the slots
 *                            before the first REMOTE, x > 1).  The trace ends
 *                            with a "0" line (write_trace_end).
 * Both return the byte length and write only when cap suffices.
 *   hood_write_trace_f64     the whole trace of build_hood with an
 *                            on_round_begin observer (cli.cpp:163-166) into
 *                            the file at path: the GPU runs the reference's
 *                            round loop (hood_merge_round per round, from the
 *                            input as blocks of 2) and every round's buffer is
 *                            formatted on the host.  n a power of two >= 2. */
int64_t hood_format_section(const char* label, const double* xy, int64_t n, char* buf, int64_t cap);
int64_t hood_format_trace_round(const double* slots, int64_t n, int64_t d, char* buf, int64_t cap);
int hood_write_trace_f64(hood_ctx* ctx, const double* h_pts, int64_t n, const char* path);

const char* hood_status_string(int status);
int hood_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* HOOD_B200_H */
