/*
 * dvl.h -- C ABI of the B200-native dynamic-volume-lines (DVL) library.
 *
 * What it computes (arXiv 2306.11612; "P:n" = line n of PAPER.md, readings O#/A# in
 * DESIGN.md section 3):
 *   BUILD   (once per dataset): centroid quantisation on the logical grid
 *           (P:76-82), 3D Hilbert code, radix sort of (code, cell id),
 *           permutation of levels and member scalars into curve order.
 *   UPDATE  (every transfer-function edit): per cell and member the
 *           TF alpha of the normalised scalar, local variation V_h (Eq. 1),
 *           AMR importance f = (max(V_h/maxV, eps) 2^L)^P (Eq. 3; minimum
 *           importance P:138-139) as u64 fixed point, prefix sum (Eq. 4),
 *           projection of the x pairs onto W pixel bins, per-bin/member
 *           count, min, max, mean of the normalised scalar and the TF applied to the mean
 *           (P:250-256).
 *
 * Conventions
 *   - Every function returns dvl_status; on failure the context is left unchanged and
 *     dvl_last_error() holds a one-line description.  A context is not thread-safe;
 *     distinct contexts are independent.
 *   - All device work is enqueued on the context's CUDA stream.  Input pointers are
 *     borrowed for the duration of the call only; output buffers are owned by the caller.
 *   - dvl_mem says whether a pointer argument is host memory (DVL_MEM_HOST) or device
 *     memory of the context's device (DVL_MEM_DEVICE).  Calls taking host outputs
 *     synchronise the context stream before returning.
 *   - No C++ types, exceptions or torch types cross this boundary.
 */
#ifndef DVL_H
#define DVL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dvl_ctx dvl_ctx;

typedef enum {
    DVL_OK = 0,
    DVL_E_INVAL = 1,      /* invalid argument (see each call) */
    DVL_E_STATE = 2,      /* call out of order (e.g. update before build) */
    DVL_E_RANGE = 3,      /* logical extent > 2^21, n >= 2^30, or ceil(Lmax*P) > 100 */
    DVL_E_OVERLAP = 4,    /* duplicate or overlapping AMR cells (found after the sort) */
    DVL_E_DEGENERATE = 5, /* sum of all fixed-point weights is 0 (only with eps = 0) */
    DVL_E_NOMEM = 6,      /* device or pinned host allocation failed */
    DVL_E_CUDA = 7,       /* a CUDA runtime error; text in dvl_last_error */
    DVL_E_NCCL = 8        /* a collective failed (or libnccl.so.2 is missing); text in dvl_last_error */
} dvl_status;

typedef enum { DVL_MEM_HOST = 0, DVL_MEM_DEVICE = 1 } dvl_mem;

/* max(V_h) used to normalise Eq. 3 (reading A8):
 *   CONSERVATIVE (default, "R2"): max over members m and TF entries a in [i, j] of
 *       A(m,a) minus the min over the same set, [i, j] from the members' data ranges;
 *   PER_ENTRY ("R1"): max over a in [i, j] of (max_m A(m,a) - min_m A(m,a)) -- the
 *       literal eq:va;
 *   EXACT: max over all cells of V_h (one extra pass over the cells). */
typedef enum {
    DVL_MAXV_CONSERVATIVE = 0,
    DVL_MAXV_PER_ENTRY = 1,
    DVL_MAXV_EXACT = 2
} dvl_maxv_mode;

/* Optional device allocator (e.g. PyTorch's caching allocator).  Both NULL: the
 * library uses cudaMallocAsync/cudaFreeAsync on the context stream. */
typedef void *(*dvl_alloc_fn)(size_t bytes, void *cuda_stream, void *user);
typedef void (*dvl_free_fn)(void *ptr, size_t bytes, void *cuda_stream, void *user);

#define DVL_FLAG_TIMING 1u   /* record CUDA events around every kernel (dvl_get_timings) */
#define DVL_FLAG_GENERIC 2u  /* use the portable one-tile-per-CTA update kernels instead of
                                the persistent TMA-pipelined ones (always used for M > 16) */
/* Test / diagnostic flags: they select among kernels that return identical bits. */
#define DVL_FLAG_NO_EDIT_CACHE 4u  /* every TF edit streams every member (no edit cache) */
#define DVL_FLAG_PASS2_INLINE 8u   /* pass 2 folds its boundary warp tiles itself ... */
#define DVL_FLAG_PASS2_LIST 16u    /* ... or lists them for the GPU-wide boundary kernel
                                      (default: chosen from W, the tiles and the SM count) */
#define DVL_FLAG_LSD_SORT 32u      /* build with the onesweep LSD radix sort even where the
                                      bucket sort applies (3b <= 36) */
#define DVL_FLAG_PASS2_JOBS 64u    /* pass 2 folds the single-pixel jobs several per warp and
                                      takes the others one warp each (default when the
                                      warp-tile statistics exceed 32 MB and there are >= 16
                                      pass-2 jobs per pixel) */

typedef struct {
    int device;             /* CUDA device ordinal */
    void *cuda_stream;      /* cudaStream_t to enqueue on; NULL: the context creates one */
    dvl_alloc_fn alloc;     /* optional, see above */
    dvl_free_fn free;
    void *user;             /* passed back to alloc/free */
    uint32_t flags;         /* DVL_FLAG_* */
} dvl_init;

/* One polyline vertex = one pixel bin of one member.
 * t_* are statistics of the member's normalised scalar t in [0,1] over the cells whose
 * x interval overlaps the bin (reading A15-A17); y is the TF alpha at t_mean (the
 * polyline height), r/g/b the TF colour at t_mean; count the
 * number of such cells (the paper's per-bin counter).  32 bytes. */
typedef struct {
    float t_min, t_max, t_mean, y, r, g, b;
    uint32_t count;
} dvl_vertex;

typedef struct {
    uint64_t n;             /* cells */
    uint32_t members;       /* M */
    uint32_t extent;        /* E: max over cells/axes of lower + 2^L */
    int32_t bits;           /* b = max(1, ceil(log2 E)), Hilbert bits per axis */
    int32_t Lmax;           /* coarsest level present */
    int32_t key_bytes;      /* 4 if 3b <= 32 else 8 */
    int32_t tf_size;        /* N, entries per transfer function */
    float P, eps;           /* exponent and minimum importance */
    int32_t maxv_mode;      /* dvl_maxv_mode */
    int32_t shift;          /* s of the u64 fixed point (reading O11); valid after an update */
    float maxV;             /* normaliser of the last update */
    uint64_t Qtot;          /* sum of all fixed-point weights of the last update */
    uint64_t device_bytes;  /* device memory held by the context */
    int32_t cells_per_tile; /* tile size of the update kernels */
    int32_t reserved;
} dvl_info_t;

/* Point location for brushing and linking: for each of npts
 * integer points xyz[3 * i + 0..2] of the logical grid, the index in curve order (global:
 * with the shard's offset; the order of dvl_get_sorted and of the bin ranges) of the cell
 * whose 2^L cube contains it, or -1 if no cell of this context does (a gap, or outside
 * [0, 2^b)^3).  A pixel brush [x0, x1] selects the cells [lo[x0], hi[x1]] of
 * dvl_get_bin_ranges, so a point is inside the brushed region iff its index is in that
 * range.  xyz and cell are in memory space `where` (host: synchronises).  Errors: STATE,
 * INVAL, NOMEM, CUDA. */
dvl_status dvl_locate(dvl_ctx *ctx, uint64_t npts, const uint32_t *xyz, int64_t *cell,
                      dvl_mem where);

/* Brushing ("We use the ROIs' first and last Hilbert codes as selection ranges"):
 * the cells selected by brushing pixels x0..x1 (0 <= x0 <= x1 < W) of the last polylines of
 * width W are the curve-order range [lo(x0), hi(x1)] of the bin ranges; out4 = {first cell,
 * last cell (global curve-order indices), the first cell's code, the last cell's code}.  A
 * sharded context with a communicator calls it collectively (every rank gets both codes);
 * without one, a code of a cell held by another shard is ~0.  Synchronises.  Errors: STATE
 * (no polylines of width W yet), INVAL. */
dvl_status dvl_brush(dvl_ctx *ctx, uint32_t W, uint32_t x0, uint32_t x1, uint64_t *out4);

/* The 3D side of brushing and linking: for each integer point of the logical
 * grid, 1 if the cell containing it (dvl_locate) has a code in [code_lo, code_hi] (the ROI
 * as Hilbert codes, from dvl_brush), else 0 (also for points in no cell).  flag: npts int64
 * in memory space `where`.  Errors: as dvl_locate. */
dvl_status dvl_roi_contains(dvl_ctx *ctx, uint64_t npts, const uint32_t *xyz, uint64_t code_lo,
                            uint64_t code_hi, int64_t *flag, dvl_mem where);

/* Milliseconds of the last build / update / get_polylines, measured with CUDA events on
 * the context stream (only with DVL_FLAG_TIMING; otherwise all zero). */
typedef struct {
    float ingest_ms, encode_ms, sort_ms, gather_ms;      /* build phases */
    float maxv_ms, weights_scan_ms;                      /* dvl_update_tf */
    float bin_reduce_ms, epilogue_ms;                    /* dvl_get_polylines: pass 2
                                                            (with its boundary warp tiles),
                                                            epilogue */
    float bin_boundary_ms;                               /* 0: kept for the layout (the
                                                            boundary warp tiles are part of
                                                            pass 2) */
    int32_t sort_passes;
    int32_t launches;     /* kernels launched since the previous dvl_get_timings call */
} dvl_timings;

/* Create a context on init->device.  out receives the handle.  Errors: INVAL (NULL
 * arguments, bad device), CUDA. */
dvl_status dvl_create(const dvl_init *init, dvl_ctx **out);

/* Free everything the context owns (after synchronising its stream).  NULL is a no-op. */
void dvl_destroy(dvl_ctx *ctx);

/* Text of the last error of this context ("" if none); owned by the context. */
const char *dvl_last_error(const dvl_ctx *ctx);

/* Name of a status code ("DVL_OK", ...). */
const char *dvl_status_string(dvl_status s);

/* BUILD (readings O1-O5).
 *   n          number of cells, 1 <= n < 2^30
 *   lower_xyz  n x 3 uint32, AoS, the cell's lower corner on the logical grid; every
 *              coordinate must be a multiple of 2^level
 *   level      n uint8, AMR level (0 = finest, cell width 2^L, L <= 20)
 *   members    M, 1 <= M <= 64 ensemble members / fields
 *   scalars    M pointers, each to n float32 values in the same cell order
 *   where      memory space of lower_xyz, level and the M scalar arrays
 * Computes E, b, Lmax, member data ranges (finite values only), the Hilbert code of every
 * cell's floored centroid lower + (2^L >> 1), sorts the cells by code and stores levels
 * and scalars in curve order (structure of arrays).  Synchronous.  Rebuilding replaces
 * the dataset and resets every TF to the identity ramp (N = 256) and every domain to the
 * member's data range; P/eps/maxV mode are kept.
 * Errors: INVAL (n = 0, M out of range, L > 20, misaligned lower), RANGE (E > 2^21 or
 * n >= 2^30), OVERLAP (two cells overlap), NOMEM, CUDA. */
dvl_status dvl_build(dvl_ctx *ctx, uint64_t n, const uint32_t *lower_xyz, const uint8_t *level,
                     uint32_t members, const float *const *scalars, dvl_mem where);

/* Exponent P in [0, 16] (Eq. 3), minimum importance eps in [0, 1], and the
 * max(V_h) mode.  Defaults 1, 0.025, CONSERVATIVE.  Takes effect at the next
 * dvl_update_tf.  EXACT on a shard takes the max over every shard's cells (an all_reduce on
 * the context's communicator: this call and every TF install are then collective; without
 * a communicator such a shard fails with STATE).  Errors: INVAL (NaN or out of range),
 * RANGE (after a build: ceil(Lmax * P) > 100, fp32 weight overflow, reading A29). */
dvl_status dvl_set_params(dvl_ctx *ctx, float P, float eps, dvl_maxv_mode mode);

/* The level factor of the importance (Eq. 3): the cell width, f = (V/maxV 2^L)^P
 * (default), or "another sensible choice ... by their volume", f =
 * (V/maxV 2^3L)^P; the shift s becomes 61 - ceil(log2 n) - ceil(3 Lmax P).  Takes effect
 * immediately (weights recomputed).  Errors: INVAL, RANGE (after a build: ceil(3 Lmax P) >
 * 100). */
typedef enum { DVL_SCALE_WIDTH = 0, DVL_SCALE_VOLUME = 1 } dvl_level_scale;
dvl_status dvl_set_level_scale(dvl_ctx *ctx, dvl_level_scale scale);

/* Normalisation domain [lo, hi] of one member (reading O6/A7): t =
 * clamp((v - lo) * inv, 0, 1) with inv = hi > lo ? 1/(hi - lo) : 0.  Default after a
 * build: the member's finite data range.  Errors: STATE (before build), INVAL (member
 * >= M, non-finite bounds, hi < lo). */
dvl_status dvl_set_domain(dvl_ctx *ctx, uint32_t member, float lo, float hi);

/* Replace member `member`'s transfer function and recompute the importance, the
 * fixed-point weights and their prefix sum (U0-U2).
 *   rgba  N x 4 float32 (r, g, b, alpha per entry), host memory, each in [0, 1];
 *         entries are sampled piecewise-linearly on t * (N - 1) (reading O8)
 *   N     2 <= N <= 4096, and equal to the size of the other members' TFs (all members
 *         share N; dvl_reset_tfs changes it for all)
 * Asynchronous on the context stream.  Errors: STATE, INVAL, CUDA. */
dvl_status dvl_update_tf(dvl_ctx *ctx, uint32_t member, const float *rgba, uint32_t N);

/* Set every member's TF to the identity alpha ramp with grey rgb, of size N (2..4096),
 * and recompute the weights.  Errors: STATE, INVAL. */
dvl_status dvl_reset_tfs(dvl_ctx *ctx, uint32_t N);

/* Project the cells onto W pixel bins and reduce them (U3-U5).
 *   W    2 <= W <= 65536
 *   out  M x W dvl_vertex, member-major (out[m * W + x]), in memory space `where`
 * Uses the weights of the last update (the identity TFs after a build).  Host output
 * synchronises; page-locked host output (16-byte aligned) is written by the last kernel
 * directly (zero copy), pageable host output through one device-to-host copy.  Errors:
 * STATE, INVAL, DEGENERATE (all weights are 0), CUDA. */
dvl_status dvl_get_polylines(dvl_ctx *ctx, uint32_t W, dvl_vertex *out, dvl_mem where);

/* ---- sharding: one context per GPU, each holding a contiguous range of the global curve
 * order.  Only two things cross shards per TF edit: the scan offset (the
 * sum of the earlier shards' fixed-point weights) and the per-pixel accumulators, which
 * are integers and merge exactly with a MAX and a SUM collective.  Either the context
 * runs them itself on its own NCCL communicator (dvl_set_comm: libnccl.so.2 is loaded at
 * run time with dlopen, so there is no link-time NCCL dependency), or the caller runs them
 * between dvl_shard_reduce and dvl_shard_finish (e.g. torch.distributed over gloo). ------- */

/* Hilbert bits of the whole dataset, used by the next dvl_build of this shard instead of
 * the shard's own extent (codes depend on b, so all shards must agree).  0 = own extent.
 * Errors: INVAL (bits outside [0, 21]); the build fails with RANGE if the shard's extent
 * exceeds 2^bits. */
dvl_status dvl_set_global_bits(dvl_ctx *ctx, int bits);

typedef struct {
    uint64_t cell_offset;   /* global curve index of this shard's first cell */
    uint64_t n_global;      /* cells of all shards (enters the fixed-point shift s) */
    int32_t lmax_global;    /* coarsest level of all shards (enters s) */
    int32_t reserved;
    const float *vmin;      /* M global finite data minima (host), or NULL: keep this shard's */
    const float *vmax;      /* M global finite data maxima (host), or NULL */
} dvl_shard_info;

/* Declare this context a shard of a larger dataset (after dvl_build).  Resets every
 * member's domain to the (global) data range and recomputes the weights.  Errors: STATE,
 * INVAL (cell_offset + n > n_global, lmax below this shard's Lmax). */
dvl_status dvl_set_shard(dvl_ctx *ctx, const dvl_shard_info *info);

/* Local sum of the fixed-point weights of the last update (one u64), copied
 * asynchronously to device memory total_dev (e.g. a slot of an all-gather buffer). */
dvl_status dvl_shard_total(dvl_ctx *ctx, uint64_t *total_dev);

/* Number of int64 words of the accumulator export for width W: 2 (W + M W) + 3 M W. */
uint64_t dvl_shard_export_words(dvl_ctx *ctx, uint32_t W);

/* The context's own NCCL communicator over the shards (NCCL over NVLink, loaded
 * at run time from libnccl.so.2).  dvl_nccl_unique_id writes a 128-byte ncclUniqueId (call
 * on one rank, broadcast it); dvl_set_comm (on every rank, collectively: blocks until all
 * ranks join) makes rank `rank` of `nranks`.  A sharded context (dvl_set_shard) with a
 * communicator runs the whole sharded edit in dvl_get_polylines: all_gather of the Q totals,
 * pass 2 with the global offset, the accumulator export and one grouped MAX + SUM all_reduce
 * of it, the merged epilogue -- the same result as dvl_shard_total / _reduce / _finish with
 * the caller's collectives, in one call.  Errors: INVAL, NCCL, CUDA. */
dvl_status dvl_nccl_unique_id(void *id128);
dvl_status dvl_set_comm(dvl_ctx *ctx, int nranks, int rank, const void *id128);

/* An in-process group of nranks contexts (driven by nranks host threads of one process, on
 * one or several devices): the same collectives as NCCL, done as device-to-device copies
 * between the ranks' buffers with a host barrier.  It lets the whole distributed path run
 * through this ABI on a single GPU (NCCL cannot place two ranks on one device).  The group
 * handle is reference counted: destroy it whenever; the contexts keep their share. */
dvl_status dvl_local_group_create(int nranks, void **group);
void dvl_local_group_destroy(void *group);
dvl_status dvl_set_local_comm(dvl_ctx *ctx, void *group, int rank);

/* Distributed build (SURVEY 8(e) "Build"; the order of P:309-311 over all ranks).  When the
 * context has a communicator (dvl_set_comm / dvl_set_local_comm), dvl_build is collective:
 * every rank passes its own slice of the cells (any slice, possibly empty, same member
 * count), and the library runs the Hilbert-key sample sort: all_reduce of the extent /
 * Lmax / n (one global code width b), local encode + sort + gather, 1024 regular samples per
 * rank all_gathered, G-1 splitters by dvl_select_splitters' rule, send ranges by binary
 * search, the G x G counts all_gathered, the codes / global input ids / levels / member rows
 * exchanged (grouped send / recv), the received sorted runs combined by the bucket placement
 * of distinct codes, the dyadic overlap rule checked inside and across the rank
 * boundaries, member ranges and offsets agreed.  Each rank then holds one contiguous range
 * of the global curve order as a shard (dvl_get_shard), and dvl_get_polylines runs the
 * sharded edit.  dvl_get_sorted returns the global input ids (the slices' concatenation in
 * rank order).  All ranks return the same status. */
dvl_status dvl_get_shard(dvl_ctx *ctx, dvl_shard_info *out);   /* vmin / vmax set to NULL */

/* The sample sort's splitter rule, on the host: samples = nranks rows of per_rank codes
 * (rank p's first min(per_rank, counts[p]) entries are its regular samples), counts[p] =
 * cells of rank p.  Writes nranks-1 strictly increasing splitters (the weighted global
 * quantiles k n / nranks).  Errors: INVAL (no strictly increasing choice exists). */
dvl_status dvl_select_splitters(const uint64_t *samples, const uint64_t *counts, int nranks,
                                int per_rank, uint64_t *splitters);

/* Pass 2 of this shard (U3+U4) with the global scan offset and Qtot derived on the device
 * from totals_dev[nshards] (the gathered dvl_shard_total values, shard order), then export
 * of the per-pixel accumulators to export_dev (device, dvl_shard_export_words int64): the
 * negated MIN plane (-first cell, -tmin bits), the MAX plane (last cell, tmax bits) and the
 * SUM plane (128-bit sums as limbs of weight 2^0, 2^32, 2^64, each < 2^33), see
 * csrc/shard.cu.  Merge: element-wise
 * MAX over the first 2 (W + M W) words, SUM over the rest.  Asynchronous.  Errors: STATE,
 * INVAL. */
dvl_status dvl_shard_reduce(dvl_ctx *ctx, uint32_t W, const uint64_t *totals_dev, int nshards,
                            int shard, int64_t *export_dev);

/* U5 from the merged export (element-wise MAX over all shards of the -MIN and MAX planes,
 * SUM of the SUM plane): out = M x W vertices as dvl_get_polylines.  Host output synchronises.
 * Errors: STATE, INVAL, DEGENERATE (merged Qtot = 0, checked with host output). */
dvl_status dvl_shard_finish(dvl_ctx *ctx, uint32_t W, const int64_t *merged_dev,
                            dvl_vertex *out, dvl_mem where);

/* ---- introspection / validation exports (copy-out; not on the timed path) ---------- */

/* Scalars describing the dataset and the last update.  Synchronises. */
dvl_status dvl_info(dvl_ctx *ctx, dvl_info_t *info);

/* Sorted Hilbert codes (n x u64) and, for each sorted position, the input cell id
 * (n x u64).  Either pointer may be NULL.  Errors: STATE, CUDA. */
dvl_status dvl_get_sorted(dvl_ctx *ctx, uint64_t *codes, uint64_t *ids, dvl_mem where);

/* Levels (n x u8) and member scalars (M x n f32, member-major) in curve order. */
dvl_status dvl_get_sorted_data(dvl_ctx *ctx, uint8_t *level_sorted, float *scalars_sorted,
                               dvl_mem where);

/* Inclusive prefix Q(h) of the fixed-point weights of the last update (n x u64; the
 * per-cell weight is q(h) = Q(h) - Q(h-1)).  Recomputes them from the current TFs with
 * the same kernels and an export flag on.  Errors: STATE, CUDA. */
dvl_status dvl_get_prefix(dvl_ctx *ctx, uint64_t *Q, dvl_mem where);

/* First and last sorted cell index of every bin of the last dvl_get_polylines with
 * this W (W x u64 each).  Errors: STATE (no polylines for this W yet), CUDA. */
dvl_status dvl_get_bin_ranges(dvl_ctx *ctx, uint32_t W, uint64_t *lo, uint64_t *hi,
                              dvl_mem where);

/* Per-phase CUDA-event times of the last calls (see dvl_timings). */
dvl_status dvl_get_timings(dvl_ctx *ctx, dvl_timings *t);

/* Switch the per-kernel CUDA events of DVL_FLAG_TIMING on (enable != 0) or off, e.g. to time
 * a sequence of calls without the event records between its kernels.  Errors: INVAL. */
dvl_status dvl_set_timing(dvl_ctx *ctx, int enable);

/* The context's CUDA stream (cudaStream_t), for callers that enqueue work around it. */
void *dvl_stream(dvl_ctx *ctx);

/* Host-side evaluation of the library's table-driven Hilbert encoder (the same state
 * tables the GPU kernel loads, reading A1): codes of n points (n x 3 uint32,
 * AoS, each coordinate < 2^bits) with 1 <= bits <= 21.  Needs no GPU.  Errors: INVAL. */
dvl_status dvl_hilbert_encode_host(uint64_t n, const uint32_t *xyz, int bits, uint64_t *codes);

/* Number of states of the derived Hilbert state machine (for tests/documentation). */
int dvl_hilbert_states(void);

#ifdef __cplusplus
}
#endif

#endif /* DVL_H */
