/*
 * pct.h — C ABI of the B200 point-cloud-tomography library (libpct.so).
 *
 * Drop-in boundary for the hot path of the reference package `tomoplan`
 * (arXiv 2403.07631): tomogram build -> traversability evaluation -> slice
 * simplification.  The reference is pure Python with no FFI of its own; each
 * entry point below names the reference function it replaces (file:line under
 * /root/reference/pkg/src/tomoplan/).  The Python mirror of the reference API
 * (paper_2403_07631_b200/*.py) binds these with ctypes; INTEGRATION.md shows the
 * binding a tomoplan maintainer would add.
 *
 * Conventions
 *  - Plain C types only.  `xyz` is an (n, 3) row-major array of float32
 *    (dtype PCT_F32) or float64 (PCT_F64).  Layers are float32, row-major
 *    (rows, cols) per slice, slices contiguous: index (k*rows + i)*cols + j.
 *    Invalid cells are NaN with bits 0x7FC00000 (numpy's NaN).
 *  - Every function returns 0 (PCT_OK) or a negative PCT_E* code and never
 *    throws; pct_last_error(ctx) holds the message.  Argument errors are
 *    reported with the reference's exception text where one exists.
 *  - A context owns one device, one CUDA stream and its scratch; it is not
 *    re-entrant.  Device pointers passed in must live on the context's device.
 *  - Functions that return host-visible results synchronise the context
 *    stream; the others are stream-ordered (pct_sync waits).
 */
#ifndef PCT_H_
#define PCT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCT_ABI_VERSION 1

enum {
  PCT_OK = 0,
  PCT_E_INVALID = -1,    /* ValueError in the reference */
  PCT_E_GRID = -2,       /* GridSizeError (tomogram.py:25-26,141-142) */
  PCT_E_CUDA = -3,       /* CUDA runtime failure -> RuntimeError */
  PCT_E_NOMEM = -4,      /* device or pinned allocation failed */
  PCT_E_EMPTY = -5,      /* CloudFormatError("zero valid points"), cloud_io.py:38-39 */
  PCT_E_NONFINITE = -6,  /* ValueError non-finite coordinates, cloud_io.py:40-41 */
  PCT_E_NOCOST = -7,     /* ValueError "slice has no cost layer" simplify.py:34-35 */
  PCT_E_RANGE = -8,      /* IndexError, simplify.py:49-50 */
  PCT_E_IO = -9          /* CloudFormatError: unreadable / truncated file, cloud_io.py:142-144 */
};

enum { PCT_F32 = 0, PCT_F64 = 1 };
enum { PCT_LAYER_GROUND = 0, PCT_LAYER_CEILING = 1, PCT_LAYER_COST = 2 };

/* TravParams (traversability.py:21-56) with patch_radius resolved for r_g. */
typedef struct {
  double d_min, d_ref, theta_b, theta_s, theta_p, c_barrier;
  double alpha_d, alpha_b, alpha_s;
  int32_t patch_radius;
  int32_t _pad;
} pct_trav_params;

/* Grid frame of tomogram.py:134-145. heights are z_min + d_s*(k+1). */
typedef struct {
  double origin_x, origin_y, z_min, d_s, r_g;
  int32_t rows, cols, n_slices;
  int32_t _pad;
} pct_frame;

typedef struct pct_ctx pct_ctx;
typedef struct pct_tomo pct_tomo; /* device-resident tomogram (ground/ceiling/cost stacks) */

/* ---- context --------------------------------------------------------- */
int pct_abi_version(void);
int pct_ctx_create(int device, pct_ctx **out);
int pct_ctx_destroy(pct_ctx *ctx);
const char *pct_last_error(const pct_ctx *ctx);
int pct_sync(pct_ctx *ctx);
/* Kernel launches issued by this context since creation (evidence counter). */
int64_t pct_launch_count(const pct_ctx *ctx);
/* Use an external stream (cudaStream_t as void*); NULL restores the own stream.
 * Work already queued on the previous stream is ordered before anything the
 * context issues on the new one (event join). */
int pct_set_stream(pct_ctx *ctx, void *stream);

/* ---- memory helpers (device / pinned host, owned by the caller) ------- */
int pct_malloc(pct_ctx *ctx, size_t bytes, void **dptr);
int pct_free(pct_ctx *ctx, void *dptr);
int pct_host_alloc(pct_ctx *ctx, size_t bytes, void **hptr);
int pct_host_free(pct_ctx *ctx, void *hptr);
/* Page-lock existing host memory (e.g. a shared-memory segment several
   processes write their bands into) for DMA; unregister before unmapping. */
int pct_host_register(pct_ctx *ctx, void *hptr, size_t bytes);
int pct_host_unregister(pct_ctx *ctx, void *hptr);
int pct_memcpy_h2d(pct_ctx *ctx, void *dst, const void *src, size_t bytes);
int pct_memcpy_d2h(pct_ctx *ctx, void *dst, const void *src, size_t bytes); /* syncs */
int pct_memcpy_d2h_async(pct_ctx *ctx, void *dst, const void *src, size_t bytes);

/* ---- stage 0: bounds (cloud_io.py:47-50, PointCloud.bounds) ------------ */
/* Exact float64 min/max of device xyz. Fails with PCT_E_NONFINITE on NaN/Inf. */
int pct_bounds(pct_ctx *ctx, const void *xyz, int64_t n, int dtype, double lo[3], double hi[3]);

/* Host-only grid frame (tomogram.py:134-145); heights_out may be NULL. */
int pct_frame_compute(const double lo[3], const double hi[3], double d_s, double r_g,
                      int64_t max_grid_side, pct_frame *fr, double *heights_out,
                      int32_t heights_cap);

/* ---- stage 1: tomogram build (tomogram.py:127-213) -------------------- */
/* Device in, device out: ground/ceiling are (S, rows, cols) float32. */
int pct_build(pct_ctx *ctx, const void *xyz, int64_t n, int dtype, const pct_frame *fr,
              const double *heights, float *ground, float *ceiling);

/* ---- stage 2: traversability (traversability.py:59-236) ---------------- */
/* kernel_w: host (kside x kside) float32 weights from build_kernel
   (traversability.py:194-202). Fused interval+terrain+fuse+inflate per slice. */
int pct_evaluate(pct_ctx *ctx, const float *ground, const float *ceiling, int32_t n_slices,
                 int32_t rows, int32_t cols, double r_g, const pct_trav_params *p,
                 const float *kernel_w, int32_t kside, float *cost);
/* pct_evaluate with the slice-change masks of the stacks (the ones the
   build wrote, pct_tomo_masks): the terrain walk then skips deriving them
   (one pass over ground + ceiling).  masks: device [2][rows*cols] uint64,
   bit k = ground / ceiling of slice k differs from slice k-1, bit 0 set;
   NULL (or n_slices > 64) behaves as pct_evaluate. */
int pct_evaluate_masked(pct_ctx *ctx, const float *ground, const float *ceiling, int32_t n_slices,
                        int32_t rows, int32_t cols, double r_g, const pct_trav_params *p,
                        const float *kernel_w, int32_t kside, const uint64_t *masks,
                        float *cost);
/* pct_evaluate_masked that also records, per evaluation tile, the slices
   whose costs may differ from the slice below: tile_masks (device uint64,
   pct_tile_masks_bytes(rows, cols) bytes), tile_geom[2] = the tile height
   and width (0, 0 when this evaluation path recorded none).  With the
   build's masks they let pct_simplify_masked read only where values
   change. */
int64_t pct_tile_masks_bytes(int32_t rows, int32_t cols);
int pct_evaluate_tiles(pct_ctx *ctx, const float *ground, const float *ceiling, int32_t n_slices,
                       int32_t rows, int32_t cols, double r_g, const pct_trav_params *p,
                       const float *kernel_w, int32_t kside, const uint64_t *masks, float *cost,
                       uint64_t *tile_masks, int32_t *tile_geom);
/* per-op entry points on one (rows, cols) layer, device pointers */
int pct_interval_cost(pct_ctx *ctx, const float *ground, const float *ceiling, int32_t rows,
                      int32_t cols, const pct_trav_params *p, float *out);      /* :59-73 */
int pct_ground_cost(pct_ctx *ctx, const float *ground, int32_t rows, int32_t cols, double r_g,
                    const pct_trav_params *p, float *out);                      /* :150-159 */
int pct_slope_magnitudes(pct_ctx *ctx, const float *ground, int32_t rows, int32_t cols,
                         double r_g, double *m_xy, double *m_grad, uint8_t *isolated); /* :106-114 */
int pct_fuse_costs(pct_ctx *ctx, const float *c_interval, const float *c_ground,
                   const uint8_t *ground_valid, int32_t rows, int32_t cols,
                   const pct_trav_params *p, float *out);                       /* :162-170 */
int pct_inflate(pct_ctx *ctx, const float *cost, int32_t rows, int32_t cols,
                const float *kernel_w, int32_t kside, float *out);              /* :205-213 */
int pct_gentle_fraction(pct_ctx *ctx, const uint8_t *gentle, int32_t rows, int32_t cols,
                        int32_t radius, double *out);                           /* :117-128 */
int pct_terrain_cost_values(pct_ctx *ctx, const double *m_xy, const double *m_grad,
                            const double *p_s, int64_t n, const pct_trav_params *p,
                            double *out);                                       /* :131-147 */

/* ---- stage 3: simplification (simplify.py:18-73) ---------------------- */
/* Runs the reference's forward sweep to a fixpoint; writes the surviving
   original slice indices (ascending) to keep_host[0..*n_keep). */
int pct_simplify(pct_ctx *ctx, const float *ground, const float *cost, int32_t n_slices,
                 int32_t rows, int32_t cols, double eps_e, double c_barrier,
                 int32_t *keep_host, int32_t *n_keep);
/* pct_simplify with the build's slice-change masks of the ground stack and
   the tile masks pct_evaluate_tiles recorded for the cost stack (same
   slices); NULL / zero geometry behaves as pct_simplify. */
int pct_simplify_masked(pct_ctx *ctx, const float *ground, const float *cost, int32_t n_slices,
                        int32_t rows, int32_t cols, double eps_e, double c_barrier,
                        const uint64_t *masks, const uint64_t *tile_masks,
                        const int32_t *tile_geom, int32_t *keep_host, int32_t *n_keep);
/* unique-cell mask of slice k given neighbour slices (-1 = none), simplify.py:31-53 */
int pct_unique_mask(pct_ctx *ctx, const float *ground, const float *cost, int32_t rows,
                    int32_t cols, int32_t k, int32_t below, int32_t above, double eps_e,
                    double c_barrier, uint8_t *mask);

/* ---- row-band sharding of one map over several GPUs (SURVEY.md §8 e) ---- */
/* Partition points by owner band: band b owns global rows
   [band_starts[b], band_starts[b+1]) of the frame (tomogram.py:148
   rasterisation).  out receives the points grouped by band (same dtype);
   counts_host[b] their numbers.  nbands <= 64. */
int pct_partition_rows(pct_ctx *ctx, const void *xyz, int64_t n, int dtype, const pct_frame *fr,
                       const int32_t *band_starts, int32_t nbands, void *out,
                       int64_t *counts_host);
/* Build rows [row0, row0+nrows) of the GLOBAL frame (points of other rows are
   ignored); slice k is written at k*out_slice_stride floats (0 = dense). */
int pct_build_band(pct_ctx *ctx, const void *xyz, int64_t n, int dtype, const pct_frame *fr,
                   const double *heights, int32_t row0, int32_t nrows, int64_t out_slice_stride,
                   float *ground, float *ceiling);
/* Strided slice copy on the device (halo packing / unpacking, gathering
   the kept slices of a band into a full-grid stack): for m < n,
   dst[m * dst_slice_stride .. + block_elems) = src[k * src_slice_stride ..)
   with k = slice_idx_host[m] (host array; NULL: k = m), n <= 4096.  All
   strides and sizes in floats.  Stream-ordered, no host synchronisation. */
int pct_copy_slices(pct_ctx *ctx, float *dst, int64_t dst_slice_stride, const float *src,
                    int64_t src_slice_stride, const int32_t *slice_idx_host, int32_t n,
                    int64_t block_elems);
/* ---- compacted read-back of layer slices (Layer.values / materialize of
   tomogram.py:36-62, 65-96: the layers the reference returns as numpy
   arrays) --------------------------------------------------------------------
   A slice is sent as a bitmap of its non-empty cells (bits != 0x7FC00000,
   numpy's NaN the reference writes for empty cells, tomogram.py:203-204) and
   those cells' values in cell order; pct_xfer_expand rebuilds it on the
   host.  Lossless for every bit pattern.  Slices m < n are
   src + slice_idx_host[m] * slice_stride (floats), n <= 4096.  delta = 1:
   a delta chain -- slice m > 0 is compared with (and rebuilt from) slice
   m - 1 of the list instead of the empty NaN (consecutive kept slices share
   most cells).
   pct_xfer_count: the number of non-empty cells of each slice (synchronous);
   pct_xfer_count_async: the same, stream-ordered (totals_host, page-locked,
   is valid once the stream synchronises).
   pct_xfer_pack: device buffers bitmaps [n][ceil(cells/32)] u32, packed
   (slice m's values at packed_off_host[m]), chunk_off [n][ceil(cells /
   pct_xfer_chunk_cells())] i64 (absolute packed index of each chunk's first
   value); stream-ordered.  pct_xfer_fence / pct_xfer_wait: record event
   slot (0..7) on the stream / wait for it on the host (e.g. one stack's
   packed copies landed while later copies are still in flight).
   pct_xfer_expand: host function (no context), nthreads host threads.
   pct_xfer_expand_from: the same for a delta chain continued from `base`
   (the already rebuilt slice before slice 0 of this call; its part of a
   chain whose bitmaps / chunk offsets start at slice 0 of the call), so a
   long chain can be rebuilt in parts while its later slices still cross
   PCIe. */
int pct_xfer_count(pct_ctx *ctx, const float *src, int64_t slice_stride,
                   const int32_t *slice_idx_host, int32_t n, int64_t cells, int32_t delta,
                   int64_t *totals_host);
int pct_xfer_pack(pct_ctx *ctx, const float *src, int64_t slice_stride,
                  const int32_t *slice_idx_host, int32_t n, int64_t cells, int32_t delta,
                  const int64_t *packed_off_host, uint32_t *bitmaps, float *packed,
                  int64_t *chunk_off);
int pct_xfer_count_async(pct_ctx *ctx, const float *src, int64_t slice_stride,
                         const int32_t *slice_idx_host, int32_t n, int64_t cells, int32_t delta,
                         int64_t *totals_host);
int64_t pct_xfer_chunk_cells(void);
int pct_xfer_fence(pct_ctx *ctx, int32_t slot);
int pct_xfer_wait(pct_ctx *ctx, int32_t slot);
int pct_xfer_expand(const uint32_t *bitmaps, const float *packed, const int64_t *chunk_off,
                    int32_t n, int64_t cells, int32_t delta, float *const *outs,
                    int32_t nthreads);
/* pct_xfer_count_keep: pct_xfer_count_async that also keeps the chunk and
   warp counts in counts_dev (device, pct_xfer_counts_bytes(cells, n) bytes);
   pct_xfer_pack_counted: pct_xfer_pack from those counts (same slices, same
   delta flag, the stack unchanged in between) without counting again. */
int64_t pct_xfer_counts_bytes(int64_t cells, int32_t n);
int pct_xfer_count_keep(pct_ctx *ctx, const float *src, int64_t slice_stride,
                        const int32_t *slice_idx_host, int32_t n, int64_t cells, int32_t delta,
                        int64_t *totals_host, uint32_t *counts_dev);
int pct_xfer_pack_counted(pct_ctx *ctx, const float *src, int64_t slice_stride,
                          const int32_t *slice_idx_host, int32_t n, int64_t cells, int32_t delta,
                          const int64_t *packed_off_host, const uint32_t *counts_dev,
                          uint32_t *bitmaps, float *packed, int64_t *chunk_off);
int pct_xfer_expand_from(const uint32_t *bitmaps, const float *packed, const int64_t *chunk_off,
                         int32_t n, int64_t cells, int32_t delta, float *const *outs,
                         int32_t nthreads, const float *base);
/* Sweep primitives for a distributed simplify (simplify.py:18-73): the any()
   table of the first pass (bit j of table[k]: below = k-1-j, j < 16; bit 32:
   no lower neighbour; upper neighbour k+1) and any() flags of explicit
   (below, k, above) triples (-1 = none).  Ranks OR-reduce both, then replay
   the same sweep. */
int pct_simplify_window(pct_ctx *ctx, const float *ground, const float *cost, int32_t n_slices,
                        int64_t cells, int64_t slice_stride, double eps_e, double c_barrier,
                        uint64_t *table_host);
int pct_simplify_triples(pct_ctx *ctx, const float *ground, const float *cost, int32_t n_slices,
                         int64_t cells, int64_t slice_stride, double eps_e, double c_barrier,
                         const int32_t *triples, int32_t n_triples, int32_t *flags_host);

/* ---- planner context precompute (planner.py:65-93, SURVEY.md §8 f) ----- */
/* Canonical-node arrays of an evaluated (or simplified) tomogram: canon[k]
   = first slice of the run of equal ground (|dz| <= eps_e, both valid) that
   contains slice k, cn[k] = the run's minimum cost (inf without ground). */
int pct_planner_context(pct_ctx *ctx, const float *ground, const float *cost, int32_t n_slices,
                        int32_t rows, int32_t cols, double eps_e, int32_t *canon, float *cn);

/* ---- binary PCD ingest (cloud_io.py:123-146 + _keep_finite :53-55) ----- */
/* Records of record_bytes bytes whose little-endian float32 x, y, z sit at
   byte offsets xyz_offsets[0..2] (the numpy record dtype of cloud_io.py:
   132-138; the caller parses the header).  Rows with a non-finite coordinate
   are dropped; the survivors are written in record order to xyz_out, a
   device (n_records, 3) float32 array, and counted in *n_valid (the reference
   up-casts to float64, which is exact).  Syncs. */
int pct_pcd_extract(pct_ctx *ctx, const void *records, int64_t n_records, int64_t record_bytes,
                    const int64_t xyz_offsets[3], int records_on_host, float *xyz_out,
                    int64_t *n_valid);
/* The same straight from the file: payload at byte data_offset of path
   (after the DATA line), read in chunks of chunk_bytes (<= 0: 64 MiB) by
   native threads into pinned buffers, DMA'd while the next chunk is read.
   PCT_E_IO with "<path>: truncated binary payload" if the file is short. */
int pct_pcd_load(pct_ctx *ctx, const char *path, int64_t data_offset, int64_t n_records,
                 int64_t record_bytes, const int64_t xyz_offsets[3], int64_t chunk_bytes,
                 float *xyz_out, int64_t *n_valid);

/* ---- trajectory ceiling inflation (trajectory.py:277-317, §8 f) -------- */
/* For n_slices ceiling layers (device, float32, NaN = no ceiling): flat =
   min filter over the disk of radius ceil(erosion/res) cells (<= 64) with
   +inf for invalid / outside cells; skirted = min(60, ceil(0.8/(slope*res)))
   Jacobi sweeps of the 8-neighbour chamfer descent skirt over flat.  Both
   float64 (n_slices, rows, cols) device arrays, bit-identical to
   _inflate_ceiling. */
int pct_ceiling_inflate(pct_ctx *ctx, const float *ceiling, int32_t n_slices, int32_t rows,
                        int32_t cols, double res, double erosion, double skirt_slope,
                        double *flat, double *skirted);

/* ---- whole pipeline on a device-resident tomogram ---------------------- */
/* xyz may be a device pointer (xyz_on_host = 0) or host memory (1; pinned
   memory from pct_host_alloc is fastest).  Allocates the stacks. */
int pct_tomo_build(pct_ctx *ctx, const void *xyz, int64_t n, int dtype, int xyz_on_host,
                   double d_s, double r_g, int64_t max_grid_side, pct_tomo **out);
/* Wrap caller-provided host stacks (e.g. a reference Tomogram) for evaluation. */
int pct_tomo_upload(pct_ctx *ctx, const pct_frame *fr, const double *heights,
                    const float *ground_host, const float *ceiling_host, pct_tomo **out);
int pct_tomo_evaluate(pct_ctx *ctx, pct_tomo *t, const pct_trav_params *p,
                      const float *kernel_w, int32_t kside);
int pct_tomo_simplify(pct_ctx *ctx, pct_tomo *t, double eps_e, double c_barrier,
                      int32_t *keep_host, int32_t *n_keep);
/* build -> evaluate -> simplify in one call (the whole hot path of one map;
   keep_host needs room for the slice count, at most 65536). */
int pct_tomo_run(pct_ctx *ctx, const void *xyz, int64_t n, int dtype, int xyz_on_host,
                 double d_s, double r_g, int64_t max_grid_side, const pct_trav_params *p,
                 const float *kernel_w, int32_t kside, double eps_e, double c_barrier,
                 pct_tomo **out, int32_t *keep_host, int32_t *n_keep);
/* pct_tomo_run for n_maps independent maps (BASELINE config 4; the reference
   runs one map per call, tomoplan/bench.py:50-57).  Maps are spread over the
   n_ctx contexts (one stream + scratch each, same device) and issued phase by
   phase with one synchronisation per phase.  xyz[m]: device points of map m
   (n_points[m] x 3, dtype).  keep_host: n_maps x keep_stride slice indices,
   n_keep[m] their count.  out (optional): per-map tomogram handles, else the
   stacks are freed. */
int pct_tomo_run_batch(pct_ctx **ctxs, int32_t n_ctx, int32_t n_maps, const void *const *xyz,
                       const int64_t *n_points, int dtype, double d_s, double r_g,
                       int64_t max_grid_side, const pct_trav_params *p, const float *kernel_w,
                       int32_t kside, double eps_e, double c_barrier, pct_tomo **out,
                       int32_t *keep_host, int32_t keep_stride, int32_t *n_keep);
/* Stage timing of pct_tomo_run with CUDA events on the context stream:
   ms[0] = bounds + frame + build, ms[1] = evaluate, ms[2] = simplify. */
int pct_set_timing(pct_ctx *ctx, int on);
int pct_last_stage_ms(pct_ctx *ctx, float ms[3]);
int pct_tomo_frame(const pct_tomo *t, pct_frame *fr, double *heights, int32_t heights_cap);
/* the build's slice-change masks of a tomogram (device; NULL if none), see
   pct_evaluate_masked */
const uint64_t *pct_tomo_masks(const pct_tomo *t);
/* device pointer of a layer stack (NULL if absent), e.g. for zero-copy consumers */
const float *pct_tomo_layer(const pct_tomo *t, int layer);
/* copy slice k of a layer (or all slices if k < 0) to host memory; syncs */
int pct_tomo_download(pct_ctx *ctx, const pct_tomo *t, int layer, int32_t k, float *host);
int pct_tomo_free(pct_ctx *ctx, pct_tomo *t);

#ifdef __cplusplus
}
#endif
#endif /* PCT_H_ */
