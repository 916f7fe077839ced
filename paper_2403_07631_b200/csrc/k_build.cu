// k_build.cu — K0 bounds, K1/K2 point binning + ground/ceiling scatter-reduce,
// K3 per-cell bin scan.  Replaces cloud_io.py:47-50 (bounds) and
// tomogram.py:147-213 (rasterise, z-sort, split, ufunc.at max/min passes,
// NaN encoding).
//
// Design: no sort.  Each point is binned on the device into
// b = #{k : h_k < z} (ties go to ground, tomogram.py:156-157) and reduced into
// per-(bin, cell) float32 max / min scratch planes with order-preserving
// uint32 atomics (max/min are commutative, so the result is independent of
// point order, like the reference).  A per-cell scan over bins then produces
// ground[k] = max over bins <= k and ceiling[k] = min over bins > k, writing
// numpy's NaN (0x7FC00000) where a cell is empty.
#include <cuda.h>  // CUtensorMap (the encoder is fetched with cudaGetDriverEntryPoint)
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "pct_internal.h"

namespace pct {
namespace {

#include "bulk.cuh"

__device__ __forceinline__ unsigned long long dkey(double d) {
  unsigned long long u = (unsigned long long)__double_as_longlong(d);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__host__ inline double dkey_inv(unsigned long long k) {
  unsigned long long u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  double d;
  std::memcpy(&d, &u, 8);
  return d;
}
__device__ __forceinline__ double dkey_inv_dev(unsigned long long k) {
  const unsigned long long u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double((long long)u);
}

// ---------------------------------------------------------------- K0 bounds
// keys[0..2] = min (atomicMin), keys[3..5] = max (atomicMax), keys[6] = #non-finite
// min/max in the input precision (exact), widened to float64 only at the end
template <typename T>
struct MinMax3 {
  T lo[3], hi[3];
  unsigned nonfinite;
};

template <typename T>
__device__ __forceinline__ void mm_point(MinMax3<T> &m, T x, T y, T z) {
  const T v[3] = {x, y, z};
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    if (!isfinite(v[c])) m.nonfinite++;
    m.lo[c] = v[c] < m.lo[c] ? v[c] : m.lo[c];
    m.hi[c] = v[c] > m.hi[c] ? v[c] : m.hi[c];
  }
}

template <typename T>
__device__ __forceinline__ void bounds_body(const T *__restrict__ xyz, int64_t n,
                                            unsigned long long *keys) {
  MinMax3<T> m;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    m.lo[c] = INFINITY;
    m.hi[c] = -INFINITY;
  }
  m.nonfinite = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool vec = false;
  if constexpr (sizeof(T) == 4) {
    if ((reinterpret_cast<uintptr_t>(xyz) & 15) == 0) {
      // 4 points = 12 floats = 3 x float4 per step (xyz is 16 B aligned)
      vec = true;
      const int64_t groups = n / 4;
      const float4 *v = reinterpret_cast<const float4 *>(xyz);
      for (int64_t g = t; g < groups; g += stride) {
        float4 a = __ldg(v + 3 * g), b = __ldg(v + 3 * g + 1), c = __ldg(v + 3 * g + 2);
        mm_point(m, a.x, a.y, a.z);
        mm_point(m, a.w, b.x, b.y);
        mm_point(m, b.z, b.w, c.x);
        mm_point(m, c.y, c.z, c.w);
      }
      for (int64_t p = groups * 4 + t; p < n; p += stride)
        mm_point(m, xyz[3 * p], xyz[3 * p + 1], xyz[3 * p + 2]);
    }
  }
  if (!vec) {  // float64, or a float32 view that is not 16 B aligned
    for (int64_t p = t; p < n; p += stride)
      mm_point(m, __ldg(xyz + 3 * p), __ldg(xyz + 3 * p + 1), __ldg(xyz + 3 * p + 2));
  }
  // warp reduce, then one atomic per warp per component
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const T a = __shfl_xor_sync(0xffffffffu, m.lo[c], off);
      const T b = __shfl_xor_sync(0xffffffffu, m.hi[c], off);
      m.lo[c] = a < m.lo[c] ? a : m.lo[c];
      m.hi[c] = b > m.hi[c] ? b : m.hi[c];
    }
    m.nonfinite += __shfl_xor_sync(0xffffffffu, m.nonfinite, off);
  }
  // block reduce through shared memory: one atomic per block and component
  // (per-warp atomics on 6 addresses serialised in L2 and dominated the kernel)
  __shared__ unsigned long long red[8][7];
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      red[warp][c] = dkey((double)m.lo[c]);
      red[warp][3 + c] = dkey((double)m.hi[c]);
    }
    red[warp][6] = m.nonfinite;
  }
  __syncthreads();
  if (threadIdx.x < 7) {
    const int c = threadIdx.x;
    unsigned long long v = red[0][c];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      const unsigned long long u = red[w][c];
      v = c < 3 ? (u < v ? u : v) : (c < 6 ? (u > v ? u : v) : v + u);
    }
    if (c < 3) atomicMin(keys + c, v);
    else if (c < 6) atomicMax(keys + c, v);
    else if (v) atomicAdd(keys + 6, v);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) bounds_kernel(const T *__restrict__ xyz, int64_t n,
                                                     unsigned long long *keys) {
  bounds_body(xyz, n, keys);
}

// ------------------------------------------------------- K1+K2 bin/scatter
constexpr int kMaxStagedHeights = 4096;

struct BinArgs {
  double x0, y0, z0, r_g, d_s, inv_rg, inv_ds;
  const double *heights;  // (S,) device
  int64_t cells;          // band_rows * cols
  int rows, cols, S;      // rows = band rows; the frame is global
  int row0;               // first global row of the band
  int derive;             // heights[k] == z0 + d_s (k + 1): staged from the formula, not loaded
};

// the plane heights of pct_frame_compute, evaluated the same way (no contraction)
__device__ __forceinline__ double plane_height(const BinArgs &a, int k) {
  return __dadd_rn(a.z0, __dmul_rn(a.d_s, (double)k + 1.0));
}

template <typename T>
__device__ __forceinline__ void scatter_body(const T *__restrict__ xyz, int64_t n, const BinArgs &a,
                                             uint32_t *__restrict__ gkey,
                                             uint32_t *__restrict__ ckey,
                                             unsigned long long *outside) {
  // plane heights staged in shared memory for the bin fix-ups (dynamic
  // shared size is 0 when S is too large; then they are read from global)
  extern __shared__ double hsm[];
  const bool staged = a.S <= kMaxStagedHeights;
  if (staged)
    for (int k = threadIdx.x; k < a.S; k += blockDim.x)
      hsm[k] = a.derive ? plane_height(a, k) : a.heights[k];
  __syncthreads();
  const double *hts = staged ? hsm : a.heights;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
    const double x = (double)__ldg(xyz + 3 * p);
    const double y = (double)__ldg(xyz + 3 * p + 1);
    const double z = (double)__ldg(xyz + 3 * p + 2);
    // rasterisation in float64 (tomogram.py:148-149); the division is the
    // correctly rounded Markstein form (== IEEE (y - y0) / r_g)
    const double fi = floor(div_const(y - a.y0, a.r_g, a.inv_rg) + 0.5) - (double)a.row0;
    const double fj = floor(div_const(x - a.x0, a.r_g, a.inv_rg) + 0.5);
    if (!(fi >= 0.0 && fi < (double)a.rows && fj >= 0.0 && fj < (double)a.cols)) {
      if (outside) atomicAdd(outside, 1ull);
      continue;
    }
    const int64_t cell = (int64_t)fi * a.cols + (int64_t)fj;
    // b = #{k : h_k < z}: estimate from the plane spacing, then fix up
    // against the exact float64 heights (searchsorted side="right", :157)
    double est = floor((z - a.z0) * a.inv_ds);  // estimate only; fixed up exactly below
    int b = est < 0.0 ? 0 : (est > (double)a.S ? a.S : (int)est);
    while (b > 0 && hts[b - 1] >= z) --b;
    while (b < a.S && hts[b] < z) ++b;
    const uint32_t key = f32_key(__double2float_rn(z));
    if (b < a.S) atomicMax(gkey + (int64_t)b * a.cells + cell, key);
    if (b > 0) atomicMin(ckey + (int64_t)(b - 1) * a.cells + cell, key);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) scatter_kernel(const T *__restrict__ xyz, int64_t n,
                                                      BinArgs a, uint32_t *__restrict__ gkey,
                                                      uint32_t *__restrict__ ckey,
                                                      unsigned long long *outside) {
  scatter_body(xyz, n, a, gkey, ckey, outside);
}

// Speculative scatter (single maps): the grid frame of pct_frame_compute
// derived on the device from the bounds keys (same IEEE operations, no
// contraction), so the scatter can run before the host has read the bounds.
// ok = 0 when the frame would not take the atomic single-map path
// (non-finite points, grid over the limit, too many slices to stage, keys
// beyond the buffer half or the tiled-build threshold).
struct SpecFrame {
  BinArgs a;
  int ok;
};
constexpr int kSpecMaxS = 512;  // the launch stages at most this many heights (4 KB)

__global__ void spec_frame_kernel(const unsigned long long *__restrict__ keys, double d_s,
                                  double r_g, int64_t max_side, double half_bytes,
                                  double max_key_bytes, SpecFrame *__restrict__ f) {
  if (threadIdx.x != 0) return;
  f->ok = 0;
  if (keys[6]) return;
  double lo[3], hi[3];
  for (int c = 0; c < 3; ++c) {
    lo[c] = dkey_inv_dev(keys[c]);
    hi[c] = dkey_inv_dev(keys[3 + c]);
  }
  const double qy = __ddiv_rn(__dsub_rn(hi[1], lo[1]), r_g);
  const double qx = __ddiv_rn(__dsub_rn(hi[0], lo[0]), r_g);
  const double qz = __ddiv_rn(__dsub_rn(hi[2], lo[2]), d_s);
  const double rows_d = floor(__dadd_rn(qy, 0.5)) + 2.0;
  const double cols_d = floor(__dadd_rn(qx, 0.5)) + 2.0;
  double s = ceil(__dsub_rn(qz, 1e-9));
  if (s < 1) s = 1;
  if (rows_d > (double)max_side || cols_d > (double)max_side || s > (double)kSpecMaxS) return;
  const int rows = (int)rows_d, cols = (int)cols_d, S = (int)s;
  const int64_t cells = (int64_t)rows * cols;
  const double kb = 4.0 * (double)S * (double)cells;
  if (kb > half_bytes || 2.0 * (double)S * (double)cells * 4.0 > max_key_bytes) return;
  f->a = BinArgs{lo[0], lo[1], lo[2], r_g, d_s, __ddiv_rn(1.0, r_g), __ddiv_rn(1.0, d_s),
                 nullptr, cells, rows, cols, S, 0, 1};
  f->ok = 1;
}

template <typename T>
__global__ void __launch_bounds__(256) spec_scatter_kernel(const T *__restrict__ xyz, int64_t n,
                                                           const SpecFrame *__restrict__ f,
                                                           uint32_t *__restrict__ keys,
                                                           int64_t half_words) {
  if (!f->ok) return;  // uniform
  const BinArgs a = f->a;
  scatter_body(xyz, n, a, keys, keys + half_words, nullptr);
}

// -------------------------------------------- tile-partitioned build (T1-T4)
// Alternative build for S <= kTileMaxS (PCT_BUILD=tiled).  Instead of S x cells scratch planes
// per reduction (memset, scattered global atomics, a full scan pass), points
// are partitioned by 16 x 16-cell tile and each tile is reduced in shared
// memory:
//   T1 tile_count: points per tile (warp-aggregated atomics)
//   T2 tile_offsets: exclusive prefix sum (one block)
//   T3 tile_scatter: one 8-byte record per point into its tile's range:
//      key(f32 z) << 32 | bin << 8 | cell within the tile
// Tiles are 8 rows x 32 columns (a warp stores whole 128-byte row segments);
// T1 / T3 give each block a contiguous range of points, so that spatially
// coherent inputs (scanner order) spread the tile counters over many tiles
// at any moment instead of serialising all blocks on a few.
//   T4 tile_reduce: one CTA per tile: shared-memory max / min per (bin, cell),
//      then the per-cell bin scan writes the tile's ground / ceiling columns
constexpr int kTBH = 8, kTBW = 32;  // tile rows x columns
constexpr int kTB2 = kTBH * kTBW;    // cells per tile (8-bit local index)
constexpr int kTileMaxS = 96;     // 2 x S x 256 x 4 B of shared memory
constexpr int kTileNT = 2 * kTB2;  // reduce: two threads per cell (ground / ceiling side)

// cell and bin of one point (tomogram.py:147-157): false when outside the band
template <bool BIN = true>
__device__ __forceinline__ bool point_cell_bin(double x, double y, double z, const BinArgs &a,
                                               const double *hts, int &fi_out, int &fj_out,
                                               int &b_out) {
  const double fi = floor(div_const(y - a.y0, a.r_g, a.inv_rg) + 0.5) - (double)a.row0;
  const double fj = floor(div_const(x - a.x0, a.r_g, a.inv_rg) + 0.5);
  if (!(fi >= 0.0 && fi < (double)a.rows && fj >= 0.0 && fj < (double)a.cols)) return false;
  fi_out = (int)fi;
  fj_out = (int)fj;
  if (!BIN) return true;  // the tile count needs the cell only
  double est = floor((z - a.z0) * a.inv_ds);  // estimate only; fixed up exactly below
  int b = est < 0.0 ? 0 : (est > (double)a.S ? a.S : (int)est);
  while (b > 0 && hts[b - 1] >= z) --b;
  while (b < a.S && hts[b] < z) ++b;
  b_out = b;
  return true;
}

// T1 / T3: every batch of 256 points (one per thread) is merged per tile in
// a shared-memory hash table, so a tile costs one global atomic per batch
// however many of the batch's points it holds (scanner-ordered inputs put
// whole batches into one tile: pillars, walls).
#ifndef PCT_PPT_COUNT
#define PCT_PPT_COUNT 4
#endif
#ifndef PCT_PPT_SCATTER
#define PCT_PPT_SCATTER 1
#endif
// points per thread per batch: the count pass merges 1024-point batches
// (cfg3 1.44 ms at 256, 1.08 at 512, 1.00 at 1024: fewer barriers and
// global atomics per point); the scatter pass keeps 256 (512: no gain);
// slots = power of 2 >= 2 x batch
template <bool SCATTER>
struct TilePass {
  static constexpr int PPT = SCATTER ? PCT_PPT_SCATTER : PCT_PPT_COUNT;
  static constexpr int HASH = 512 * PPT;
};
constexpr int kCtrPad = 32;  // tile counters / cursors: one per 128-byte line
#ifndef PCT_TILE_L2
#define PCT_TILE_L2 4
#endif
constexpr int kTileL2 = PCT_TILE_L2;  // batches of L2 prefetch ahead in the tile passes
template <typename T, bool SCATTER>
__global__ void __launch_bounds__(256) tile_pass_kernel(const T *__restrict__ xyz, int64_t n,
                                                        BinArgs a, int ntx,
                                                        unsigned *__restrict__ counter,
                                                        unsigned long long *__restrict__ recs,
                                                        unsigned long long *outside) {
  extern __shared__ double hsm[];
  constexpr int kPPT = TilePass<SCATTER>::PPT, kHash = TilePass<SCATTER>::HASH;
  __shared__ int h_tile[kHash];
  __shared__ unsigned h_cnt[kHash];
  const bool staged = a.S <= kMaxStagedHeights;
  if (staged)
    for (int k = threadIdx.x; k < a.S; k += blockDim.x)
      hsm[k] = a.derive ? plane_height(a, k) : a.heights[k];
  for (int h = threadIdx.x; h < kHash; h += blockDim.x) {
    h_tile[h] = -1;
    h_cnt[h] = 0u;
  }
  __syncthreads();
  const double *hts = staged ? hsm : a.heights;
  constexpr int BATCH = 256 * kPPT;
  const int64_t chunk = ((n + gridDim.x - 1) / gridDim.x + BATCH - 1) / BATCH * BATCH;
  const int64_t p0 = (int64_t)blockIdx.x * chunk;
  const int64_t p1 = p0 + chunk < n ? p0 + chunk : n;
  for (int64_t pb = p0; pb < p1; pb += BATCH) {  // block-uniform trip count
    if (threadIdx.x == 0 && pb + kTileL2 * BATCH < p1) {  // a later batch: DRAM -> L2
      const int64_t q0 = pb + kTileL2 * BATCH;
      const int64_t q1 = q0 + BATCH < p1 ? q0 + BATCH : p1;
      const uintptr_t a0 = reinterpret_cast<uintptr_t>(xyz + 3 * q0) & ~(uintptr_t)15;
      const uintptr_t a1 = (reinterpret_cast<uintptr_t>(xyz + 3 * q1) + 15) & ~(uintptr_t)15;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((unsigned)(a1 - a0))
                   : "memory");
    }
    int slot[kPPT], fi[kPPT], fj[kPPT], bin[kPPT];
    unsigned rank[kPPT];
    float z32[kPPT];
#pragma unroll
    for (int u = 0; u < kPPT; ++u) {
      const int64_t p = pb + u * 256 + threadIdx.x;  // coalesced per u
      bool in = false;
      slot[u] = -1;
      if (p < p1) {
        const double x = (double)__ldg(xyz + 3 * p);
        const double y = (double)__ldg(xyz + 3 * p + 1);
        const double z = SCATTER ? (double)__ldg(xyz + 3 * p + 2) : 0.0;
        in = point_cell_bin<SCATTER>(x, y, z, a, hts, fi[u], fj[u], bin[u]);
        z32[u] = __double2float_rn(z);
        if (!in && !SCATTER && outside) atomicAdd(outside, 1ull);
      }
      if (in) {
        const int tile = (fi[u] / kTBH) * ntx + fj[u] / kTBW;
        int sl = (int)(((unsigned)tile * 2654435761u) >> 20) & (kHash - 1);
        while (true) {
          const int prev = atomicCAS(&h_tile[sl], -1, tile);
          if (prev == -1 || prev == tile) break;
          sl = (sl + 1) & (kHash - 1);
        }
        slot[u] = sl;
        rank[u] = atomicAdd(&h_cnt[sl], 1u);
      }
    }
    __syncthreads();
    // one global atomic per occupied slot; the slot count becomes its base
    for (int h = threadIdx.x; h < kHash; h += blockDim.x) {
      const int tl = h_tile[h];
      if (tl >= 0) {
        // one counter per 128-byte line: atomics on neighbouring tiles do not
        // serialise in one L2 line
        if (SCATTER) h_cnt[h] = atomicAdd(counter + (int64_t)tl * kCtrPad, h_cnt[h]);
        else atomicAdd(counter + (int64_t)tl * kCtrPad, h_cnt[h]);  // RED
      }
    }
    __syncthreads();
    if (SCATTER) {
#pragma unroll
      for (int u = 0; u < kPPT; ++u)
        if (slot[u] >= 0) {
          const unsigned pos = h_cnt[slot[u]] + rank[u];
          const unsigned local = (unsigned)((fi[u] % kTBH) * kTBW + fj[u] % kTBW);
          recs[pos] = ((unsigned long long)f32_key(z32[u]) << 32) |
                      ((unsigned long long)bin[u] << 8) | local;
        }
    }
    __syncthreads();
    for (int h = threadIdx.x; h < kHash; h += blockDim.x) {
      h_tile[h] = -1;
      h_cnt[h] = 0u;
    }
    __syncthreads();
  }
}

// exclusive prefix sum of the n (padded) tile counts, reduce-then-scan over
// blocks of 1024 tiles (the counters sit one per 128-byte line: a one-block
// scan was load-latency bound, 140 us for cfg3's 62.6k tiles): T2a sums each
// block's counts, T2b adds the sums of the blocks before it and scans its
// own; offs[n] = total.  The cursors (padded) are the copy T3 advances.
__device__ __forceinline__ unsigned block_incl_scan(unsigned x, unsigned *wsum, unsigned &total) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned y = __shfl_up_sync(0xFFFFFFFFu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    unsigned w = wsum[lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned y = __shfl_up_sync(0xFFFFFFFFu, w, d);
      if (lane >= d) w += y;
    }
    wsum[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  total = wsum[31];
  return (warp ? wsum[warp - 1] : 0u) + x;
}

__global__ void __launch_bounds__(1024) tile_sums_kernel(const unsigned *__restrict__ cnt, int n,
                                                         unsigned *__restrict__ bsum,
                                                         int stride) {
  __shared__ unsigned wsum[32];
  const int i = blockIdx.x * 1024 + threadIdx.x;
  unsigned total;
  block_incl_scan(i < n ? __ldcg(cnt + (int64_t)i * stride) : 0u, wsum, total);
  if (threadIdx.x == 0) bsum[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024) tile_offsets_kernel(const unsigned *__restrict__ cnt,
                                                            int n, const unsigned *__restrict__ bsum,
                                                            unsigned *__restrict__ offs,
                                                            unsigned *__restrict__ cursor,
                                                            int stride) {
  __shared__ unsigned wsum[32];
  __shared__ unsigned base;
  const int t = threadIdx.x;
  if (t < 32) {  // sum of the blocks before this one
    unsigned s = 0;
    for (int b = t; b < (int)blockIdx.x; b += 32) s += bsum[b];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, d);
    if (t == 0) base = s;
  }
  const int i = blockIdx.x * 1024 + t;
  const unsigned v = i < n ? __ldcg(cnt + (int64_t)i * stride) : 0u;
  unsigned total;
  const unsigned incl = block_incl_scan(v, wsum, total);  // its barriers also publish `base`
  const unsigned excl = base + incl - v;
  if (i < n) {
    offs[i] = excl;
    if (cursor) cursor[(int64_t)i * stride] = excl;
  }
  if (blockIdx.x == gridDim.x - 1 && t == 0) offs[n] = base + total;
}

__global__ void __launch_bounds__(kTileNT) tile_reduce_kernel(
    const unsigned long long *__restrict__ recs, const unsigned *__restrict__ offs, int ntx,
    int rows, int cols, int S, int64_t out_stride, float *__restrict__ ground,
    float *__restrict__ ceiling) {
  extern __shared__ uint32_t tk[];  // [S][256] max keys, then [S][256] min keys
  uint32_t *gk = tk, *ck = tk + S * kTB2;
  const int tile = blockIdx.x;
  const int t = threadIdx.x;
  const unsigned r0 = offs[tile], r1 = offs[tile + 1];
  if (t == 0 && r1 > r0) {  // the tile's records DRAM -> L2 while the keys are initialised
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(recs + r0) & ~(uintptr_t)15;
    const uintptr_t a1 = (reinterpret_cast<uintptr_t>(recs + r1) + 15) & ~(uintptr_t)15;
    for (uintptr_t a = a0; a < a1; a += 65536) {
      const unsigned n = (unsigned)(a1 - a < 65536 ? a1 - a : 65536);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(n) : "memory");
    }
  }
  for (int q = t; q < S * kTB2; q += kTileNT) {
    gk[q] = kKeyEmptyMax;
    ck[q] = kKeyEmptyMin;
  }
  __syncthreads();
  for (unsigned r = r0 + t; r < r1; r += kTileNT) {
    const unsigned long long rec = __ldcs(recs + r);
    const unsigned local = (unsigned)(rec & 0xFFu);
    const int b = (int)((rec >> 8) & 0xFFFFFFu);
    const uint32_t key = (uint32_t)(rec >> 32);
    if (b < S) atomicMax(gk + b * kTB2 + local, key);
    if (b > 0) atomicMin(ck + (b - 1) * kTB2 + local, key);
  }
  __syncthreads();
  // threads 0..255 walk a cell's ground bins up, 256..511 its ceiling bins down
  const int c = t & (kTB2 - 1);
  const int ti = tile / ntx, tj = tile - ti * ntx;
  const int i = ti * kTBH + c / kTBW, j = tj * kTBW + c % kTBW;
  if (i >= rows || j >= cols) return;
  const int64_t cell = (int64_t)i * cols + j;
  if (t < kTB2) {
    uint32_t run = kKeyEmptyMax;
    for (int k = 0; k < S; ++k) {
      const uint32_t v = gk[k * kTB2 + c];
      run = v > run ? v : run;
      __stcs(ground + (int64_t)k * out_stride + cell, decode_ground(run));
    }
  } else {
    uint32_t run = kKeyEmptyMin;
    for (int k = S - 1; k >= 0; --k) {
      const uint32_t v = ck[k * kTB2 + c];
      run = v < run ? v : run;
      __stcs(ceiling + (int64_t)k * out_stride + cell, decode_ceiling(run));
    }
  }
}

// ---------------------------------------- histogram-partitioned build (H)
// The tile build's hash-merged passes replaced by per-CTA histograms: the
// grid is exactly one CTA per SM and CTA c always takes the same contiguous
// chunk of points, so
//   H1 hist_count: each CTA counts its points per bucket (16 x 32 cells) in a
//      private shared-memory histogram (plain shared atomics, no hashing, no
//      global atomics) and writes it out whole: cnt[c][b];
//   H2 hist_colscan + block scans: per bucket the column prefix over the
//      CTAs and the bucket totals, then the exclusive scan of the totals, so
//      CTA c's records of bucket b start at offs[b] + cnt[c][b];
//   H3 hist_scatter: the same chunk again, one 8-byte record per point
//      (key(f32 z) << 32 | bin << 9 | cell within the bucket) written at a
//      shared-memory cursor -- deterministic positions, no global atomics;
//   H4 hist_reduce: one CTA per bucket reduces max keys per (bin, cell) in
//      shared memory and writes the ground planes, then re-reads the
//      bucket's records (L2 hits) for the min keys and the ceiling planes
//      (half the shared memory of a two-sided reduce: two CTAs per SM).
// Traffic: 2 reads of the points + 8 B records out and back + the planes.
#ifndef PCT_HBW
#define PCT_HBW 64
#endif
constexpr int kHBW = PCT_HBW, kHBH = 512 / PCT_HBW;  // bucket: kHBH rows x kHBW columns
constexpr int kHB2 = kHBH * kHBW;          // 512 cells per bucket (9-bit local index)
constexpr int kHistNT = 1024;              // H1 / H3 threads per CTA
constexpr int kHistMaxBuckets = 48 * 1024;  // 192 KB of shared histogram
constexpr int kHistMaxS = 100;             // H4: S x 512 x 4 B <= 200 KB

template <typename T>
__device__ __forceinline__ void load_point(const T *__restrict__ xyz, int64_t p, double &x,
                                           double &y, double &z) {
  x = (double)__ldg(xyz + 3 * p);
  y = (double)__ldg(xyz + 3 * p + 1);
  z = (double)__ldg(xyz + 3 * p + 2);
}

// warp-aggregated scatter cursors (__match_any_sync): measured much slower
// at cfg3 (build 6.36 vs 3.83 ms), compile-time opt-in only
#ifndef PCT_SCATTER_MATCH
#define PCT_SCATTER_MATCH 0
#endif
// one quad of float32 points (three 16-byte vectors): count its buckets, or
// (SCATTER) place its records -- the 4 cells, bins and records first, then
// the 4 cursor atomics, then the 4 stores (independent chains in flight)
template <bool SCATTER>
// Called by every lane of the warp (the cursor aggregation is warp-wide);
// lanes without a quad pass valid = false.
__device__ __forceinline__ void hist_quad(const float4 A, const float4 B, const float4 Cv,
                                          bool valid, const BinArgs &a, const double *hts,
                                          int nbx, unsigned *h,
                                          unsigned long long *__restrict__ recs,
                                          unsigned long long *outside) {
  const double px[4] = {A.x, A.w, B.z, Cv.y}, py[4] = {A.y, B.x, B.w, Cv.z},
               pz[4] = {A.z, B.y, Cv.x, Cv.w};
  if (SCATTER) {
    int bk[4];
    unsigned long long rec[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int fi, fj, bin = 0;
      bk[u] = -1;
      if (valid && point_cell_bin<true>(px[u], py[u], pz[u], a, hts, fi, fj, bin)) {
        bk[u] = (fi / kHBH) * nbx + fj / kHBW;
        rec[u] = ((unsigned long long)f32_key(__double2float_rn(pz[u])) << 32) |
                 ((unsigned long long)bin << 9) | (unsigned)((fi % kHBH) * kHBW + fj % kHBW);
      }
    }
    unsigned pos[4];
#if PCT_SCATTER_MATCH
    // warp-aggregated cursors: lanes placing into one bucket take one atomic
    // (the leader's) and consecutive slots by lane order, so scanner-ordered
    // inputs (walls, pillars: many lanes per bucket) do not serialise on a
    // shared-memory address.  Record order inside a bucket does not change
    // any layer (max / min).
    const unsigned lane = threadIdx.x & 31u;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const unsigned act = __ballot_sync(0xFFFFFFFFu, bk[u] >= 0);
      if (bk[u] >= 0) {
        const unsigned peers = __match_any_sync(act, bk[u]);
        const int leader = __ffs(peers) - 1;
        unsigned base = 0u;
        if ((int)lane == leader) base = atomicAdd(&h[bk[u]], (unsigned)__popc(peers));
        base = __shfl_sync(peers, base, leader);
        pos[u] = base + (unsigned)__popc(peers & ((1u << lane) - 1u));
      }
    }
#else
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (bk[u] >= 0) pos[u] = atomicAdd(&h[bk[u]], 1u);
#endif
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (bk[u] >= 0) recs[pos[u]] = rec[u];
  } else {
    if (!valid) return;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int fi, fj, bin = 0;
      if (point_cell_bin<false>(px[u], py[u], pz[u], a, hts, fi, fj, bin))
        atomicAdd(&h[(fi / kHBH) * nbx + fj / kHBW], 1u);
      else if (outside)
        atomicAdd(outside, 1ull);
    }
  }
}

template <typename T, bool SCATTER>
__global__ void __launch_bounds__(kHistNT, 1) hist_pass_kernel(
    const T *__restrict__ xyz, int64_t n, BinArgs a, int nbx, int nb,
    unsigned *__restrict__ cnt, const unsigned *__restrict__ offs,
    unsigned long long *__restrict__ recs, unsigned long long *outside) {
  extern __shared__ __align__(128) unsigned char hsmem[];
  unsigned *h = reinterpret_cast<unsigned *>(hsmem);
  double *hsm = reinterpret_cast<double *>(hsmem + (((size_t)nb * 4 + 15) & ~(size_t)15));
  const int c = blockIdx.x, G = gridDim.x;
  unsigned *mine = cnt + (int64_t)c * nb;
  for (int b = threadIdx.x; b < nb; b += kHistNT) h[b] = SCATTER ? offs[b] + mine[b] : 0u;
  const bool staged = a.S <= kMaxStagedHeights;
  if (SCATTER && staged)
    for (int k = threadIdx.x; k < a.S; k += kHistNT)
      hsm[k] = a.derive ? plane_height(a, k) : a.heights[k];
  __syncthreads();
  const double *hts = staged ? hsm : a.heights;
  auto one = [&](double x, double y, double z) {
    int fi, fj, bin = 0;
    if (!point_cell_bin<SCATTER>(x, y, z, a, hts, fi, fj, bin)) {
      if (!SCATTER && outside) atomicAdd(outside, 1ull);
      return;
    }
    const int b = (fi / kHBH) * nbx + fj / kHBW;
    if (SCATTER) {
      const unsigned pos = atomicAdd(&h[b], 1u);
      const unsigned local = (unsigned)((fi % kHBH) * kHBW + fj % kHBW);
      recs[pos] = ((unsigned long long)f32_key(__double2float_rn(z)) << 32) |
                  ((unsigned long long)bin << 9) | local;
    } else {
      atomicAdd(&h[b], 1u);
    }
  };
  // CTA c's chunk (the same in both passes), quad-aligned: float32 points
  // are read 4 at a time as three 16-byte vectors (every load of a quad is
  // issued before its arithmetic)
  const int64_t p0 = (n * c / G) & ~(int64_t)3;
  const int64_t p1 = c + 1 == G ? n : (n * (c + 1) / G) & ~(int64_t)3;
  int64_t pq = p0;
  if (sizeof(T) == 4 && (reinterpret_cast<uintptr_t>(xyz) & 15) == 0) {
    const float4 *v = reinterpret_cast<const float4 *>(xyz);
    const int64_t q1 = p1 >> 2;  // whole quads
    // warp-uniform trip count: lanes past the end run with valid = false
    const int64_t lane0 = (p0 >> 2) + (threadIdx.x & ~31);
    for (int64_t qw = lane0; qw < q1; qw += kHistNT) {
      const int64_t q = qw + (threadIdx.x & 31);
      const bool ok = q < q1;
      const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
      hist_quad<SCATTER>(ok ? __ldg(v + 3 * q) : z4, ok ? __ldg(v + 3 * q + 1) : z4,
                         ok ? __ldg(v + 3 * q + 2) : z4, ok, a, hts, nbx, h, recs, outside);
    }
    pq = q1 << 2;
  }
  for (int64_t p = pq + threadIdx.x; p < p1; p += kHistNT) {
    double x, y, z;
    load_point(xyz, p, x, y, z);
    one(x, y, z);
  }
  if (!SCATTER) {
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += kHistNT) mine[b] = h[b];
  }
}

// H1 / H3 with the points staged through shared memory: the CTA's chunk
// (16-byte aligned float32 quads) arrives in kBulkQ-quad stages by 1-D bulk
// copies (cp.async.bulk, completion on a `full` mbarrier), kBulkStages
// stages in flight, so the loads never stall the arithmetic; a stage is
// refilled once all warps have arrived on its `empty` mbarrier.  Thread t
// takes quad t of every stage.  Same chunks, counts and records as
// hist_pass_kernel.
constexpr int kBulkQ = kHistNT;        // quads per stage
constexpr int kBulkBytes = kBulkQ * 48;  // 48 KB
constexpr int kBulkStages = 2;
#ifndef PCT_BULK_LASTWARP
#define PCT_BULK_LASTWARP 1
#endif
template <bool SCATTER>
__global__ void __launch_bounds__(kHistNT, 1) hist_pass_bulk_kernel(
    const float *__restrict__ xyz, int64_t n, BinArgs a, int nbx, int nb,
    unsigned *__restrict__ cnt, const unsigned *__restrict__ offs,
    unsigned long long *__restrict__ recs, unsigned long long *outside) {
  extern __shared__ __align__(128) unsigned char hsmem[];
  const size_t hist_b = ((size_t)nb * 4 + 127) & ~(size_t)127;
  // (launched only with S <= kMaxStagedHeights: the heights are always in
  // shared memory, so the bin search reads them with LDS, not generic loads)
  const size_t hts_b = SCATTER ? (((size_t)a.S * 8 + 127) & ~(size_t)127) : 0;
  unsigned *h = reinterpret_cast<unsigned *>(hsmem);
  double *hsm = reinterpret_cast<double *>(hsmem + hist_b);
  float4 *stage = reinterpret_cast<float4 *>(hsmem + hist_b + hts_b);
  uint64_t *full = reinterpret_cast<uint64_t *>(hsmem + hist_b + hts_b +
                                                (size_t)kBulkStages * kBulkBytes);
  uint64_t *empty = full + kBulkStages;
  const int c = blockIdx.x, G = gridDim.x, tid = threadIdx.x;
  unsigned *mine = cnt + (int64_t)c * nb;
  const int64_t p0 = (n * c / G) & ~(int64_t)3;
  const int64_t p1 = c + 1 == G ? n : (n * (c + 1) / G) & ~(int64_t)3;
  const int64_t q0 = p0 >> 2, q1 = p1 >> 2;
  const int64_t nst = (q1 - q0 + kBulkQ - 1) / kBulkQ;
  const float4 *v = reinterpret_cast<const float4 *>(xyz);
  auto issue = [&](int64_t i) {  // stage i -> buffer i % kBulkStages
    const int s = (int)(i % kBulkStages);
    const int64_t qa = q0 + i * kBulkQ;
    const int64_t qn = q1 - qa < kBulkQ ? q1 - qa : kBulkQ;
    mbar_expect_tx(&full[s], (uint32_t)(qn * 48));
    bulk_load_1d(stage + (size_t)s * kBulkQ * 3, v + 3 * qa, (uint32_t)(qn * 48), &full[s]);
  };
  if (tid == 0) {
    for (int s = 0; s < kBulkStages; ++s) {
      mbar_init(&full[s], 1);
#if PCT_BULK_LASTWARP
      reinterpret_cast<unsigned *>(empty)[s] = 0u;
#else
      mbar_init(&empty[s], kHistNT / 32);
#endif
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int64_t i = 0; i < kBulkStages && i < nst; ++i) issue(i);
  }
  for (int b = tid; b < nb; b += kHistNT) h[b] = SCATTER ? offs[b] + mine[b] : 0u;
  if (SCATTER)
    for (int k = tid; k < a.S; k += kHistNT) hsm[k] = a.derive ? plane_height(a, k) : a.heights[k];
  __syncthreads();
  const double *hts = hsm;
  for (int64_t i = 0; i < nst; ++i) {
    const int s = (int)(i % kBulkStages);
    const uint32_t ph = (uint32_t)((i / kBulkStages) & 1);
    mbar_wait(&full[s], ph);
    const int64_t qn = q1 - (q0 + i * kBulkQ);
    {  // every lane calls (warp-wide cursor aggregation); lanes past the
       // stage's end read a stale (valid) slot and pass valid = false
      const float4 *sq = stage + (size_t)s * kBulkQ * 3 + 3 * tid;
      hist_quad<SCATTER>(sq[0], sq[1], sq[2], tid < qn, a, hts, nbx, h, recs, outside);
    }
    __syncwarp();
#if PCT_BULK_LASTWARP
    // the last warp done with the stage refills it (no thread waits for the
    // others: warp 0 is not held back behind the slowest warp every stage)
    if ((tid & 31) == 0) {
      unsigned *done = reinterpret_cast<unsigned *>(empty) + s;
      __threadfence_block();
      if (atomicAdd(done, 1u) == kHistNT / 32 - 1) {
        *done = 0u;  // next used after this refill lands
        __threadfence_block();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (i + kBulkStages < nst) issue(i + kBulkStages);
      }
    }
#else
    if ((tid & 31) == 0) mbar_arrive(&empty[s]);
    if (tid == 0 && i + kBulkStages < nst) {
      mbar_wait(&empty[s], ph);
      issue(i + kBulkStages);
    }
#endif
  }
  for (int64_t p = (q1 << 2) + tid; p < p1; p += kHistNT) {  // the tail (< 4 points)
    const float4 A = make_float4(xyz[3 * p], xyz[3 * p + 1], xyz[3 * p + 2], 0.f);
    int fi, fj, bin = 0;
    if (point_cell_bin<SCATTER>((double)A.x, (double)A.y, (double)A.z, a, hts, fi, fj, bin)) {
      const int b = (fi / kHBH) * nbx + fj / kHBW;
      if (SCATTER) {
        const unsigned pos = atomicAdd(&h[b], 1u);
        recs[pos] = ((unsigned long long)f32_key(A.z) << 32) | ((unsigned long long)bin << 9) |
                    (unsigned)((fi % kHBH) * kHBW + fj % kHBW);
      } else {
        atomicAdd(&h[b], 1u);
      }
    } else if (!SCATTER && outside) {
      atomicAdd(outside, 1ull);
    }
  }
  if (!SCATTER) {
    __syncthreads();
    for (int b = tid; b < nb; b += kHistNT) mine[b] = h[b];
  }
}
// shared memory of hist_pass_bulk_kernel (0 if it does not fit one CTA)
inline size_t hist_bulk_smem(int nb, int S, bool scatter) {
  const size_t hist_b = ((size_t)nb * 4 + 127) & ~(size_t)127;
  if (S > kMaxStagedHeights) return 0;
  const size_t hts_b = scatter ? (((size_t)S * 8 + 127) & ~(size_t)127) : 0;
  const size_t tot = hist_b + hts_b + (size_t)kBulkStages * kBulkBytes + 2 * kBulkStages * 8;
  return tot <= 226 * 1024 ? tot : 0;
}

// per bucket: column prefix over the CTAs (in place) and the bucket total.
// A block takes 64 buckets x 4 segments of the G CTA rows: each thread sums
// its segment (independent loads), the segment sums are exchanged in shared
// memory, then each thread rewrites its segment from its base (the rows are
// still in L2).
constexpr int kColSeg = 4, kColB = 64;
__global__ void __launch_bounds__(kColSeg * kColB) hist_colscan_kernel(unsigned *__restrict__ cnt,
                                                                      int G, int nb,
                                                                      unsigned *__restrict__ tot) {
  __shared__ unsigned part[kColSeg][kColB];
  const int x = threadIdx.x % kColB, sg = threadIdx.x / kColB;
  const int b = blockIdx.x * kColB + x;
  const int c0 = G * sg / kColSeg, c1 = G * (sg + 1) / kColSeg;
  constexpr int U = 8;  // independent loads in flight
  unsigned sum = 0;
  if (b < nb) {
    int c = c0;
    for (; c + U <= c1; c += U) {
      unsigned v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = cnt[(int64_t)(c + u) * nb + b];
#pragma unroll
      for (int u = 0; u < U; ++u) sum += v[u];
    }
    for (; c < c1; ++c) sum += cnt[(int64_t)c * nb + b];
  }
  part[sg][x] = sum;
  __syncthreads();
  if (b >= nb) return;
  unsigned run = 0;
  for (int k = 0; k < sg; ++k) run += part[k][x];
  if (sg == kColSeg - 1) tot[b] = run + sum;
  int c = c0;
  for (; c + U <= c1; c += U) {
    unsigned v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = cnt[(int64_t)(c + u) * nb + b];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      cnt[(int64_t)(c + u) * nb + b] = run;
      run += v[u];
    }
  }
  for (; c < c1; ++c) {
    const unsigned v = cnt[(int64_t)c * nb + b];
    cnt[(int64_t)c * nb + b] = run;
    run += v;
  }
}

// TMA bulk tensor store of a [S][kHBH][kHBW] float box from shared memory
__device__ __forceinline__ void bulk_store_box(const CUtensorMap *map, const void *src, int x, int y) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(src);
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(map),
      "r"(x), "r"(y), "r"(0), "r"(sa)
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// One slice of a reduce scan: v beats the running key (max for ground, min
// for ceiling) -> take it, its decoded float bits (shift + one LOP3) and
// the slice's change bit, all under one predicate.
template <bool MAX>
__device__ __forceinline__ void scan_update(uint32_t v, uint32_t &run, uint32_t &o, uint32_t &m,
                                            uint32_t bit) {
  if (MAX)
    asm("{\n\t.reg .pred p;\n\t.reg .b32 s;\n\t"
        "setp.gt.u32 p, %3, %0;\n\t"
        "shr.s32 s, %3, 31;\n\t"
        "@p mov.b32 %0, %3;\n\t"
        "@p lop3.b32 %1, %3, s, 0x80000000, 0x4B;\n\t"
        "@p or.b32 %2, %2, %4;\n\t}"
        : "+r"(run), "+r"(o), "+r"(m)
        : "r"(v), "r"(bit));
  else
    asm("{\n\t.reg .pred p;\n\t.reg .b32 s;\n\t"
        "setp.lt.u32 p, %3, %0;\n\t"
        "shr.s32 s, %3, 31;\n\t"
        "@p mov.b32 %0, %3;\n\t"
        "@p lop3.b32 %1, %3, s, 0x80000000, 0x4B;\n\t"
        "@p or.b32 %2, %2, %4;\n\t}"
        : "+r"(run), "+r"(o), "+r"(m)
        : "r"(v), "r"(bit));
}

// streaming store, then step the pointer by a run-time stride (kept as one
// 64-bit add per slice)
__device__ __forceinline__ void store_step(float *&out, uint32_t o, int64_t step) {
  asm volatile("st.global.cs.b32 [%0], %1;" ::"l"(out), "r"(o) : "memory");
  asm("add.s64 %0, %0, %1;" : "+l"(out) : "l"(step));
}

template <bool TMA>
__global__ void __launch_bounds__(kHB2) hist_reduce_kernel(
    const unsigned long long *__restrict__ recs, const unsigned *__restrict__ offs, int nbx,
    int rows, int cols, int S, int64_t out_stride, float *__restrict__ ground,
    float *__restrict__ ceiling, unsigned long long *__restrict__ masks, float *sink, int ahead,
    const __grid_constant__ CUtensorMap gmap, const __grid_constant__ CUtensorMap cmap) {
  // [S][512] max keys, then min keys; with TMA the decoded layers are written
  // back in place ([S][16][32] floats = one box) and leave by bulk stores
  extern __shared__ __align__(128) uint32_t hk[];
  const int b = blockIdx.x, t = threadIdx.x;
  const unsigned r0 = offs[b], r1 = offs[b + 1];
  // records DRAM -> L2 ahead of use: the first `ahead` CTAs fetch their own
  // bucket, every CTA the bucket `ahead` places on (about one wave of
  // resident CTAs later), so a CTA's first pass finds its records in L2
  auto prefetch = [&](unsigned q0, unsigned q1) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(recs + q0) & ~(uintptr_t)15;
    const uintptr_t a1 = (reinterpret_cast<uintptr_t>(recs + q1) + 15) & ~(uintptr_t)15;
    for (uintptr_t q = a0; q < a1; q += 65536) {
      const unsigned nbytes = (unsigned)(a1 - q < 65536 ? a1 - q : 65536);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(q), "r"(nbytes) : "memory");
    }
  };
  if (t == 0) {
    if (b < ahead && r1 > r0) prefetch(r0, r1);
    if (b + ahead < (int)gridDim.x) {
      const unsigned f0 = offs[b + ahead], f1 = offs[b + ahead + 1];
      if (f1 > f0) prefetch(f0, f1);
    }
  }
  const int bi = b / nbx, bj = b - bi * nbx;
  const int i = bi * kHBH + t / kHBW, j = bj * kHBW + t % kHBW;
  const bool live = i < rows && j < cols;
  const int64_t cell = (int64_t)i * cols + j;
  // The low 32 bits of a record are bin * 512 + cell-in-bucket, the key
  // slot itself; records outside the stack's bins go to a per-thread dummy
  // word past the keys (no branch around the atomic).
  const uint32_t lim = (uint32_t)S * kHB2, dummy = lim + (uint32_t)t;
  // ground: max key per (bin, cell), bins 0 .. S-1 (16-byte stores)
  uint4 *hk4 = reinterpret_cast<uint4 *>(hk);
  for (int q = t; q < S * (kHB2 / 4); q += kHB2)
    hk4[q] = make_uint4(kKeyEmptyMax, kKeyEmptyMax, kKeyEmptyMax, kKeyEmptyMax);
  __syncthreads();
  auto gmax = [&](unsigned long long rec) {
    const uint32_t lo = (uint32_t)rec;
    atomicMax(hk + (lo < lim ? lo : dummy), (uint32_t)(rec >> 32));
  };
  auto cmin = [&](unsigned long long rec) {  // bins 1 .. S stored at bin - 1
    const uint32_t lo = (uint32_t)rec - (uint32_t)kHB2;
    atomicMin(hk + (lo < lim ? lo : dummy), (uint32_t)(rec >> 32));
  };
  // The first kKeep records of each thread stay in registers from the ground
  // pass to the ceiling pass (all their loads issued at once; buckets of up
  // to kKeep x 512 records are read once); the rest, if any, stream from
  // memory in both passes.  An absent record is all ones: both atomics then
  // land on the dummy word.
  constexpr int kKeep = 16;
  unsigned long long keep[kKeep];
#pragma unroll
  for (int u = 0; u < kKeep; ++u) {
    const unsigned idx = r0 + t + u * kHB2;
    keep[u] = idx < r1 ? __ldg(recs + idx) : ~0ull;
  }
#pragma unroll
  for (int u = 0; u < kKeep; ++u) gmax(keep[u]);
  constexpr int U = 8;  // records in flight per thread (beyond the kept ones)
  const unsigned rs = r0 + t + kKeep * kHB2;
  unsigned r = rs;
  for (; r + (U - 1) * kHB2 < r1; r += U * kHB2) {
    unsigned long long v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(recs + r + u * kHB2);  // kept in L2: read again
#pragma unroll
    for (int u = 0; u < U; ++u) gmax(v[u]);
  }
  for (; r < r1; r += kHB2) gmax(__ldg(recs + r));
  __syncthreads();
  // Scans: the running max (min) and its decoded float change only where a
  // slice's key beats it, so the decode and the slice-change bit sit under
  // that one predicate; the 64-bit mask is kept as two 32-bit words.
  const uint32_t *col = hk + t;
  {
    // slice-change mask: bit k set when the running max (and so the decoded
    // layer, a bijection of it) grows at slice k; bit 0 always
    uint32_t run = col[0];
    uint32_t o = run == kKeyEmptyMax ? kNaNBits : f32_bits(key_f32(run));
    uint32_t mw[2] = {1u, 0u};
    // cells outside the map store into one scratch word instead (no predicate)
    float *out = live ? ground + cell : sink;
    const int64_t step_b = live ? out_stride * 4 : 0;
    // (plain stores: each slot this thread read is reset to the ceiling
    // pass's empty key on the way, in place of an init pass and a barrier)
    auto step = [&](int k, uint32_t bit, uint32_t &m) {
      scan_update<true>(col[k * kHB2], run, o, m, bit);
      if (TMA) {
        hk[k * kHB2 + t] = o;
      } else {
        hk[k * kHB2 + t] = kKeyEmptyMin;
        store_step(out, o, step_b);
      }
    };
    if (TMA) {
      hk[t] = o;
    } else {
      hk[t] = kKeyEmptyMin;
      store_step(out, o, step_b);
    }
    const int k1 = S < 32 ? S : 32;
    uint32_t bit = 2u;
#pragma unroll 4
    for (int k = 1; k < k1; ++k, bit <<= 1) step(k, bit, mw[0]);
    bit = 1u;
#pragma unroll 4
    for (int k = 32; k < S; ++k, bit <<= 1) step(k, bit, mw[1]);
    if (masks && live) masks[(int64_t)i * cols + j] = (unsigned long long)mw[1] << 32 | mw[0];
  }
  if (TMA) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (t == 0) {
      bulk_store_box(&gmap, hk, bj * kHBW, bi * kHBH);
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // hk free again
    }
  }
  __syncthreads();
  // ceiling: min key per (bin, cell), bins 1 .. S stored at bin - 1
  if (TMA) {  // (the plain-store scan has reset the keys already)
    for (int q = t; q < S * (kHB2 / 4); q += kHB2)
      hk4[q] = make_uint4(kKeyEmptyMin, kKeyEmptyMin, kKeyEmptyMin, kKeyEmptyMin);
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < kKeep; ++u) cmin(keep[u]);
  r = rs;
  for (; r + (U - 1) * kHB2 < r1; r += U * kHB2) {
    unsigned long long v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(recs + r + u * kHB2);
#pragma unroll
    for (int u = 0; u < U; ++u) cmin(v[u]);
  }
  for (; r < r1; r += kHB2) cmin(__ldcs(recs + r));
  __syncthreads();
  {
    // bit k+1 set when the running min (walking down) shrinks at slice k:
    // ceiling[k] differs from ceiling[k+1]
    uint32_t run = col[(S - 1) * kHB2];
    uint32_t o = run == kKeyEmptyMin ? kNaNBits : f32_bits(key_f32(run));
    uint32_t mw[2] = {1u, 0u};
    float *out = live ? ceiling + cell + (int64_t)(S - 1) * out_stride : sink;
    const int64_t step_b = live ? -out_stride * 4 : 0;
    auto step = [&](int k, uint32_t bit, uint32_t &m) {
      scan_update<false>(col[k * kHB2], run, o, m, bit);
      if (TMA) hk[k * kHB2 + t] = o;
      else store_step(out, o, step_b);
    };
    if (TMA) hk[(S - 1) * kHB2 + t] = o;
    else store_step(out, o, step_b);
    // slices S-2 .. 31 set bits S-1 .. 32 (word 1), slices 30 .. 0 bits 31 .. 1
    int k = S - 2;
    uint32_t bit = (S >= 33 && S <= 64) ? 1u << (S - 33) : 0u;
#pragma unroll 4
    for (; k >= 31; --k, bit >>= 1) step(k, bit, mw[1]);
    bit = 1u << (k + 1 < 31 ? k + 1 : 31);
#pragma unroll 4
    for (; k >= 0; --k, bit >>= 1) step(k, bit, mw[0]);
    if (masks && live) masks[(int64_t)rows * cols + (int64_t)i * cols + j] = (unsigned long long)mw[1] << 32 | mw[0];
  }
  if (TMA) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (t == 0) {
      bulk_store_box(&cmap, hk, bj * kHBW, bi * kHBH);
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // before the CTA leaves
    }
  }
}

// Per-cell slice scans of the reduce (plain stores): ground walks up with the
// running max key, ceiling walks down with the running min key; `col` is
// the cell's key column ([S] keys kHB2 apart).  Returns the slice-change
// mask (bits as hist_reduce_kernel's).
__device__ __forceinline__ unsigned long long scan_ground_col(const uint32_t *col, int S,
                                                              float *out, int64_t step_b) {
  uint32_t run = col[0];
  uint32_t o = run == kKeyEmptyMax ? kNaNBits : key_bits(run);
  uint32_t mw0 = 1u, mw1 = 0u;
  store_step(out, o, step_b);
  const int k1 = S < 32 ? S : 32;
  uint32_t bit = 2u;
#pragma unroll 4
  for (int k = 1; k < k1; ++k, bit <<= 1) {
    scan_update<true>(col[k * kHB2], run, o, mw0, bit);
    store_step(out, o, step_b);
  }
  bit = 1u;
#pragma unroll 4
  for (int k = 32; k < S; ++k, bit <<= 1) {
    scan_update<true>(col[k * kHB2], run, o, mw1, bit);
    store_step(out, o, step_b);
  }
  return (unsigned long long)mw1 << 32 | mw0;
}
__device__ __forceinline__ unsigned long long scan_ceiling_col(const uint32_t *col, int S,
                                                               float *out, int64_t step_b) {
  uint32_t run = col[(S - 1) * kHB2];
  uint32_t o = run == kKeyEmptyMin ? kNaNBits : key_bits(run);
  uint32_t mw0 = 1u, mw1 = 0u;
  store_step(out, o, step_b);
  int k = S - 2;
  uint32_t bit = (S >= 33 && S <= 64) ? 1u << (S - 33) : 0u;
#pragma unroll 4
  for (; k >= 31; --k, bit >>= 1) {
    scan_update<false>(col[k * kHB2], run, o, mw1, bit);
    store_step(out, o, step_b);
  }
  bit = 1u << (k + 1 < 31 ? k + 1 : 31);
#pragma unroll 4
  for (; k >= 0; --k, bit >>= 1) {
    scan_update<false>(col[k * kHB2], run, o, mw0, bit);
    store_step(out, o, step_b);
  }
  return (unsigned long long)mw1 << 32 | mw0;
}

// H4, one pass: 1024 threads, both key planes in shared memory ([S][512]
// max keys, [S][512] min keys, 1024 dummy words: 2 x S x 2 KB + 4 KB), each
// record read once for both atomics; then threads 0-511 scan the ground
// columns and 512-1023 the ceiling columns at the same time.  One CTA per SM.
__global__ void __launch_bounds__(2 * kHB2, 1) hist_reduce_both_kernel(
    const unsigned long long *__restrict__ recs, const unsigned *__restrict__ offs, int nbx,
    int rows, int cols, int S, int64_t out_stride, float *__restrict__ ground,
    float *__restrict__ ceiling, unsigned long long *__restrict__ masks, float *sink) {
  extern __shared__ __align__(128) uint32_t hk[];
  const int b = blockIdx.x, t = threadIdx.x;
  const unsigned r0 = offs[b], r1 = offs[b + 1];
  if (t == 0 && r1 > r0) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(recs + r0) & ~(uintptr_t)15;
    const uintptr_t a1 = (reinterpret_cast<uintptr_t>(recs + r1) + 15) & ~(uintptr_t)15;
    for (uintptr_t q = a0; q < a1; q += 65536) {
      const unsigned nbytes = (unsigned)(a1 - q < 65536 ? a1 - q : 65536);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(q), "r"(nbytes) : "memory");
    }
  }
  const uint32_t lim = (uint32_t)S * kHB2, dummy = 2 * lim + (uint32_t)t;
  uint4 *hk4 = reinterpret_cast<uint4 *>(hk);
  const int nq = S * (kHB2 / 4);
  for (int q = t; q < 2 * nq; q += 2 * kHB2) {
    const uint32_t e = q < nq ? kKeyEmptyMax : kKeyEmptyMin;
    hk4[q] = make_uint4(e, e, e, e);
  }
  __syncthreads();
  auto both = [&](unsigned long long rec) {
    const uint32_t lo = (uint32_t)rec, key = (uint32_t)(rec >> 32);
    const uint32_t lc = lo - (uint32_t)kHB2;  // ceiling: bins 1 .. S at bin - 1
    atomicMax(hk + (lo < lim ? lo : dummy), key);
    atomicMin(hk + (lc < lim ? lim + lc : dummy), key);
  };
  constexpr int U = 8;
  unsigned r = r0 + t;
  for (; r + (U - 1) * 2 * kHB2 < r1; r += U * 2 * kHB2) {
    unsigned long long v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(recs + r + u * 2 * kHB2);
#pragma unroll
    for (int u = 0; u < U; ++u) both(v[u]);
  }
  for (; r < r1; r += 2 * kHB2) both(__ldcs(recs + r));
  __syncthreads();
  const int side = t / kHB2, c = t - side * kHB2;  // warp-uniform side
  const int bi = b / nbx, bj = b - bi * nbx;
  const int i = bi * kHBH + c / kHBW, j = bj * kHBW + c % kHBW;
  const bool live = i < rows && j < cols;
  const int64_t cell = (int64_t)i * cols + j;
  unsigned long long m;
  if (side == 0) {
    m = scan_ground_col(hk + c, S, live ? ground + cell : sink, live ? out_stride * 4 : 0);
  } else {
    m = scan_ceiling_col(hk + lim + c, S,
                         live ? ceiling + cell + (int64_t)(S - 1) * out_stride : sink,
                         live ? -out_stride * 4 : 0);
  }
  if (masks && live) masks[(int64_t)side * rows * cols + cell] = m;
}

// H4, split scan: the same reduction, with the per-cell slice scans shared by
// all 512 threads: thread t takes 4 adjacent cells (one 16-byte vector of
// keys per slice) and a quarter of the slices; each quarter first reduces its
// slices, the quarters exchange their maxima (minima) through shared memory,
// then scan their own slices from the incoming running value.  3x fewer
// instructions than one thread walking all slices of one cell.
__global__ void __launch_bounds__(kHB2) hist_reduce_split_kernel(
    const unsigned long long *__restrict__ recs, const unsigned *__restrict__ offs, int nbx,
    int rows, int cols, int S, int64_t out_stride, float *__restrict__ ground,
    float *__restrict__ ceiling, unsigned long long *__restrict__ masks) {
  extern __shared__ __align__(128) uint32_t hk[];     // [S][512] keys
  uint4 *xfer = reinterpret_cast<uint4 *>(hk + (size_t)S * kHB2);            // [4][128]
  unsigned long long *msk = reinterpret_cast<unsigned long long *>(xfer + 4 * 128);  // [2][512]
  const int b = blockIdx.x, t = threadIdx.x;
  const unsigned r0 = offs[b], r1 = offs[b + 1];
  if (t == 0 && r1 > r0) {  // the bucket's records DRAM -> L2 while the keys are initialised
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(recs + r0) & ~(uintptr_t)15;
    const uintptr_t a1 = (reinterpret_cast<uintptr_t>(recs + r1) + 15) & ~(uintptr_t)15;
    for (uintptr_t q = a0; q < a1; q += 65536) {
      const unsigned nbytes = (unsigned)(a1 - q < 65536 ? a1 - q : 65536);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(q), "r"(nbytes) : "memory");
    }
  }
  const int bi = b / nbx, bj = b - bi * nbx;
  // scan roles: quad q of 4 adjacent cells, slice quarter g
  const int q = t & 127, g = t >> 7;
  const int qi = bi * kHBH + (4 * q) / kHBW, qj = bj * kHBW + (4 * q) % kHBW;
  const int kb = S * g / 4, ke = S * (g + 1) / 4;
  const bool row_ok = qi < rows;
  const bool vec = (cols & 3) == 0 && (out_stride & 3) == 0 && qj + 3 < cols;
  uint4 *hk4 = reinterpret_cast<uint4 *>(hk);
  auto init = [&](uint32_t v) {
    for (int x = t; x < S * (kHB2 / 4); x += kHB2) hk4[x] = make_uint4(v, v, v, v);
  };
  auto put = [&](float *layer, int k, const float (&o)[4]) {
    if (!row_ok) return;
    float *p = layer + (int64_t)k * out_stride + (int64_t)qi * cols + qj;
    if (vec) {
      __stcs(reinterpret_cast<float4 *>(p), make_float4(o[0], o[1], o[2], o[3]));
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (qj + c < cols) __stcs(p + c, o[c]);
    }
  };
  constexpr int U = 4;  // records in flight per thread
  // ---- ground: max key per (bin, cell), bins 0 .. S-1
  init(kKeyEmptyMax);
  msk[t] = 0ull;
  msk[kHB2 + t] = 0ull;
  __syncthreads();
  {
    unsigned r = r0 + t;
    for (; r + (U - 1) * kHB2 < r1; r += U * kHB2) {
      unsigned long long v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldg(recs + r + u * kHB2);  // kept in L2: read again
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int bin = (int)((v[u] >> 9) & 0x7FFFFFu);
        if (bin < S) atomicMax(hk + bin * kHB2 + (unsigned)(v[u] & 511u), (uint32_t)(v[u] >> 32));
      }
    }
    for (; r < r1; r += kHB2) {
      const unsigned long long rec = __ldg(recs + r);
      const int bin = (int)((rec >> 9) & 0x7FFFFFu);
      if (bin < S) atomicMax(hk + bin * kHB2 + (unsigned)(rec & 511u), (uint32_t)(rec >> 32));
    }
  }
  __syncthreads();
  {
    uint4 lm = make_uint4(kKeyEmptyMax, kKeyEmptyMax, kKeyEmptyMax, kKeyEmptyMax);
    for (int k = kb; k < ke; ++k) {
      const uint4 v = hk4[k * (kHB2 / 4) + q];
      lm.x = max(lm.x, v.x); lm.y = max(lm.y, v.y); lm.z = max(lm.z, v.z); lm.w = max(lm.w, v.w);
    }
    xfer[g * 128 + q] = lm;
    __syncthreads();
    uint32_t run[4] = {kKeyEmptyMax, kKeyEmptyMax, kKeyEmptyMax, kKeyEmptyMax};
    for (int h = 0; h < g; ++h) {  // running max entering this quarter
      const uint4 x = xfer[h * 128 + q];
      run[0] = max(run[0], x.x); run[1] = max(run[1], x.y);
      run[2] = max(run[2], x.z); run[3] = max(run[3], x.w);
    }
    unsigned long long m[4] = {0ull, 0ull, 0ull, 0ull};
    if (g == 0) m[0] = m[1] = m[2] = m[3] = 1ull;  // bit 0 always
    for (int k = kb; k < ke; ++k) {
      const uint4 v4 = hk4[k * (kHB2 / 4) + q];
      const uint32_t v[4] = {v4.x, v4.y, v4.z, v4.w};
      float o[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (v[c] > run[c]) {
          run[c] = v[c];
          m[c] |= 1ull << (k & 63);
        }
        o[c] = decode_ground(run[c]);
      }
      put(ground, k, o);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (m[c]) atomicOr(&msk[4 * q + c], m[c]);
  }
  __syncthreads();
  // ---- ceiling: min key per (bin, cell), bins 1 .. S stored at bin - 1
  init(kKeyEmptyMin);
  __syncthreads();
  {
    unsigned r = r0 + t;
    for (; r + (U - 1) * kHB2 < r1; r += U * kHB2) {
      unsigned long long v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldcs(recs + r + u * kHB2);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int bin = (int)((v[u] >> 9) & 0x7FFFFFu);
        if (bin > 0)
          atomicMin(hk + (bin - 1) * kHB2 + (unsigned)(v[u] & 511u), (uint32_t)(v[u] >> 32));
      }
    }
    for (; r < r1; r += kHB2) {
      const unsigned long long rec = __ldcs(recs + r);
      const int bin = (int)((rec >> 9) & 0x7FFFFFu);
      if (bin > 0) atomicMin(hk + (bin - 1) * kHB2 + (unsigned)(rec & 511u), (uint32_t)(rec >> 32));
    }
  }
  __syncthreads();
  {
    uint4 lm = make_uint4(kKeyEmptyMin, kKeyEmptyMin, kKeyEmptyMin, kKeyEmptyMin);
    for (int k = kb; k < ke; ++k) {
      const uint4 v = hk4[k * (kHB2 / 4) + q];
      lm.x = min(lm.x, v.x); lm.y = min(lm.y, v.y); lm.z = min(lm.z, v.z); lm.w = min(lm.w, v.w);
    }
    xfer[g * 128 + q] = lm;
    __syncthreads();
    uint32_t run[4] = {kKeyEmptyMin, kKeyEmptyMin, kKeyEmptyMin, kKeyEmptyMin};
    for (int h = g + 1; h < 4; ++h) {  // running min entering this quarter from above
      const uint4 x = xfer[h * 128 + q];
      run[0] = min(run[0], x.x); run[1] = min(run[1], x.y);
      run[2] = min(run[2], x.z); run[3] = min(run[3], x.w);
    }
    unsigned long long m[4] = {0ull, 0ull, 0ull, 0ull};
    for (int k = ke - 1; k >= kb; --k) {
      const uint4 v4 = hk4[k * (kHB2 / 4) + q];
      const uint32_t v[4] = {v4.x, v4.y, v4.z, v4.w};
      float o[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (v[c] < run[c]) {
          run[c] = v[c];
          if (k < S - 1) m[c] |= 1ull << ((k + 1) & 63);
        }
        o[c] = decode_ceiling(run[c]);
      }
      put(ceiling, k, o);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (m[c]) atomicOr(&msk[kHB2 + 4 * q + c], m[c]);
  }
  if (masks) {
    __syncthreads();
    const int i = bi * kHBH + t / kHBW, j = bj * kHBW + t % kHBW;
    if (i < rows && j < cols) {
      masks[(int64_t)i * cols + j] = msk[t];
      masks[(int64_t)rows * cols + (int64_t)i * cols + j] = msk[kHB2 + t] | 1ull;
    }
  }
}

// ------------------------------------------------------------- K3 bin scan
// ground[k] = max(bins 0..k), ceiling[k] = min(bins k+1..S); scratch bin
// plane k of ckey holds bin k+1.
__device__ __forceinline__ void scan_body(uint32_t *__restrict__ gkey, uint32_t *__restrict__ ckey,
                                          int64_t cells, int S, int64_t out_stride,
                                          float *__restrict__ ground, float *__restrict__ ceiling,
                                          bool ground_side,
                                          unsigned long long *__restrict__ masks = nullptr) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cells) return;
  // scratch planes are dense (stride cells); output slice k of the band lives
  // at k * out_stride (== cells for a whole grid, larger inside a halo'd band)
  // batches of 8 independent loads keep enough bytes in flight per thread;
  // blockIdx.y = 0 walks the ground planes up, = 1 the ceiling planes down
  // (two threads per cell double the loads in flight)
  constexpr int U = 8;
  uint32_t run = kKeyEmptyMax;
  int k = 0;
  // slice-change mask of the layer written (bit k: differs from slice k-1)
  unsigned long long m = 1ull;
  uint32_t prev = 0u;
  auto note = [&](int kk, float o, bool ascending) {
    if (ascending ? kk > 0 : kk < S - 1) {
      if (f32_bits(o) != prev) m |= 1ull << ((ascending ? kk : kk + 1) & 63);
    }
    prev = f32_bits(o);
  };
  if (ground_side) {
  for (; k + U <= S; k += U) {
    uint32_t v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(gkey + (int64_t)(k + u) * cells + c);
#pragma unroll
    for (int u = 0; u < U; ++u)  // reset the (few) non-empty keys for the next build
      if (v[u] != kKeyEmptyMax) gkey[(int64_t)(k + u) * cells + c] = kKeyEmptyMax;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      run = v[u] > run ? v[u] : run;
      const float o = decode_ground(run);
      note(k + u, o, true);
      __stcs(ground + (int64_t)(k + u) * out_stride + c, o);
    }
  }
  for (; k < S; ++k) {
    const uint32_t v = __ldcs(gkey + (int64_t)k * cells + c);
    if (v != kKeyEmptyMax) gkey[(int64_t)k * cells + c] = kKeyEmptyMax;
    run = v > run ? v : run;
    const float o = decode_ground(run);
    note(k, o, true);
    __stcs(ground + (int64_t)k * out_stride + c, o);
  }
  if (masks) masks[c] = m;
  return;
  }
  run = kKeyEmptyMin;
  k = S - 1;
  for (; k - U + 1 >= 0; k -= U) {
    uint32_t v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(ckey + (int64_t)(k - u) * cells + c);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (v[u] != kKeyEmptyMin) ckey[(int64_t)(k - u) * cells + c] = kKeyEmptyMin;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      run = v[u] < run ? v[u] : run;
      const float o = decode_ceiling(run);
      note(k - u, o, false);
      __stcs(ceiling + (int64_t)(k - u) * out_stride + c, o);
    }
  }
  for (; k >= 0; --k) {
    const uint32_t v = __ldcs(ckey + (int64_t)k * cells + c);
    if (v != kKeyEmptyMin) ckey[(int64_t)k * cells + c] = kKeyEmptyMin;
    run = v < run ? v : run;
    const float o = decode_ceiling(run);
    note(k, o, false);
    __stcs(ceiling + (int64_t)k * out_stride + c, o);
  }
  if (masks) masks[cells + c] = m;
}

__global__ void __launch_bounds__(256) scan_kernel(uint32_t *__restrict__ gkey,
                                                   uint32_t *__restrict__ ckey,
                                                   int64_t cells, int S, int64_t out_stride,
                                                   float *__restrict__ ground,
                                                   float *__restrict__ ceiling,
                                                   unsigned long long *__restrict__ masks) {
  scan_body(gkey, ckey, cells, S, out_stride, ground, ceiling, blockIdx.y == 0, masks);
}

// ------------------------------------------------ batched maps (config 4)
// One launch per stage for a whole batch of independent maps; blockIdx.y
// (bounds, scatter, scan: z) selects the map's descriptor.
struct BuildMap {
  const void *xyz;
  int64_t n;
  BinArgs a;  // a.heights: device, per map
  uint32_t *gkey, *ckey;
  float *ground, *ceiling;
  unsigned long long *bkeys;  // 7 bounds keys
};

template <typename T>
__global__ void __launch_bounds__(256) bounds_batch_kernel(const BuildMap *__restrict__ maps) {
  const BuildMap &m = maps[blockIdx.y];
  bounds_body(static_cast<const T *>(m.xyz), m.n, m.bkeys);
}

template <typename T>
__global__ void __launch_bounds__(256) scatter_batch_kernel(const BuildMap *__restrict__ maps,
                                                            unsigned long long *outside) {
  const BuildMap &m = maps[blockIdx.y];
  scatter_body(static_cast<const T *>(m.xyz), m.n, m.a, m.gkey, m.ckey, outside);
}

__global__ void __launch_bounds__(256) scan_batch_kernel(const BuildMap *__restrict__ maps) {
  const BuildMap &m = maps[blockIdx.z];
  scan_body(m.gkey, m.ckey, m.a.cells, m.a.S, m.a.cells, m.ground, m.ceiling, blockIdx.y == 0);
}

int grid_for(pct_ctx *ctx, int64_t work, int block, int per_sm = 8) {
  int64_t g = (work + block - 1) / block;
  int64_t cap = (int64_t)ctx->num_sms * per_sm;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

int launch_bounds(pct_ctx *ctx, const void *xyz, int64_t n, int dtype, double lo[3],
                  double hi[3]) {
  if (n <= 0) return fail(ctx, PCT_E_EMPTY, "zero valid points");
  unsigned long long *keys = static_cast<unsigned long long *>(ctx->dsmall);
  unsigned long long init[7] = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull, 0ull};
  unsigned long long *hk = static_cast<unsigned long long *>(ctx->hsmall);
  PCT_CUDA(ctx, upload_async(ctx, keys, init, sizeof(init)));
  if (dtype == PCT_F32) {  // float4 path when 16 B aligned, scalar otherwise
    bounds_kernel<float><<<grid_for(ctx, (n + 3) / 4, 256), 256, 0, ctx->stream>>>(
        static_cast<const float *>(xyz), n, keys);
  } else {
    bounds_kernel<double><<<grid_for(ctx, n, 256), 256, 0, ctx->stream>>>(
        static_cast<const double *>(xyz), n, keys);
  }
  if (int rc = check_launch(ctx, "bounds_kernel")) return rc;
  PCT_CUDA(ctx, readback_async(ctx, hk, keys, sizeof(init)));
  PCT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (hk[6]) return fail(ctx, PCT_E_NONFINITE, "point cloud contains non-finite coordinates");
  for (int c = 0; c < 3; ++c) {
    lo[c] = dkey_inv(hk[c]);
    hi[c] = dkey_inv(hk[3 + c]);
  }
  return PCT_OK;
}

int launch_bounds_spec(pct_ctx *ctx, const void *xyz, int64_t n, int dtype, double d_s,
                       double r_g, int64_t max_grid_side, double lo[3], double hi[3],
                       pct_frame *dev_frame, bool *scattered) {
  *scattered = false;
  if (n <= 0) return fail(ctx, PCT_E_EMPTY, "zero valid points");
  const char *bmode = getenv("PCT_BUILD");
  const char *sv = getenv("PCT_BUILD_SPEC");
  const bool spec = ctx->keys && ctx->keys_clean && !(sv && sv[0] == '0') &&
                    !(bmode && bmode[0] == 't');
  unsigned long long *keys = static_cast<unsigned long long *>(ctx->dsmall);
  SpecFrame *df = reinterpret_cast<SpecFrame *>(static_cast<char *>(ctx->dsmall) + 64);
  unsigned long long init[7] = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull, 0ull};
  char *hb = static_cast<char *>(ctx->hsmall);
  PCT_CUDA(ctx, upload_async(ctx, keys, init, sizeof(init)));
  if (dtype == PCT_F32)
    bounds_kernel<float><<<grid_for(ctx, (n + 3) / 4, 256), 256, 0, ctx->stream>>>(
        static_cast<const float *>(xyz), n, keys);
  else
    bounds_kernel<double><<<grid_for(ctx, n, 256), 256, 0, ctx->stream>>>(
        static_cast<const double *>(xyz), n, keys);
  if (int rc = check_launch(ctx, "bounds_kernel")) return rc;
  if (spec) {
    const int64_t half = (int64_t)(ctx->keys_bytes / 2) / 4;  // words per half
    // the atomic path's key-size limit (launch_build's big_keys), unless forced
    const double max_key = (bmode && bmode[0] == 'a') ? 1e300 : 1.5e9;
    spec_frame_kernel<<<1, 32, 0, ctx->stream>>>(keys, d_s, r_g, max_grid_side,
                                                 4.0 * (double)half, max_key, df);
    if (int rc = check_launch(ctx, "spec_frame_kernel")) return rc;
    // bounds + frame come back while the scatter runs: the host waits on an
    // event recorded before the scatter, not on the stream
    PCT_CUDA(ctx, readback_async(ctx, hb, keys, 64 + sizeof(SpecFrame)));
    if (!ctx->spec_ev) PCT_CUDA(ctx, cudaEventCreateWithFlags(&ctx->spec_ev, cudaEventDisableTiming));
    PCT_CUDA(ctx, cudaEventRecord(ctx->spec_ev, ctx->stream));
    uint32_t *kw = static_cast<uint32_t *>(ctx->keys);
    const size_t hs = (size_t)kSpecMaxS * sizeof(double);
    if (dtype == PCT_F32)
      spec_scatter_kernel<float><<<grid_for(ctx, n, 256, 16), 256, hs, ctx->stream>>>(
          static_cast<const float *>(xyz), n, df, kw, half);
    else
      spec_scatter_kernel<double><<<grid_for(ctx, n, 256, 16), 256, hs, ctx->stream>>>(
          static_cast<const double *>(xyz), n, df, kw, half);
    if (int rc = check_launch(ctx, "spec_scatter_kernel")) return rc;
    PCT_CUDA(ctx, cudaEventSynchronize(ctx->spec_ev));
  } else {
    PCT_CUDA(ctx, readback_async(ctx, hb, keys, 56));
    PCT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  }
  const unsigned long long *hk = reinterpret_cast<const unsigned long long *>(hb);
  if (spec) {
    const SpecFrame *hf = reinterpret_cast<const SpecFrame *>(hb + 64);
    if (hf->ok) {
      *scattered = true;
      ctx->keys_clean = false;  // until a scan of this frame consumes them
      dev_frame->rows = hf->a.rows;
      dev_frame->cols = hf->a.cols;
      dev_frame->n_slices = hf->a.S;
      dev_frame->origin_x = hf->a.x0;
      dev_frame->origin_y = hf->a.y0;
      dev_frame->z_min = hf->a.z0;
    }
  }
  if (hk[6]) return fail(ctx, PCT_E_NONFINITE, "point cloud contains non-finite coordinates");
  for (int c = 0; c < 3; ++c) {
    lo[c] = dkey_inv(hk[c]);
    hi[c] = dkey_inv(hk[3 + c]);
  }
  return PCT_OK;
}

// ------------------------------------------------ batched maps (host side)
// descriptors + per-map scratch live in the context buffers; the caller keeps
// the batch's inputs / outputs alive until the stream is synchronised
int launch_bounds_batch(pct_ctx *ctx, int n_maps, const void *const *xyz, const int64_t *n,
                        int dtype, unsigned long long *keys_host) {
  // keys (7 per map, padded to 8) in dsmall; descriptors in the scratch
  if ((size_t)n_maps * 64 > 65536) return fail(ctx, PCT_E_INVALID, "batch too large for bounds");
  std::vector<BuildMap> d(n_maps);
  unsigned long long *dk = static_cast<unsigned long long *>(ctx->dsmall);
  int64_t nmax = 1;
  for (int m = 0; m < n_maps; ++m) {
    d[m] = BuildMap{};
    d[m].xyz = xyz[m];
    d[m].n = n[m];
    d[m].bkeys = dk + 8 * (size_t)m;
    nmax = std::max<int64_t>(nmax, n[m]);
    const unsigned long long init[8] = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
    std::memcpy(keys_host + 8 * (size_t)m, init, sizeof(init));
  }
  if (int rc = ensure_scratch(ctx, sizeof(BuildMap) * (size_t)n_maps)) return rc;
  BuildMap *dd = static_cast<BuildMap *>(ctx->scratch);
  PCT_CUDA(ctx, upload_async(ctx, dd, d.data(), sizeof(BuildMap) * n_maps));
  PCT_CUDA(ctx, cudaMemcpyAsync(dk, keys_host, 64 * (size_t)n_maps, cudaMemcpyHostToDevice,
                                ctx->stream));
  const int per_map = std::max(1, std::min(grid_for(ctx, (nmax + 3) / 4, 256), 64));
  if (dtype == PCT_F32)
    bounds_batch_kernel<float><<<dim3(per_map, n_maps), 256, 0, ctx->stream>>>(dd);
  else
    bounds_batch_kernel<double><<<dim3(per_map, n_maps), 256, 0, ctx->stream>>>(dd);
  if (int rc = check_launch(ctx, "bounds_batch_kernel")) return rc;
  PCT_CUDA(ctx, cudaMemcpyAsync(keys_host, dk, 64 * (size_t)n_maps, cudaMemcpyDeviceToHost,
                                ctx->stream));
  return PCT_OK;
}

int launch_build_batch(pct_ctx *ctx, int n_maps, const void *const *xyz, const int64_t *n,
                       int dtype, const pct_frame *frames, const double *const *heights,
                       float *const *ground, float *const *ceiling) {
  // scratch: descriptors | heights (all maps) | outside counter
  int64_t key_words = 0, hcount = 0, nmax = 1;
  int smax = 1;
  uint64_t tag = 1469598103934665603ull;  // FNV-1a over the batch layout
  for (int m = 0; m < n_maps; ++m) {
    const int64_t cells = (int64_t)frames[m].rows * frames[m].cols;
    key_words += 2 * (int64_t)frames[m].n_slices * cells;
    hcount += frames[m].n_slices;
    nmax = std::max<int64_t>(nmax, n[m]);
    smax = std::max(smax, frames[m].n_slices);
    for (uint64_t v : {(uint64_t)frames[m].n_slices, (uint64_t)cells}) tag = (tag ^ v) * 1099511628211ull;
  }
  const size_t dbytes = ((sizeof(BuildMap) * (size_t)n_maps + 255) / 256) * 256;
  const size_t hbytes = (((size_t)hcount * 8 + 255) / 256) * 256;
  if (int rc = ensure_scratch(ctx, dbytes + hbytes + 256)) return rc;
  char *base = static_cast<char *>(ctx->scratch);
  BuildMap *dd = reinterpret_cast<BuildMap *>(base);
  double *hd = reinterpret_cast<double *>(base + dbytes);
  unsigned long long *outside = reinterpret_cast<unsigned long long *>(base + dbytes + hbytes);
  // keys of every map in the context's key buffer; the scans reset them, so
  // the same batch layout needs no memset next time
  const size_t kbytes = (size_t)key_words * 4;
  if (ctx->keys_bytes < kbytes) {
    if (ctx->keys) {
      cudaStreamSynchronize(ctx->stream);
      cudaFree(ctx->keys);
      ctx->keys = nullptr;
      ctx->keys_bytes = 0;
    }
    PCT_CUDA(ctx, cudaMalloc(&ctx->keys, kbytes));
    ctx->keys_bytes = kbytes;
    ctx->keys_tag[0] = -1;
    ctx->keys_clean = false;
  }
  std::vector<BuildMap> d(n_maps);
  std::vector<double> hh((size_t)hcount);
  int64_t koff = 0, hoff = 0;
  uint32_t *kb = static_cast<uint32_t *>(ctx->keys);
  for (int m = 0; m < n_maps; ++m) {
    const pct_frame &fr = frames[m];
    const int64_t cells = (int64_t)fr.rows * fr.cols;
    std::memcpy(hh.data() + hoff, heights[m], sizeof(double) * fr.n_slices);
    d[m] = BuildMap{};
    d[m].xyz = xyz[m];
    d[m].n = n[m];
    d[m].a = BinArgs{fr.origin_x, fr.origin_y, fr.z_min, fr.r_g, fr.d_s, 1.0 / fr.r_g,
                     1.0 / fr.d_s, hd + hoff, cells, fr.rows, fr.cols, fr.n_slices, 0};
    d[m].gkey = kb + koff;
    d[m].ckey = kb + koff + (int64_t)fr.n_slices * cells;
    d[m].ground = ground[m];
    d[m].ceiling = ceiling[m];
    koff += 2 * (int64_t)fr.n_slices * cells;
    hoff += fr.n_slices;
  }
  PCT_CUDA(ctx, upload_async(ctx, dd, d.data(), sizeof(BuildMap) * n_maps));
  PCT_CUDA(ctx, upload_async(ctx, hd, hh.data(), sizeof(double) * hcount));
  const int64_t tagi = (int64_t)(tag >> 1);
  if (ctx->keys_tag[0] != -2 || ctx->keys_tag[1] != tagi) {  // -2: a batch layout
    int64_t off = 0;
    for (int m = 0; m < n_maps; ++m) {  // gkey -> 0x00, ckey -> 0xFF per map
      const int64_t sc = (int64_t)frames[m].n_slices * frames[m].rows * frames[m].cols;
      PCT_CUDA(ctx, cudaMemsetAsync(kb + off, 0x00, sc * 4, ctx->stream));
      PCT_CUDA(ctx, cudaMemsetAsync(kb + off + sc, 0xFF, sc * 4, ctx->stream));
      off += 2 * sc;
    }
  }
  ctx->keys_tag[0] = -1;  // dirty until the scans are launched
  ctx->keys_clean = false;  // the single-map layout must be cleared again
  PCT_CUDA(ctx, cudaMemsetAsync(outside, 0, 8, ctx->stream));
  const size_t hsm = smax <= kMaxStagedHeights ? (size_t)smax * sizeof(double) : 0;
  const int gx = std::max(1, std::min(grid_for(ctx, nmax, 256, 16), 64));
  if (dtype == PCT_F32)
    scatter_batch_kernel<float><<<dim3(gx, n_maps), 256, hsm, ctx->stream>>>(dd, outside);
  else
    scatter_batch_kernel<double><<<dim3(gx, n_maps), 256, hsm, ctx->stream>>>(dd, outside);
  if (int rc = check_launch(ctx, "scatter_batch_kernel")) return rc;
  int64_t cmax = 1;
  for (int m = 0; m < n_maps; ++m) cmax = std::max<int64_t>(cmax, (int64_t)frames[m].rows * frames[m].cols);
  scan_batch_kernel<<<dim3((unsigned)((cmax + 255) / 256), 2, n_maps), 256, 0, ctx->stream>>>(dd);
  if (int rc = check_launch(ctx, "scan_batch_kernel")) return rc;
  ctx->keys_tag[0] = -2;
  ctx->keys_tag[1] = tagi;
  return PCT_OK;
}

// bounds without the host synchronisation: the 7 keys land in keys_host
// (pinned; decode with bounds_from_keys after the stream is synchronised)
int launch_bounds_async(pct_ctx *ctx, const void *xyz, int64_t n, int dtype,
                        unsigned long long *keys_host, const unsigned long long *init_host) {
  unsigned long long *keys = static_cast<unsigned long long *>(ctx->dsmall);
  PCT_CUDA(ctx, cudaMemcpyAsync(keys, init_host, 7 * sizeof(unsigned long long),
                                cudaMemcpyHostToDevice, ctx->stream));
  if (dtype == PCT_F32)
    bounds_kernel<float><<<grid_for(ctx, (n + 3) / 4, 256), 256, 0, ctx->stream>>>(
        static_cast<const float *>(xyz), n, keys);
  else
    bounds_kernel<double><<<grid_for(ctx, n, 256), 256, 0, ctx->stream>>>(
        static_cast<const double *>(xyz), n, keys);
  if (int rc = check_launch(ctx, "bounds_kernel")) return rc;
  PCT_CUDA(ctx, cudaMemcpyAsync(keys_host, keys, 7 * sizeof(unsigned long long),
                                cudaMemcpyDeviceToHost, ctx->stream));
  return PCT_OK;
}

bool bounds_from_keys(const unsigned long long *k, double lo[3], double hi[3]) {
  for (int c = 0; c < 3; ++c) {
    lo[c] = dkey_inv(k[c]);
    hi[c] = dkey_inv(k[3 + c]);
  }
  return k[6] == 0;  // no non-finite coordinate
}

int launch_build(pct_ctx *ctx, const void *xyz, int64_t n, int dtype, const pct_frame &fr,
                 const double *heights_host, float *ground, float *ceiling, int row0, int nrows,
                 int64_t out_stride, bool keys_scattered) {
  const int S = fr.n_slices;
  if (nrows < 0) {  // whole grid
    row0 = 0;
    nrows = fr.rows;
  }
  const int64_t cells = (int64_t)nrows * fr.cols;
  if (out_stride <= 0) out_stride = cells;
  const size_t plane = (size_t)cells * sizeof(uint32_t);
  // scratch: gkey (S planes) | ckey (S planes) | heights (S doubles) | outside counter
  const size_t hbytes = ((size_t)S * sizeof(double) + 255) & ~(size_t)255;
  const char *bmode = getenv("PCT_BUILD");
  // Atomic build while the key planes stay within reach of L2 / the TLB;
  // beyond ~1.5 GB of keys every RED becomes a DRAM read-modify-write of a
  // sector (cfg3, 5.6 GB of keys: atomic scatter 11.5 ms + scan 2.1 ms vs
  // tiled 7.0 ms; cfg1 141 vs 211 us and cfg2 ~660 vs 781 us the other way,
  // profiles/r01d_build_variants.txt).  PCT_BUILD=atomic / tiled forces one.
  const bool big_keys = 2.0 * (double)S * (double)cells * 4.0 > 1.5e9;
  // heights that follow the frame formula are derived in the kernels (no
  // upload); points outside a whole-grid frame cannot occur, so the
  // diagnostic outside-counter is only kept for bands
  bool derive = S <= kMaxStagedHeights;
  for (int k = 0; derive && k < S; ++k) {
    volatile double t = fr.d_s * ((double)k + 1.0);
    derive = heights_host[k] == fr.z_min + t;
  }
  const bool whole = row0 == 0 && nrows == fr.rows;
  const bool tiled = bmode ? (bmode[0] == 't' || bmode[0] == 'h') : big_keys;
  const int hbx = (fr.cols + kHBW - 1) / kHBW, hby = (nrows + kHBH - 1) / kHBH;
  const int64_t hnb = (int64_t)hbx * hby;
  if (tiled && !(bmode && bmode[0] == 't') && S <= kHistMaxS && hnb <= kHistMaxBuckets &&
      n > 0 && n < (int64_t)UINT32_MAX) {
    // histogram-partitioned build: scratch = heights | outside | cnt [G][nb] |
    // totals | offsets | block sums | records
    const int G = ctx->num_sms;
    const size_t cbytes = ((size_t)G * hnb * 4 + 255) & ~(size_t)255;
    const size_t tbytes = ((size_t)(hnb + 1) * 4 + 255) & ~(size_t)255;
    const size_t sbytes = ((size_t)((hnb + 1023) / 1024) * 4 + 255) & ~(size_t)255;
    if (int rc = ensure_scratch(ctx, hbytes + 256 + cbytes + 2 * tbytes + sbytes + (size_t)n * 8))
      return rc;
    char *b0 = static_cast<char *>(ctx->scratch);
    double *hd = reinterpret_cast<double *>(b0);
    unsigned long long *outs = reinterpret_cast<unsigned long long *>(b0 + hbytes);
    unsigned *cnt = reinterpret_cast<unsigned *>(b0 + hbytes + 256);
    unsigned *tot = reinterpret_cast<unsigned *>(b0 + hbytes + 256 + cbytes);
    unsigned *offs = reinterpret_cast<unsigned *>(b0 + hbytes + 256 + cbytes + tbytes);
    unsigned *bsum = reinterpret_cast<unsigned *>(b0 + hbytes + 256 + cbytes + 2 * tbytes);
    unsigned long long *recs = reinterpret_cast<unsigned long long *>(
        b0 + hbytes + 256 + cbytes + 2 * tbytes + sbytes);
    float *sink = reinterpret_cast<float *>(b0 + hbytes + 128);  // unused bytes of `outs`
    if (!derive) PCT_CUDA(ctx, upload_async(ctx, hd, heights_host, (size_t)S * sizeof(double)));
    if (whole) outs = nullptr;
    else PCT_CUDA(ctx, cudaMemsetAsync(outs, 0, 8, ctx->stream));
    BinArgs a{fr.origin_x, fr.origin_y, fr.z_min, fr.r_g, fr.d_s, 1.0 / fr.r_g, 1.0 / fr.d_s,
              hd, cells, nrows, fr.cols, S, row0, derive ? 1 : 0};
    const size_t hist = ((size_t)hnb * 4 + 15) & ~(size_t)15;
    const size_t hsm = hist + (S <= kMaxStagedHeights ? (size_t)S * sizeof(double) : 0);
    const int nbi = (int)hnb;
    // points staged through shared memory by bulk copies when the histogram
    // leaves room for the stages (PCT_HIST_BULK=0: direct loads)
    const char *hb = getenv("PCT_HIST_BULK");
    const bool bulk_ok = dtype == PCT_F32 && (reinterpret_cast<uintptr_t>(xyz) & 15) == 0 &&
                         !(hb && hb[0] == '0');
    const size_t bsm_c = bulk_ok ? hist_bulk_smem(nbi, S, false) : 0;
    const size_t bsm_s = bulk_ok ? hist_bulk_smem(nbi, S, true) : 0;
    if (bsm_c) {
      PCT_CUDA(ctx, cudaFuncSetAttribute(hist_pass_bulk_kernel<false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm_c));
      hist_pass_bulk_kernel<false><<<G, kHistNT, bsm_c, ctx->stream>>>(
          static_cast<const float *>(xyz), n, a, hbx, nbi, cnt, nullptr, nullptr, outs);
    } else if (dtype == PCT_F32) {
      PCT_CUDA(ctx, cudaFuncSetAttribute(hist_pass_kernel<float, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm));
      hist_pass_kernel<float, false><<<G, kHistNT, hist, ctx->stream>>>(
          static_cast<const float *>(xyz), n, a, hbx, nbi, cnt, nullptr, nullptr, outs);
    } else {
      PCT_CUDA(ctx, cudaFuncSetAttribute(hist_pass_kernel<double, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm));
      hist_pass_kernel<double, false><<<G, kHistNT, hist, ctx->stream>>>(
          static_cast<const double *>(xyz), n, a, hbx, nbi, cnt, nullptr, nullptr, outs);
    }
    if (int rc = check_launch(ctx, "hist_count_kernel")) return rc;
    hist_colscan_kernel<<<(unsigned)((hnb + kColB - 1) / kColB), kColSeg * kColB, 0, ctx->stream>>>(
        cnt, G, nbi, tot);
    if (int rc = check_launch(ctx, "hist_colscan_kernel")) return rc;
    const unsigned nsb = (unsigned)((hnb + 1023) / 1024);
    tile_sums_kernel<<<nsb, 1024, 0, ctx->stream>>>(tot, nbi, bsum, 1);
    if (int rc = check_launch(ctx, "tile_sums_kernel")) return rc;
    tile_offsets_kernel<<<nsb, 1024, 0, ctx->stream>>>(tot, nbi, bsum, offs, nullptr, 1);
    if (int rc = check_launch(ctx, "tile_offsets_kernel")) return rc;
    if (bsm_s) {
      PCT_CUDA(ctx, cudaFuncSetAttribute(hist_pass_bulk_kernel<true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm_s));
      hist_pass_bulk_kernel<true><<<G, kHistNT, bsm_s, ctx->stream>>>(
          static_cast<const float *>(xyz), n, a, hbx, nbi, cnt, offs, recs, outs);
    } else if (dtype == PCT_F32) {
      PCT_CUDA(ctx, cudaFuncSetAttribute(hist_pass_kernel<float, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm));
      hist_pass_kernel<float, true><<<G, kHistNT, hsm, ctx->stream>>>(
          static_cast<const float *>(xyz), n, a, hbx, nbi, cnt, offs, recs, outs);
    } else {
      PCT_CUDA(ctx, cudaFuncSetAttribute(hist_pass_kernel<double, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm));
      hist_pass_kernel<double, true><<<G, kHistNT, hsm, ctx->stream>>>(
          static_cast<const double *>(xyz), n, a, hbx, nbi, cnt, offs, recs, outs);
    }
    if (int rc = check_launch(ctx, "hist_scatter_kernel")) return rc;
    const size_t rsm = (size_t)S * kHB2 * 4;
    const size_t rsm1 = rsm + kHB2 * 4;  // + one dummy word per thread
    // records prefetched one wave of resident CTAs ahead (PCT_REDUCE_AHEAD)
    // (0: each CTA its own bucket; one wave ahead measured slower at cfg3,
    // 4.32 vs 4.22 ms build)
    int ahead = 0;
    if (const char *av = getenv("PCT_REDUCE_AHEAD")) ahead = atoi(av);
    unsigned long long *mk = (whole && S <= 64) ? ctx->build_masks : nullptr;
    // the layers leave by TMA bulk tensor stores when their rows are 16-byte
    // pitched (one [S][16][32] box per bucket and layer)
    CUtensorMap gmap, cmap;
    std::memset(&gmap, 0, sizeof(gmap));
    std::memset(&cmap, 0, sizeof(cmap));
    bool tma = false;
    {
      // measured slower at cfg3 (2.26 vs 2.09 ms: the CTA waits for the
      // bulk store's read of its keys before the ceiling pass): opt-in
      const char *tv = getenv("PCT_BUILD_TMA");
      static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
      if (!encode) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
                cudaSuccess && fn && q == cudaDriverEntryPointSuccess)
          encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        cudaGetLastError();
      }
      if (encode && (tv && tv[0] == '1') && (fr.cols & 3) == 0 && (out_stride & 3) == 0 &&
          S <= 256 && ((reinterpret_cast<uintptr_t>(ground) | reinterpret_cast<uintptr_t>(ceiling)) & 15) == 0) {
        const cuuint64_t dims[3] = {(cuuint64_t)fr.cols, (cuuint64_t)nrows, (cuuint64_t)S};
        const cuuint64_t str[2] = {(cuuint64_t)fr.cols * 4, (cuuint64_t)out_stride * 4};
        const cuuint32_t box[3] = {(cuuint32_t)kHBW, (cuuint32_t)kHBH, (cuuint32_t)S};
        const cuuint32_t estr[3] = {1, 1, 1};
        tma = encode(&gmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ground, dims, str, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
                  CUDA_SUCCESS &&
              encode(&cmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ceiling, dims, str, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
                  CUDA_SUCCESS;
      }
    }
    // the split-scan reduce measured slower at cfg3 (2.42 vs 2.18 ms):
    // opt-in (PCT_BUILD_REDUCE=2)
    const char *rv = getenv("PCT_BUILD_REDUCE");
    const size_t bsm = (size_t)2 * S * kHB2 * 4 + 2 * kHB2 * 4;
    if (!tma && rv && rv[0] == '3' && bsm <= 226 * 1024) {
      PCT_CUDA(ctx, cudaFuncSetAttribute(hist_reduce_both_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
      hist_reduce_both_kernel<<<(unsigned)hnb, 2 * kHB2, bsm, ctx->stream>>>(
          recs, offs, hbx, nrows, fr.cols, S, out_stride, ground, ceiling, mk, sink);
    } else if (!tma && rv && rv[0] == '2') {
      const size_t ssm = rsm + 4 * 128 * 16 + 2 * kHB2 * 8;
      PCT_CUDA(ctx, cudaFuncSetAttribute(hist_reduce_split_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
      hist_reduce_split_kernel<<<(unsigned)hnb, kHB2, ssm, ctx->stream>>>(
          recs, offs, hbx, nrows, fr.cols, S, out_stride, ground, ceiling, mk);
    } else if (tma) {
      PCT_CUDA(ctx, cudaFuncSetAttribute(hist_reduce_kernel<true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm1));
      hist_reduce_kernel<true><<<(unsigned)hnb, kHB2, rsm1, ctx->stream>>>(
          recs, offs, hbx, nrows, fr.cols, S, out_stride, ground, ceiling, mk, sink, ahead, gmap, cmap);
    } else {
      PCT_CUDA(ctx, cudaFuncSetAttribute(hist_reduce_kernel<false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm1));
      hist_reduce_kernel<false><<<(unsigned)hnb, kHB2, rsm1, ctx->stream>>>(
          recs, offs, hbx, nrows, fr.cols, S, out_stride, ground, ceiling, mk, sink, ahead, gmap, cmap);
    }
    if (mk) ctx->build_masks_written = true;
    return check_launch(ctx, "hist_reduce_kernel");
  }
  if (S <= kTileMaxS && n > 0 && n < (int64_t)UINT32_MAX && tiled) {
    // tile-partitioned build: scratch = heights | outside | counts | offsets |
    // cursors | records (the key planes above are not used)
    const int ntx = (fr.cols + kTBW - 1) / kTBW, nty = (nrows + kTBH - 1) / kTBH;
    const int64_t ntiles = (int64_t)ntx * nty;
    const size_t cbytes = ((size_t)(ntiles + 1) * 4 * kCtrPad + 255) & ~(size_t)255;
    const size_t sbytes = ((size_t)((ntiles + 1023) / 1024) * 4 + 255) & ~(size_t)255;
    if (int rc = ensure_scratch(ctx, hbytes + 256 + 3 * cbytes + sbytes + (size_t)n * 8)) return rc;
    char *b0 = static_cast<char *>(ctx->scratch);
    double *hd = reinterpret_cast<double *>(b0);
    unsigned long long *outs = reinterpret_cast<unsigned long long *>(b0 + hbytes);
    unsigned *cnt = reinterpret_cast<unsigned *>(b0 + hbytes + 256);
    unsigned *offs = reinterpret_cast<unsigned *>(b0 + hbytes + 256 + cbytes);
    unsigned *cur = reinterpret_cast<unsigned *>(b0 + hbytes + 256 + 2 * cbytes);
    unsigned *bsum = reinterpret_cast<unsigned *>(b0 + hbytes + 256 + 3 * cbytes);
    unsigned long long *recs =
        reinterpret_cast<unsigned long long *>(b0 + hbytes + 256 + 3 * cbytes + sbytes);
    if (!derive) PCT_CUDA(ctx, upload_async(ctx, hd, heights_host, (size_t)S * sizeof(double)));
    if (whole) outs = nullptr;
    else PCT_CUDA(ctx, cudaMemsetAsync(outs, 0, 8, ctx->stream));
    PCT_CUDA(ctx, cudaMemsetAsync(cnt, 0, (size_t)ntiles * 4 * kCtrPad, ctx->stream));
    BinArgs a{fr.origin_x, fr.origin_y, fr.z_min, fr.r_g, fr.d_s, 1.0 / fr.r_g, 1.0 / fr.d_s,
              hd, cells, nrows, fr.cols, S, row0, derive ? 1 : 0};
    const size_t hsm = S <= kMaxStagedHeights ? (size_t)S * sizeof(double) : 0;
    const int g = grid_for(ctx, n, 256, 16);
    if (dtype == PCT_F32)
      tile_pass_kernel<float, false><<<g, 256, hsm, ctx->stream>>>(
          static_cast<const float *>(xyz), n, a, ntx, cnt, nullptr, outs);
    else
      tile_pass_kernel<double, false><<<g, 256, hsm, ctx->stream>>>(
          static_cast<const double *>(xyz), n, a, ntx, cnt, nullptr, outs);
    if (int rc = check_launch(ctx, "tile_count_kernel")) return rc;
    const unsigned nb = (unsigned)((ntiles + 1023) / 1024);
    tile_sums_kernel<<<nb, 1024, 0, ctx->stream>>>(cnt, (int)ntiles, bsum, kCtrPad);
    if (int rc = check_launch(ctx, "tile_sums_kernel")) return rc;
    tile_offsets_kernel<<<nb, 1024, 0, ctx->stream>>>(cnt, (int)ntiles, bsum, offs, cur, kCtrPad);
    if (int rc = check_launch(ctx, "tile_offsets_kernel")) return rc;
    if (dtype == PCT_F32)
      tile_pass_kernel<float, true><<<g, 256, hsm, ctx->stream>>>(
          static_cast<const float *>(xyz), n, a, ntx, cur, recs, outs);
    else
      tile_pass_kernel<double, true><<<g, 256, hsm, ctx->stream>>>(
          static_cast<const double *>(xyz), n, a, ntx, cur, recs, outs);
    if (int rc = check_launch(ctx, "tile_scatter_kernel")) return rc;
    const size_t tsm = (size_t)2 * S * kTB2 * 4;
    PCT_CUDA(ctx, cudaFuncSetAttribute(tile_reduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)tsm));
    tile_reduce_kernel<<<(unsigned)ntiles, kTileNT, tsm, ctx->stream>>>(
        recs, offs, ntx, nrows, fr.cols, S, out_stride, ground, ceiling);
    return check_launch(ctx, "tile_reduce_kernel");
  }
  // key planes in their own grow-only buffer: ground keys in the first
  // half, ceiling keys in the second (fixed offsets, so any layout that fits
  // finds them empty: the scan leaves every key it reads empty again); a
  // memset only after growth or a batch build (another layout)
  if (keys_scattered && !(S <= kSpecMaxS && whole && derive && ctx->keys_bytes / 2 >= plane * S))
    return fail(ctx, PCT_E_INVALID, "speculative scatter does not match the frame");
  if (ctx->keys_bytes / 2 < plane * S) {
    if (ctx->keys) {
      cudaStreamSynchronize(ctx->stream);
      cudaFree(ctx->keys);
      ctx->keys = nullptr;
      ctx->keys_bytes = 0;
    }
    PCT_CUDA(ctx, cudaMalloc(&ctx->keys, 2 * plane * S));
    ctx->keys_bytes = 2 * plane * S;
    ctx->keys_clean = false;
  }
  if (int rc = ensure_scratch(ctx, hbytes + 256)) return rc;
  const size_t half = ctx->keys_bytes / 2;
  uint32_t *gkey = static_cast<uint32_t *>(ctx->keys);
  uint32_t *ckey = reinterpret_cast<uint32_t *>(static_cast<char *>(ctx->keys) + half);
  char *base = static_cast<char *>(ctx->scratch);
  double *hdev = reinterpret_cast<double *>(base);
  unsigned long long *outside = reinterpret_cast<unsigned long long *>(base + hbytes);
  if (!derive) PCT_CUDA(ctx, upload_async(ctx, hdev, heights_host, (size_t)S * sizeof(double)));
  if (!keys_scattered && !ctx->keys_clean) {
    PCT_CUDA(ctx, cudaMemsetAsync(gkey, 0x00, half, ctx->stream));
    PCT_CUDA(ctx, cudaMemsetAsync(ckey, 0xFF, half, ctx->stream));
  }
  ctx->keys_clean = false;  // until the scan below is launched
  ctx->keys_tag[0] = -3;    // single-map layout (the batch layout memsets again)
  if (whole) outside = nullptr;
  else PCT_CUDA(ctx, cudaMemsetAsync(outside, 0, 8, ctx->stream));
  BinArgs a{fr.origin_x, fr.origin_y, fr.z_min, fr.r_g, fr.d_s, 1.0 / fr.r_g, 1.0 / fr.d_s,
            hdev, cells, nrows, fr.cols, S, row0, derive ? 1 : 0};
  const size_t hsm_bytes = S <= kMaxStagedHeights ? (size_t)S * sizeof(double) : 0;
  if (n > 0 && !keys_scattered) {
    if (dtype == PCT_F32)
      scatter_kernel<float><<<grid_for(ctx, n, 256, 16), 256, hsm_bytes, ctx->stream>>>(
          static_cast<const float *>(xyz), n, a, gkey, ckey, outside);
    else
      scatter_kernel<double><<<grid_for(ctx, n, 256, 16), 256, hsm_bytes, ctx->stream>>>(
          static_cast<const double *>(xyz), n, a, gkey, ckey, outside);
    if (int rc = check_launch(ctx, "scatter_kernel")) return rc;
  }
  unsigned long long *mk = (whole && S <= 64) ? ctx->build_masks : nullptr;
  scan_kernel<<<dim3((unsigned)((cells + 255) / 256), 2), 256, 0, ctx->stream>>>(
      gkey, ckey, cells, S, out_stride, ground, ceiling, mk);
  if (mk) ctx->build_masks_written = true;
  if (int rc = check_launch(ctx, "scan_kernel")) return rc;
  ctx->keys_clean = true;  // the scan resets every key it reads
  return PCT_OK;
}

}  // namespace pct
