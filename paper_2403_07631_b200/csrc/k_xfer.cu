// k_xfer.cu — NaN-compacted read-back of layer slices (the layer transfer
// behind Layer.values / Tomogram.materialize, SURVEY.md §8 b).
//
// A ceiling slice is mostly the empty-cell NaN (tomogram.py:203-204: numpy's
// 0x7FC00000) -- 75 % of the cells of cfg3's kept ceilings -- and the drop-in
// chain is bound by PCIe (every surviving layer goes to host memory).  A
// compacted slice crosses PCIe as a bitmap (bit = cell is not the empty NaN)
// plus its non-empty values in cell order; host threads expand it into the
// caller's array while the dense slices are still in flight.  Lossless: a
// cell is "empty" only when its bits are exactly 0x7FC00000, every other
// value (any other NaN payload too) travels as it is.
//
// Device layout of one call over n slices (slice m = src + k_m * stride):
//   bitmaps [n][W] u32 (W = ceil(cells / 32)),
//   packed  values of slice m at packed + off[m] (off chosen by the caller),
//   chunk   [n][nchunk] i64: absolute packed index of each chunk's first
//           value (a chunk = kXChunk cells = 8 warps x 32 words).
// A warp takes 32 words (1024 cells): lane l loads cell 32 i + l of word i
// (coalesced), __ballot_sync forms word i, the lane's rank is a popcount.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "pct_internal.h"

namespace pct {
namespace {

constexpr int kXThreads = 256;
constexpr int kXWarpCells = 1024;                            // 32 words of 32 cells
constexpr int kXChunk = kXWarpCells * (kXThreads / 32);      // 8192 cells
constexpr int kXMaxSlices = 4096;

struct XferSlices {
  const float *src;
  int64_t stride;  // floats between slices
  int64_t cells;
  int n;
  int delta;  // slice m > 0 against slice m - 1 of the list (else every slice against NaN)
  int vec;    // every slice 16-byte aligned (the count kernel's vector loads)
  int32_t k[kXMaxSlices];
};

// the value slice m's cell is compared with: the empty NaN, or in a delta
// chain the previous listed slice's value
__device__ __forceinline__ const float *base_slice(const XferSlices *a, int m) {
  return (a->delta && m > 0) ? a->src + (int64_t)a->k[m - 1] * a->stride : nullptr;
}
__device__ __forceinline__ bool differs(float v, const float *b, int64_t cell) {
  return f32_bits(v) != (b ? f32_bits(__ldg(b + cell)) : kNaNBits);
}

// blockIdx.x = chunk, blockIdx.y = slice: non-empty cells of the chunk
// (wcnt, when given: the count of each warp's 1024 cells too, [n][nchunk][8])
__global__ void __launch_bounds__(kXThreads) xfer_count_kernel(const XferSlices *__restrict__ a,
                                                               unsigned *__restrict__ cnt,
                                                               int nchunk,
                                                               unsigned *__restrict__ wcnt) {
  __shared__ unsigned part[kXThreads / 32];
  const int m = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t cells = a->cells;
  const float *s = a->src + (int64_t)a->k[m] * a->stride, *bs = base_slice(a, m);
  const int64_t base = (int64_t)blockIdx.x * kXChunk + (int64_t)warp * kXWarpCells;
  unsigned c = 0;
  if (a->vec && base + kXWarpCells <= cells) {
    // a count does not depend on the cell order: 16-byte loads, lane l takes
    // cells 4 (l + 32 i) .. +3 of the warp's 1024 (slices 16-byte aligned)
    const float4 *s4 = reinterpret_cast<const float4 *>(s + base);
    const float4 *b4 = bs ? reinterpret_cast<const float4 *>(bs + base) : nullptr;
    float4 v[8], w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v[i] = __ldg(s4 + 32 * i + lane);
      w[i] = b4 ? __ldg(b4 + 32 * i + lane) : make_float4(bits_f32(kNaNBits), bits_f32(kNaNBits),
                                                           bits_f32(kNaNBits), bits_f32(kNaNBits));
    }
    unsigned n = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      n += (f32_bits(v[i].x) != f32_bits(w[i].x)) + (f32_bits(v[i].y) != f32_bits(w[i].y)) +
           (f32_bits(v[i].z) != f32_bits(w[i].z)) + (f32_bits(v[i].w) != f32_bits(w[i].w));
    c = __reduce_add_sync(0xFFFFFFFFu, n);
  } else {
#pragma unroll 8
    for (int i = 0; i < 32; ++i) {
      const int64_t cell = base + i * 32 + lane;
      const bool v = cell < cells && differs(__ldg(s + cell), bs, cell);
      c += __popc(__ballot_sync(0xFFFFFFFFu, v));
    }
  }
  if (lane == 0) {
    part[warp] = c;
    if (wcnt) wcnt[((int64_t)m * nchunk + blockIdx.x) * (kXThreads / 32) + warp] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int w = 0; w < kXThreads / 32; ++w) t += part[w];
    cnt[(int64_t)m * nchunk + blockIdx.x] = t;
  }
}

// one block per slice: exclusive prefix of its chunk counts (absolute, from
// the slice's packed offset) and the slice total
__global__ void __launch_bounds__(1024) xfer_scan_kernel(const unsigned *__restrict__ cnt,
                                                         int nchunk,
                                                         const int64_t *__restrict__ off,
                                                         int64_t *__restrict__ chunk_off,
                                                         int64_t *__restrict__ totals) {
  __shared__ int64_t wsum[32];
  __shared__ int64_t carry;
  const int m = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (t == 0) carry = off ? off[m] : 0;
  __syncthreads();
  for (int c0 = 0; c0 < nchunk; c0 += 1024) {
    const int c = c0 + t;
    int64_t v = c < nchunk ? cnt[(int64_t)m * nchunk + c] : 0;
    int64_t x = v;  // inclusive warp scan
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int64_t y = __shfl_up_sync(0xFFFFFFFFu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int64_t w = wsum[lane];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int64_t y = __shfl_up_sync(0xFFFFFFFFu, w, d);
        if (lane >= d) w += y;
      }
      wsum[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const int64_t before = carry + (warp ? wsum[warp - 1] : 0) + x - v;
    if (c < nchunk) chunk_off[(int64_t)m * nchunk + c] = before;
    __syncthreads();
    if (t == 0) carry += wsum[31];
    __syncthreads();
  }
  if (t == 0 && totals) totals[m] = carry - (off ? off[m] : 0);
}

// blockIdx.x = chunk, blockIdx.y = slice: bitmap words and packed values.
// A warp's first packed position is its chunk's offset plus the counts of
// the warps before it (from the count pass), so the warp streams its 32
// words once, 8 in flight, without holding them (cfg3: 118 registers /
// 25 % occupancy / 4.8 ms per stack before, with an in-kernel recount)
__global__ void __launch_bounds__(kXThreads) xfer_pack_kernel(const XferSlices *__restrict__ a,
                                                              const int64_t *__restrict__ chunk_off,
                                                              const unsigned *__restrict__ wcnt,
                                                              int nchunk,
                                                              uint32_t *__restrict__ bitmaps,
                                                              float *__restrict__ packed) {
  const int m = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t cells = a->cells, W = (cells + 31) / 32;
  const float *s = a->src + (int64_t)a->k[m] * a->stride, *bs = base_slice(a, m);
  const int64_t base = (int64_t)blockIdx.x * kXChunk + (int64_t)warp * kXWarpCells;
  const int64_t ci = (int64_t)m * nchunk + blockIdx.x;
  int64_t pos = chunk_off[ci];
  const unsigned *wc = wcnt + ci * (kXThreads / 32);
  for (int w = 0; w < warp; ++w) pos += wc[w];
  const unsigned lt = (1u << lane) - 1u;
  const int64_t w0 = base / 32;
  uint32_t *bm = bitmaps + (int64_t)m * W;
#ifndef PCT_XFER_PACK_U
#define PCT_XFER_PACK_U 8
#endif
  constexpr int U = PCT_XFER_PACK_U;  // words in flight
  // branch-free loads (clamped addresses, the base slice read from `s`
  // itself when there is none) so the U words' loads issue together
  const bool use_b = bs != nullptr;
  const float *bsrc = use_b ? bs : s;
#pragma unroll 1
  for (int i0 = 0; i0 < 32; i0 += U) {
    float v[U];
    uint32_t bv[U];
    bool d[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t cell = base + (i0 + u) * 32 + lane;
      const int64_t cc = cell < cells ? cell : cells - 1;
      v[u] = __ldg(s + cc);
      bv[u] = f32_bits(__ldg(bsrc + cc));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t cell = base + (i0 + u) * 32 + lane;
      d[u] = cell < cells && f32_bits(v[u]) != (use_b ? bv[u] : kNaNBits);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned bal = __ballot_sync(0xFFFFFFFFu, d[u]);
      if (d[u]) packed[pos + __popc(bal & lt)] = v[u];
      pos += __popc(bal);
      if (lane == i0 + u && w0 + i0 + u < W) bm[w0 + i0 + u] = bal;
    }
  }
}

int setup(pct_ctx *ctx, const float *src, int64_t stride, const int32_t *idx, int32_t n,
          int64_t cells, int delta, XferSlices **dargs, int *nchunk) {
  if (!ctx) return PCT_E_INVALID;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return PCT_E_CUDA;
  if (!src || !idx || n <= 0 || n > kXMaxSlices || cells <= 0 || stride < cells)
    return fail(ctx, PCT_E_INVALID, "bad arguments to the compacted read-back");
  const int64_t nc = (cells + kXChunk - 1) / kXChunk;
  if (nc > (int64_t)1 << 30) return fail(ctx, PCT_E_INVALID, "slice too large");
  *nchunk = (int)nc;
  // scratch: args | chunk counts [n][nchunk] u32 | chunk offsets [n][nchunk] i64 | totals [n]
  // (256-byte padded) | warp counts [n][nchunk][8] u32
  const size_t abytes = (sizeof(XferSlices) + 255) & ~(size_t)255;
  const size_t cbytes = ((size_t)n * nc * 4 + 255) & ~(size_t)255;
  const size_t obytes = ((size_t)n * nc * 8 + 255) & ~(size_t)255;
  const size_t tbytes = ((size_t)n * 8 + 255) & ~(size_t)255;
  const size_t wbytes = (size_t)n * nc * (kXThreads / 32) * 4;
  if (int rc = ensure_scratch(ctx, abytes + cbytes + obytes + tbytes + wbytes + 256)) return rc;
  XferSlices h;
  h.src = src;
  h.stride = stride;
  h.cells = cells;
  h.n = n;
  h.delta = delta ? 1 : 0;
  h.vec = (reinterpret_cast<uintptr_t>(src) & 15) == 0 && stride % 4 == 0;
  std::memcpy(h.k, idx, sizeof(int32_t) * (size_t)n);
  *dargs = static_cast<XferSlices *>(ctx->scratch);
  const size_t used = offsetof(XferSlices, k) + sizeof(int32_t) * (size_t)n;
  PCT_CUDA(ctx, upload_async(ctx, *dargs, &h, used));
  return PCT_OK;
}

}  // namespace
}  // namespace pct

using namespace pct;

static int xfer_count(pct_ctx *ctx, const float *src, int64_t slice_stride,
                      const int32_t *slice_idx_host, int32_t n, int64_t cells, int32_t delta,
                      int64_t *totals_host, bool sync, uint32_t *keep = nullptr) {
  XferSlices *da = nullptr;
  int nchunk = 0;
  if (int rc = setup(ctx, src, slice_stride, slice_idx_host, n, cells, delta, &da, &nchunk))
    return rc;
  if (!totals_host) return fail(ctx, PCT_E_INVALID, "pct_xfer_count: totals_host is NULL");
  char *b = static_cast<char *>(ctx->scratch);
  const size_t abytes = (sizeof(XferSlices) + 255) & ~(size_t)255;
  const size_t cbytes = ((size_t)n * nchunk * 4 + 255) & ~(size_t)255;
  const size_t obytes = ((size_t)n * nchunk * 8 + 255) & ~(size_t)255;
  // kept counts (pct_xfer_count_keep): chunk counts [n][nchunk] then warp
  // counts [n][nchunk][8] in the caller's device buffer, for pct_xfer_pack_counted
  unsigned *cnt = keep ? keep : reinterpret_cast<unsigned *>(b + abytes);
  unsigned *wcnt = keep ? keep + (size_t)n * nchunk : nullptr;
  int64_t *coff = reinterpret_cast<int64_t *>(b + abytes + cbytes);
  int64_t *tot = reinterpret_cast<int64_t *>(b + abytes + cbytes + obytes);
  xfer_count_kernel<<<dim3((unsigned)nchunk, (unsigned)n), kXThreads, 0, ctx->stream>>>(
      da, cnt, nchunk, wcnt);
  if (int rc = check_launch(ctx, "xfer_count_kernel")) return rc;
  xfer_scan_kernel<<<(unsigned)n, 1024, 0, ctx->stream>>>(cnt, nchunk, nullptr, coff, tot);
  if (int rc = check_launch(ctx, "xfer_scan_kernel")) return rc;
  PCT_CUDA(ctx, cudaMemcpyAsync(totals_host, tot, (size_t)n * 8, cudaMemcpyDeviceToHost,
                                ctx->stream));
  if (sync) PCT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return PCT_OK;
}

extern "C" int pct_xfer_count(pct_ctx *ctx, const float *src, int64_t slice_stride,
                              const int32_t *slice_idx_host, int32_t n, int64_t cells,
                              int32_t delta, int64_t *totals_host) {
  return xfer_count(ctx, src, slice_stride, slice_idx_host, n, cells, delta, totals_host, true);
}

extern "C" int pct_xfer_count_async(pct_ctx *ctx, const float *src, int64_t slice_stride,
                                    const int32_t *slice_idx_host, int32_t n, int64_t cells,
                                    int32_t delta, int64_t *totals_host) {
  return xfer_count(ctx, src, slice_stride, slice_idx_host, n, cells, delta, totals_host, false);
}

extern "C" int pct_xfer_pack(pct_ctx *ctx, const float *src, int64_t slice_stride,
                             const int32_t *slice_idx_host, int32_t n, int64_t cells,
                             int32_t delta, const int64_t *packed_off_host, uint32_t *bitmaps,
                             float *packed, int64_t *chunk_off) {
  XferSlices *da = nullptr;
  int nchunk = 0;
  if (int rc = setup(ctx, src, slice_stride, slice_idx_host, n, cells, delta, &da, &nchunk))
    return rc;
  if (!packed_off_host || !bitmaps || !packed || !chunk_off)
    return fail(ctx, PCT_E_INVALID, "pct_xfer_pack: NULL buffer");
  char *b = static_cast<char *>(ctx->scratch);
  const size_t abytes = (sizeof(XferSlices) + 255) & ~(size_t)255;
  const size_t cbytes = ((size_t)n * nchunk * 4 + 255) & ~(size_t)255;
  const size_t obytes = ((size_t)n * nchunk * 8 + 255) & ~(size_t)255;
  const size_t tbytes = ((size_t)n * 8 + 255) & ~(size_t)255;
  unsigned *cnt = reinterpret_cast<unsigned *>(b + abytes);
  int64_t *doff = reinterpret_cast<int64_t *>(b + abytes + cbytes + obytes);
  unsigned *wcnt = reinterpret_cast<unsigned *>(b + abytes + cbytes + obytes + tbytes);
  PCT_CUDA(ctx, upload_async(ctx, doff, packed_off_host, (size_t)n * 8));
  xfer_count_kernel<<<dim3((unsigned)nchunk, (unsigned)n), kXThreads, 0, ctx->stream>>>(
      da, cnt, nchunk, wcnt);
  if (int rc = check_launch(ctx, "xfer_count_kernel")) return rc;
  xfer_scan_kernel<<<(unsigned)n, 1024, 0, ctx->stream>>>(cnt, nchunk, doff, chunk_off, nullptr);
  if (int rc = check_launch(ctx, "xfer_scan_kernel")) return rc;
  xfer_pack_kernel<<<dim3((unsigned)nchunk, (unsigned)n), kXThreads, 0, ctx->stream>>>(
      da, chunk_off, wcnt, nchunk, bitmaps, packed);
  return check_launch(ctx, "xfer_pack_kernel");
}

extern "C" int64_t pct_xfer_chunk_cells(void) { return kXChunk; }

extern "C" int pct_xfer_fence(pct_ctx *ctx, int32_t slot) {
  if (!ctx) return PCT_E_INVALID;
  if (slot < 0 || slot >= kXferEvents) return fail(ctx, PCT_E_INVALID, "pct_xfer_fence: bad slot");
  if (cudaSetDevice(ctx->device) != cudaSuccess) return PCT_E_CUDA;
  if (!ctx->xfer_ev[slot])
    PCT_CUDA(ctx, cudaEventCreateWithFlags(&ctx->xfer_ev[slot], cudaEventDisableTiming));
  PCT_CUDA(ctx, cudaEventRecord(ctx->xfer_ev[slot], ctx->stream));
  return PCT_OK;
}

extern "C" int pct_xfer_wait(pct_ctx *ctx, int32_t slot) {
  if (!ctx) return PCT_E_INVALID;
  if (slot < 0 || slot >= kXferEvents) return fail(ctx, PCT_E_INVALID, "pct_xfer_wait: bad slot");
  if (!ctx->xfer_ev[slot]) return PCT_OK;
  PCT_CUDA(ctx, cudaEventSynchronize(ctx->xfer_ev[slot]));
  return PCT_OK;
}

// The host side, pct_xfer_expand, is in xfer_host.cpp (g++, AVX-512 when the
// host has it).

extern "C" int64_t pct_xfer_counts_bytes(int64_t cells, int32_t n) {
  if (cells <= 0 || n <= 0) return 0;
  const int64_t nc = (cells + kXChunk - 1) / kXChunk;
  return (int64_t)n * nc * (1 + kXThreads / 32) * 4;
}

extern "C" int pct_xfer_count_keep(pct_ctx *ctx, const float *src, int64_t slice_stride,
                                   const int32_t *slice_idx_host, int32_t n, int64_t cells,
                                   int32_t delta, int64_t *totals_host, uint32_t *counts_dev) {
  if (!counts_dev) return fail(ctx, PCT_E_INVALID, "pct_xfer_count_keep: counts_dev is NULL");
  return xfer_count(ctx, src, slice_stride, slice_idx_host, n, cells, delta, totals_host, false,
                    counts_dev);
}

extern "C" int pct_xfer_pack_counted(pct_ctx *ctx, const float *src, int64_t slice_stride,
                                     const int32_t *slice_idx_host, int32_t n, int64_t cells,
                                     int32_t delta, const int64_t *packed_off_host,
                                     const uint32_t *counts_dev, uint32_t *bitmaps, float *packed,
                                     int64_t *chunk_off) {
  XferSlices *da = nullptr;
  int nchunk = 0;
  if (int rc = setup(ctx, src, slice_stride, slice_idx_host, n, cells, delta, &da, &nchunk))
    return rc;
  if (!packed_off_host || !counts_dev || !bitmaps || !packed || !chunk_off)
    return fail(ctx, PCT_E_INVALID, "pct_xfer_pack_counted: NULL buffer");
  char *b = static_cast<char *>(ctx->scratch);
  const size_t abytes = (sizeof(XferSlices) + 255) & ~(size_t)255;
  const size_t cbytes = ((size_t)n * nchunk * 4 + 255) & ~(size_t)255;
  const size_t obytes = ((size_t)n * nchunk * 8 + 255) & ~(size_t)255;
  int64_t *doff = reinterpret_cast<int64_t *>(b + abytes + cbytes + obytes);
  PCT_CUDA(ctx, upload_async(ctx, doff, packed_off_host, (size_t)n * 8));
  xfer_scan_kernel<<<(unsigned)n, 1024, 0, ctx->stream>>>(counts_dev, nchunk, doff, chunk_off,
                                                         nullptr);
  if (int rc = check_launch(ctx, "xfer_scan_kernel")) return rc;
  xfer_pack_kernel<<<dim3((unsigned)nchunk, (unsigned)n), kXThreads, 0, ctx->stream>>>(
      da, chunk_off, counts_dev + (size_t)n * nchunk, nchunk, bitmaps, packed);
  return check_launch(ctx, "xfer_pack_kernel");
}
