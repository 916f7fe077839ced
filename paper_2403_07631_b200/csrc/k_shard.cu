// k_shard.cu — row-band sharding of one large map over several GPUs
// (SURVEY.md §8 e; north_star: "points are bucketed per tile, stencil and
// inflation halos are exchanged with NCCL send/recv over NVLink").
//
// Kernels: owner-band partition of points (counting sort by destination
// band, order inside a band irrelevant because the build is
// order-independent).  The banded build itself is launch_build with a row
// window; the sweep primitives live in k_simplify.cu.  Collectives are issued
// by the host runtime (paper_2403_07631_b200/sharded.py) on torch tensors.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "pct_internal.h"

namespace pct {

int simplify_window_table(pct_ctx *ctx, const float *ground, const float *cost, int S,
                          int64_t cells, int64_t stride, double eps_e, double c_barrier,
                          uint64_t *table_host);
int simplify_triple_flags(pct_ctx *ctx, const float *ground, const float *cost, int S,
                          int64_t cells, int64_t stride, double eps_e, double c_barrier,
                          const int32_t *triples, int n, int32_t *flags_host);

namespace {

constexpr int kMaxBands = 64;

struct PartArgs {
  double y0, r_g, inv_rg;
  int starts[kMaxBands + 1];  // band b owns global rows [starts[b], starts[b+1])
  int nbands;
};

template <typename T>
__device__ __forceinline__ int owner_band(const T *xyz, int64_t p, const PartArgs &a) {
  const double y = (double)__ldg(xyz + 3 * p + 1);
  const double fi = floor(div_const(y - a.y0, a.r_g, a.inv_rg) + 0.5);  // tomogram.py:148
  int b = 0;
  while (b + 1 < a.nbands && fi >= (double)a.starts[b + 1]) ++b;
  return b;
}

template <typename T>
__global__ void __launch_bounds__(256) band_count_kernel(const T *__restrict__ xyz, int64_t n,
                                                         PartArgs a,
                                                         unsigned long long *__restrict__ counts) {
  __shared__ unsigned int local[kMaxBands];
  for (int b = threadIdx.x; b < a.nbands; b += blockDim.x) local[b] = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride)
    atomicAdd(&local[owner_band(xyz, p, a)], 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < a.nbands; b += blockDim.x)
    if (local[b]) atomicAdd(counts + b, (unsigned long long)local[b]);
}

// cursors[b] starts at the band's offset; every point is copied to its slot
template <typename T>
__global__ void __launch_bounds__(256) band_scatter_kernel(const T *__restrict__ xyz, int64_t n,
                                                           PartArgs a,
                                                           unsigned long long *__restrict__ cursors,
                                                           T *__restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
    const int b = owner_band(xyz, p, a);
    // warp-aggregated slot reservation per destination band
    const unsigned act = __activemask();
    const unsigned peers = __match_any_sync(act, b);
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(peers) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(cursors + b, (unsigned long long)__popc(peers));
    base = __shfl_sync(peers, base, leader);
    const unsigned long long slot = base + __popc(peers & ((1u << lane) - 1u));
    out[3 * slot] = xyz[3 * p];
    out[3 * slot + 1] = xyz[3 * p + 1];
    out[3 * slot + 2] = xyz[3 * p + 2];
  }
}

// dst[m] <- src[idx[m]] for n blocks of `block` floats (slice strides in
// floats); idx == nullptr means m.  blockIdx.y = m; 16-byte vectors when the
// layout allows.
constexpr int kMaxCopyIdx = 4096;

struct CopyIdx {
  int32_t idx[kMaxCopyIdx];
};

template <bool kVec>
__global__ void __launch_bounds__(256) copy_slices_kernel(float *__restrict__ dst, int64_t dstride,
                                                          const float *__restrict__ src,
                                                          int64_t sstride, int64_t block,
                                                          const CopyIdx *__restrict__ idx) {
  const int m = blockIdx.y;
  const int64_t k = idx ? idx->idx[m] : m;
  float *d = dst + (int64_t)m * dstride;
  const float *s = src + k * sstride;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  if (kVec) {
    const int64_t nv = block >> 2;
    float4 *d4 = reinterpret_cast<float4 *>(d);
    const float4 *s4 = reinterpret_cast<const float4 *>(s);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += step)
      __stcs(d4 + i, __ldcs(s4 + i));
  } else {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < block; i += step)
      d[i] = s[i];
  }
}

}  // namespace
}  // namespace pct

using namespace pct;

extern "C" {

int pct_partition_rows(pct_ctx *ctx, const void *xyz, int64_t n, int dtype, const pct_frame *fr,
                       const int32_t *band_starts, int32_t nbands, void *out,
                       int64_t *counts_host) {
  if (!ctx) return PCT_E_INVALID;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return PCT_E_CUDA;
  if (!fr || !band_starts || !counts_host || nbands <= 0 || nbands > kMaxBands ||
      (n > 0 && (!xyz || !out)) || (dtype != PCT_F32 && dtype != PCT_F64))
    return fail(ctx, PCT_E_INVALID, "bad arguments to pct_partition_rows");
  PartArgs a;
  a.y0 = fr->origin_y;
  a.r_g = fr->r_g;
  a.inv_rg = 1.0 / fr->r_g;
  a.nbands = nbands;
  for (int b = 0; b <= nbands; ++b) a.starts[b] = band_starts[b];
  unsigned long long *d = static_cast<unsigned long long *>(ctx->dsmall);  // counts | cursors
  PCT_CUDA(ctx, cudaMemsetAsync(d, 0, sizeof(unsigned long long) * 2 * kMaxBands, ctx->stream));
  const unsigned grid = (unsigned)std::max<int64_t>(
      1, std::min<int64_t>((n + 255) / 256, 8LL * ctx->num_sms));
  if (n > 0) {
    if (dtype == PCT_F32)
      band_count_kernel<float><<<grid, 256, 0, ctx->stream>>>(static_cast<const float *>(xyz), n,
                                                              a, d);
    else
      band_count_kernel<double><<<grid, 256, 0, ctx->stream>>>(static_cast<const double *>(xyz),
                                                               n, a, d);
    if (int rc = check_launch(ctx, "band_count_kernel")) return rc;
  }
  std::vector<unsigned long long> cnt(nbands);
  PCT_CUDA(ctx, cudaMemcpyAsync(cnt.data(), d, sizeof(unsigned long long) * nbands,
                                cudaMemcpyDeviceToHost, ctx->stream));
  PCT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  std::vector<unsigned long long> off(nbands);
  unsigned long long acc = 0;
  for (int b = 0; b < nbands; ++b) {
    off[b] = acc;
    acc += cnt[b];
    counts_host[b] = (int64_t)cnt[b];
  }
  if (n > 0) {
    PCT_CUDA(ctx, cudaMemcpyAsync(d + kMaxBands, off.data(), sizeof(unsigned long long) * nbands,
                                  cudaMemcpyHostToDevice, ctx->stream));
    if (dtype == PCT_F32)
      band_scatter_kernel<float><<<grid, 256, 0, ctx->stream>>>(
          static_cast<const float *>(xyz), n, a, d + kMaxBands, static_cast<float *>(out));
    else
      band_scatter_kernel<double><<<grid, 256, 0, ctx->stream>>>(
          static_cast<const double *>(xyz), n, a, d + kMaxBands, static_cast<double *>(out));
    if (int rc = check_launch(ctx, "band_scatter_kernel")) return rc;
    PCT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));  // the offsets buffer is reused
  }
  return PCT_OK;
}

int pct_copy_slices(pct_ctx *ctx, float *dst, int64_t dst_slice_stride, const float *src,
                    int64_t src_slice_stride, const int32_t *slice_idx_host, int32_t n,
                    int64_t block_elems) {
  if (!ctx) return PCT_E_INVALID;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return PCT_E_CUDA;
  if (n < 0 || n > kMaxCopyIdx || block_elems < 0 || (n > 0 && block_elems > 0 && (!dst || !src)))
    return fail(ctx, PCT_E_INVALID, "bad arguments to pct_copy_slices");
  if (n == 0 || block_elems == 0) return PCT_OK;
  const CopyIdx *didx = nullptr;
  if (slice_idx_host) {
    // the index list goes up through the context's small device buffer
    // (after the 2 x 64 partition counters)
    static_assert(sizeof(CopyIdx) + 2 * kMaxBands * 8 <= 65536, "dsmall too small");
    CopyIdx *d = reinterpret_cast<CopyIdx *>(static_cast<char *>(ctx->dsmall) + 2 * kMaxBands * 8);
    PCT_CUDA(ctx, upload_async(ctx, d, slice_idx_host, sizeof(int32_t) * n));
    didx = d;
  }
  const bool vec = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0 &&
                   (dst_slice_stride & 3) == 0 && (src_slice_stride & 3) == 0 &&
                   (block_elems & 3) == 0;
  const int64_t work = vec ? block_elems / 4 : block_elems;
  const unsigned gx = (unsigned)std::max<int64_t>(
      1, std::min<int64_t>((work + 255) / 256, std::max<int64_t>(1, 4LL * ctx->num_sms / n)));
  dim3 grid(gx, (unsigned)n);
  if (vec)
    copy_slices_kernel<true><<<grid, 256, 0, ctx->stream>>>(dst, dst_slice_stride, src,
                                                            src_slice_stride, block_elems, didx);
  else
    copy_slices_kernel<false><<<grid, 256, 0, ctx->stream>>>(dst, dst_slice_stride, src,
                                                             src_slice_stride, block_elems, didx);
  return check_launch(ctx, "copy_slices_kernel");
}

int pct_build_band(pct_ctx *ctx, const void *xyz, int64_t n, int dtype, const pct_frame *fr,
                   const double *heights, int32_t row0, int32_t nrows, int64_t out_slice_stride,
                   float *ground, float *ceiling) {
  if (!ctx) return PCT_E_INVALID;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return PCT_E_CUDA;
  if (!fr || !heights || !ground || !ceiling || (n > 0 && !xyz) ||
      (dtype != PCT_F32 && dtype != PCT_F64) || fr->cols <= 0 || fr->n_slices <= 0 ||
      nrows <= 0 || row0 < 0 || row0 + nrows > fr->rows ||
      (out_slice_stride != 0 && out_slice_stride < (int64_t)nrows * fr->cols))
    return fail(ctx, PCT_E_INVALID, "bad arguments to pct_build_band");
  return launch_build(ctx, xyz, n, dtype, *fr, heights, ground, ceiling, row0, nrows,
                      out_slice_stride);
}

int pct_simplify_window(pct_ctx *ctx, const float *ground, const float *cost, int32_t n_slices,
                        int64_t cells, int64_t slice_stride, double eps_e, double c_barrier,
                        uint64_t *table_host) {
  if (!ctx) return PCT_E_INVALID;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return PCT_E_CUDA;
  if (!ground || !cost || !table_host || n_slices < 0 || cells < 0)
    return fail(ctx, PCT_E_INVALID, "bad arguments to pct_simplify_window");
  return simplify_window_table(ctx, ground, cost, n_slices, cells,
                               slice_stride > 0 ? slice_stride : cells, eps_e, c_barrier,
                               table_host);
}

int pct_simplify_triples(pct_ctx *ctx, const float *ground, const float *cost, int32_t n_slices,
                         int64_t cells, int64_t slice_stride, double eps_e, double c_barrier,
                         const int32_t *triples, int32_t n_triples, int32_t *flags_host) {
  if (!ctx) return PCT_E_INVALID;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return PCT_E_CUDA;
  if (!ground || !cost || !triples || !flags_host || n_triples < 0)
    return fail(ctx, PCT_E_INVALID, "bad arguments to pct_simplify_triples");
  return simplify_triple_flags(ctx, ground, cost, n_slices, cells,
                               slice_stride > 0 ? slice_stride : cells, eps_e, c_barrier, triples,
                               n_triples, flags_host);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Planner context precompute (SURVEY.md §8 f rank 2): the per-cell run merge
// of planner.py:65-93 that the CPU A* consumes.  Runs of slices whose ground
// is valid in both and differs by <= eps_e form one canonical node: canon[k]
// = first slice of the run, cn[k] = minimum member cost of the run (inf where
// the ground is invalid), broadcast to every member.  One thread per cell
// column, a forward and a backward walk over k.
namespace pct {
namespace {

__global__ void __launch_bounds__(256) planner_ctx_kernel(const float *__restrict__ ground,
                                                          const float *__restrict__ cost, int S,
                                                          int64_t cells, double eps_e,
                                                          int32_t *__restrict__ canon,
                                                          float *__restrict__ cn) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cells) return;
  const float inf = __int_as_float(0x7f800000);
  float e_prev = ground[c];
  bool v_prev = finite32(e_prev);
  int32_t run = 0;
  float cmin = v_prev ? cost[c] : inf;
  canon[c] = 0;
  cn[c] = cmin;
  for (int k = 1; k < S; ++k) {
    const float e = ground[(int64_t)k * cells + c];
    const bool v = finite32(e);
    const bool eq = v && v_prev && fabs((double)e - (double)e_prev) <= eps_e;
    const float ck = v ? cost[(int64_t)k * cells + c] : inf;
    if (eq) {
      cmin = fminf(ck, cmin);  // np.minimum(cn[k], cn[k-1]); costs are never NaN
    } else {
      run = k;
      cmin = ck;
    }
    canon[(int64_t)k * cells + c] = run;
    cn[(int64_t)k * cells + c] = cmin;
    e_prev = e;
    v_prev = v;
  }
  // backward broadcast of the run minimum (planner.py:91-92)
  for (int k = S - 2; k >= 0; --k)
    if (canon[(int64_t)(k + 1) * cells + c] == canon[(int64_t)k * cells + c])
      cn[(int64_t)k * cells + c] = cn[(int64_t)(k + 1) * cells + c];
}

}  // namespace
}  // namespace pct

extern "C" int pct_planner_context(pct_ctx *ctx, const float *ground, const float *cost,
                                   int32_t n_slices, int32_t rows, int32_t cols, double eps_e,
                                   int32_t *canon, float *cn) {
  if (!ctx) return PCT_E_INVALID;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return PCT_E_CUDA;
  if (!ground || !cost || !canon || !cn || n_slices <= 0 || rows <= 0 || cols <= 0)
    return fail(ctx, PCT_E_INVALID, "bad arguments to pct_planner_context");
  const int64_t cells = (int64_t)rows * cols;
  planner_ctx_kernel<<<(unsigned)((cells + 255) / 256), 256, 0, ctx->stream>>>(
      ground, cost, n_slices, cells, eps_e, canon, cn);
  return check_launch(ctx, "planner_ctx_kernel");
}
