// k_trajectory.cu — ceiling inflation of the trajectory optimiser
// (SURVEY.md §8 f rank 4; replaces tomoplan/trajectory.py:277-317
// `_inflate_ceiling`, which _Problem.__init__ :366-374 runs per slice).
//
//   flat    = min over the disk {di^2 + dj^2 <= r^2}, r = ceil(erosion/res),
//             of the ceiling as float64, +inf where invalid or outside
//             (ndimage.minimum_filter, mode constant, cval inf, :291-296).
//             The footprint hypot(i, j) <= r + 1e-9 of :294 is exactly the
//             integer disk (i^2 + j^2 >= r^2 + 1 exceeds it by > 1e-9).
//   skirted = n_iter Jacobi sweeps of out[x] = min(out[x], min_n out[n] + w_n)
//             over the 8 neighbours, w = step or step*sqrt(2), step =
//             slope*res, n_iter = min(60, ceil(0.8/max(step, 1e-9))) (:298-316).
//
// Exactness: min is exact, and x -> RN(x + w) is monotone, so
// min_n RN(p_n + w) == RN(min_n p_n + w): two additions per cell instead of
// eight give the reference's bytes.  A sweep sequence that reaches a fixpoint
// early stays there, so the reference's global early exit and the per-tile
// early exit here both equal running all n_iter sweeps.
//
// skirt_pass_kernel does up to kSkirtT sweeps per launch on a 64x64 tile with
// a kSkirtT-cell halo held in shared memory (temporal blocking: one global
// read and write per kSkirtT sweeps); out-of-grid cells stay +inf.
#include <cuda_runtime.h>

#include <cmath>

#include "pct_internal.h"

namespace pct {
namespace {

constexpr int kMaxErosionCells = 64;
__constant__ int c_half_width[2 * kMaxErosionCells + 1];  // disk row half-widths

__global__ void __launch_bounds__(256) ceiling_flat_kernel(const float *__restrict__ ceiling,
                                                          int rows, int cols, int radius,
                                                          double *__restrict__ flat) {
  const int64_t cells = (int64_t)rows * cols;
  const int k = blockIdx.y;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cells) return;
  const int i = (int)(c / cols), j = (int)(c - (int64_t)i * cols);
  const float *ck = ceiling + (int64_t)k * cells;
  float m = INFINITY;  // invalid (non-finite) cells count as +inf
  for (int di = -radius; di <= radius; ++di) {
    const int y = i + di;
    if (y < 0 || y >= rows) continue;
    const int hw = c_half_width[di + radius];
    const int x0 = max(0, j - hw), x1 = min(cols - 1, j + hw);
    const float *row = ck + (int64_t)y * cols;
    for (int x = x0; x <= x1; ++x) {
      const float v = __ldg(row + x);
      if (isfinite(v)) m = fminf(m, v);
    }
  }
  flat[(int64_t)k * cells + c] = (double)m;
}

constexpr int kSkirtTile = 64;
constexpr int kSkirtT = 8;
constexpr int kSkirtRS = kSkirtTile + 2 * kSkirtT;
constexpr int kSkirtNT = 256;

__global__ void __launch_bounds__(kSkirtNT) skirt_pass_kernel(const double *__restrict__ src,
                                                              double *__restrict__ dst, int rows,
                                                              int cols, int sweeps, double w_ax,
                                                              double w_dg) {
  extern __shared__ double sk[];  // two (RS x RS) buffers
  const int64_t cells = (int64_t)rows * cols;
  const int k = blockIdx.z;
  const int i0 = blockIdx.y * kSkirtTile - kSkirtT, j0 = blockIdx.x * kSkirtTile - kSkirtT;
  const double *sk_src = src + (int64_t)k * cells;
  constexpr int N = kSkirtRS * kSkirtRS;
  for (int idx = threadIdx.x; idx < N; idx += kSkirtNT) {
    const int y = idx / kSkirtRS, x = idx - y * kSkirtRS;
    const int gi = i0 + y, gj = j0 + x;
    sk[idx] = (gi >= 0 && gi < rows && gj >= 0 && gj < cols) ? sk_src[(int64_t)gi * cols + gj]
                                                            : INFINITY;
  }
  __syncthreads();
  int cur = 0;
  for (int it = 0; it < sweeps; ++it) {
    const double *p = sk + cur * N;
    double *q = sk + (cur ^ 1) * N;
    int changed = 0;
    for (int idx = threadIdx.x; idx < N; idx += kSkirtNT) {
      const int y = idx / kSkirtRS, x = idx - y * kSkirtRS;
      const int gi = i0 + y, gj = j0 + x;
      double v = p[idx];
      // the region's outer ring has no neighbours here; it lies outside the
      // cells this pass must get right (>= `sweeps` away from the tile)
      if (y > 0 && y < kSkirtRS - 1 && x > 0 && x < kSkirtRS - 1 && gi >= 0 && gi < rows &&
          gj >= 0 && gj < cols) {
        const double *r = p + idx;
        const double ax = fmin(fmin(r[-kSkirtRS], r[kSkirtRS]), fmin(r[-1], r[1]));
        const double dg = fmin(fmin(r[-kSkirtRS - 1], r[-kSkirtRS + 1]),
                               fmin(r[kSkirtRS - 1], r[kSkirtRS + 1]));
        const double nv = fmin(v, fmin(ax + w_ax, dg + w_dg));
        changed |= nv != v;
        v = nv;
      }
      q[idx] = v;
    }
    cur ^= 1;
    if (!__syncthreads_or(changed)) break;  // fixpoint: further sweeps change nothing
  }
  const double *fin = sk + cur * N;
  double *dk = dst + (int64_t)k * cells;
  for (int idx = threadIdx.x; idx < kSkirtTile * kSkirtTile; idx += kSkirtNT) {
    const int y = idx / kSkirtTile, x = idx - y * kSkirtTile;
    const int gi = i0 + kSkirtT + y, gj = j0 + kSkirtT + x;
    if (gi < rows && gj < cols)
      dk[(int64_t)gi * cols + gj] = fin[(y + kSkirtT) * kSkirtRS + x + kSkirtT];
  }
}

}  // namespace
}  // namespace pct

using namespace pct;

extern "C" int pct_ceiling_inflate(pct_ctx *ctx, const float *ceiling, int32_t n_slices,
                                   int32_t rows, int32_t cols, double res, double erosion,
                                   double skirt_slope, double *flat, double *skirted) {
  if (!ctx) return PCT_E_INVALID;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return PCT_E_CUDA;
  if (!ceiling || !flat || !skirted || n_slices <= 0 || rows <= 0 || cols <= 0 || !(res > 0))
    return fail(ctx, PCT_E_INVALID, "bad arguments to pct_ceiling_inflate");
  // trajectory.py:291 (radius <= 0: no min filter), :300-301
  const double rq = std::ceil(erosion / res);
  if (rq > kMaxErosionCells)
    return fail(ctx, PCT_E_INVALID, "ceiling erosion radius above 64 cells");
  const int radius = rq > 0 ? (int)rq : 0;
  const double step = skirt_slope * res;
  const int n_iter = (int)std::min(60.0, std::ceil(0.8 / std::max(step, 1e-9)));
  const double w_ax = step * 1.0, w_dg = step * std::sqrt(2.0);
  int hw[2 * kMaxErosionCells + 1];
  for (int di = -radius; di <= radius; ++di) {
    int h = 0;
    while ((h + 1) * (h + 1) + di * di <= radius * radius) ++h;
    hw[di + radius] = h;
  }
  ConstBank cb(ctx);
  PCT_CUDA(ctx, cb.set_symbol(c_half_width, hw, sizeof(int) * (2 * radius + 1)));
  const int64_t cells = (int64_t)rows * cols;
  ceiling_flat_kernel<<<dim3((unsigned)((cells + 255) / 256), n_slices), 256, 0, ctx->stream>>>(
      ceiling, rows, cols, radius, flat);
  ctx->launches++;
  if (int rc = check_launch(ctx, "ceiling_flat_kernel")) return rc;
  // sweeps in passes of <= kSkirtT, ping-ponging so the last pass writes `skirted`
  const int passes = (n_iter + kSkirtT - 1) / kSkirtT;
  double *tmp = skirted;
  if (passes > 1) {
    if (int rc = ensure_scratch(ctx, (size_t)n_slices * cells * sizeof(double))) return rc;
    tmp = static_cast<double *>(ctx->scratch);
  }
  const size_t smem = 2 * sizeof(double) * kSkirtRS * kSkirtRS;
  PCT_CUDA(ctx, cudaFuncSetAttribute(skirt_pass_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const dim3 grid((cols + kSkirtTile - 1) / kSkirtTile, (rows + kSkirtTile - 1) / kSkirtTile,
                  n_slices);
  const double *src = flat;
  for (int p = 0; p < passes; ++p) {
    double *dst = ((passes - 1 - p) % 2 == 0) ? skirted : tmp;
    const int sweeps = std::min(kSkirtT, n_iter - p * kSkirtT);
    skirt_pass_kernel<<<grid, kSkirtNT, smem, ctx->stream>>>(src, dst, rows, cols, sweeps, w_ax,
                                                             w_dg);
    ctx->launches++;
    if (int rc = check_launch(ctx, "skirt_pass_kernel")) return rc;
    src = dst;
  }
  return PCT_OK;
}
