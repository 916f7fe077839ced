// k_ops.cu — element-wise / small-stencil kernels behind the reference's
// per-operation API (traversability.py:106-170): slope_magnitudes,
// gentle_fraction, terrain_cost_values, fuse_costs.  The fused pipeline
// (k_evaluate.cu) does not use these; they exist so the drop-in per-op
// functions also run on the device.
#include <cuda_runtime.h>

#include "pct_internal.h"

namespace pct {
namespace {

__constant__ EvalConsts c_Kops;

__global__ void slope_kernel(const float *__restrict__ g, int rows, int cols,
                             double *__restrict__ m_xy, double *__restrict__ m_grad,
                             uint8_t *__restrict__ iso) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)rows * cols) return;
  const int i = (int)(idx / cols), j = (int)(idx - (int64_t)i * cols);
  const float nanf_ = bits_f32(kNaNBits);
  Cross c{g[idx], j > 0 ? g[idx - 1] : nanf_, j + 1 < cols ? g[idx + 1] : nanf_,
          i > 0 ? g[idx - cols] : nanf_, i + 1 < rows ? g[idx + cols] : nanf_};
  TerrainCell t = terrain_cell(c, c_Kops);
  m_xy[idx] = t.m_xy;
  m_grad[idx] = t.m_grad;
  iso[idx] = t.isolated ? 1 : 0;
}

__global__ void gentle_fraction_kernel(const uint8_t *__restrict__ gentle, int rows, int cols,
                                       int radius, double *__restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)rows * cols) return;
  const int i = (int)(idx / cols), j = (int)(idx - (int64_t)i * cols);
  int cnt = 0;
  for (int a = max(0, i - radius); a <= min(rows - 1, i + radius); ++a)
    for (int b = max(0, j - radius); b <= min(cols - 1, j + radius); ++b)
      cnt += gentle[(int64_t)a * cols + b] ? 1 : 0;
  const int side = 2 * radius + 1;
  out[idx] = (double)cnt / (double)(side * side);
}

// terrain_cost_values on arbitrary float64 inputs: true IEEE division (inputs
// may be non-finite here, where the Markstein shortcut is not valid).
__global__ void terrain_values_kernel(const double *__restrict__ m_xy,
                                      const double *__restrict__ m_grad,
                                      const double *__restrict__ p_s, int64_t n, double theta_p,
                                      double *__restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n) return;
  const EvalConsts &K = c_Kops;
  const double mx = m_xy[idx], mg = m_grad[idx], ps = p_s[idx];
  const double qb = mx / K.theta_b, qs = mg / K.theta_s;
  const double step = ps > theta_p ? K.alpha_b * (qb * qb) : K.c_barrier;
  const double gentle = K.alpha_s * (qs * qs);
  out[idx] = mx > K.theta_b ? K.c_barrier : (mg < K.theta_s ? gentle : step);
}

__global__ void fuse_kernel(const float *__restrict__ ci, const float *__restrict__ cg,
                            const uint8_t *__restrict__ valid, int64_t n,
                            float *__restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n) return;
  const EvalConsts &K = c_Kops;
  if (!valid[idx]) {
    out[idx] = (float)K.c_barrier;
    return;
  }
  const double s = (double)ci[idx] + (double)cg[idx];
  // np.minimum propagates NaN
  out[idx] = (float)(isnan(s) ? s : (K.c_barrier < s ? K.c_barrier : s));
}

inline unsigned blocks(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

int launch_slope(pct_ctx *ctx, const float *g, int rows, int cols, double r_g, double *m_xy,
                 double *m_grad, uint8_t *iso) {
  pct_trav_params p{};
  p.theta_s = 0.36;  // gentle flag unused here
  p.theta_b = 1.7;
  p.theta_p = 0.2;
  p.c_barrier = 50;
  EvalConsts K = make_consts(p, r_g);
  ConstBank cb(ctx);
  PCT_CUDA(ctx, cb.set_symbol(c_Kops, &K, sizeof(K)));
  const int64_t n = (int64_t)rows * cols;
  if (n == 0) return PCT_OK;
  slope_kernel<<<blocks(n), 256, 0, ctx->stream>>>(g, rows, cols, m_xy, m_grad, iso);
  return check_launch(ctx, "slope_kernel");
}

int launch_gentle_fraction(pct_ctx *ctx, const uint8_t *gentle, int rows, int cols, int radius,
                           double *out) {
  const int64_t n = (int64_t)rows * cols;
  if (n == 0) return PCT_OK;
  gentle_fraction_kernel<<<blocks(n), 256, 0, ctx->stream>>>(gentle, rows, cols, radius, out);
  return check_launch(ctx, "gentle_fraction_kernel");
}

int launch_terrain_values(pct_ctx *ctx, const double *m_xy, const double *m_grad,
                          const double *p_s, int64_t n, const pct_trav_params &p, double *out) {
  EvalConsts K = make_consts(p, 1.0);
  ConstBank cb(ctx);
  PCT_CUDA(ctx, cb.set_symbol(c_Kops, &K, sizeof(K)));
  if (n == 0) return PCT_OK;
  terrain_values_kernel<<<blocks(n), 256, 0, ctx->stream>>>(m_xy, m_grad, p_s, n, p.theta_p, out);
  return check_launch(ctx, "terrain_values_kernel");
}

int launch_fuse(pct_ctx *ctx, const float *ci, const float *cg, const uint8_t *valid, int64_t n,
                const pct_trav_params &p, float *out) {
  EvalConsts K = make_consts(p, 1.0);
  ConstBank cb(ctx);
  PCT_CUDA(ctx, cb.set_symbol(c_Kops, &K, sizeof(K)));
  if (n == 0) return PCT_OK;
  fuse_kernel<<<blocks(n), 256, 0, ctx->stream>>>(ci, cg, valid, n, out);
  return check_launch(ctx, "fuse_kernel");
}

}  // namespace pct
