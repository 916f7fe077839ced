// hostmath.cpp — host build of csrc/cellmath.cuh for the CPU test suite
// (tests/test_cellmath.py).  TEST SUPPORT ONLY: the product path never calls
// these; they let the per-cell arithmetic that the sm_100a kernels execute be
// checked against the numpy oracle in a container without a GPU.
#include <cmath>
#include <cstdint>
#include <vector>

#include "cellmath.cuh"

using namespace pct;

extern "C" {

void pcth_hypot(const double *x, const double *y, int64_t n, double *out) {
  for (int64_t i = 0; i < n; ++i) out[i] = glibc_hypot(x[i], y[i]);
}

void pcth_div_const(const double *a, int64_t n, double d, double *out) {
  const double y = 1.0 / d;
  for (int64_t i = 0; i < n; ++i) out[i] = div_const(a[i], d, y);
}

// c_init of one slice (interval + terrain + foothold + fuse) composed exactly
// as the device stages B-D do, without tiling.
// fast (guarded) per-cell path of eval_fast_kernel on arrays of cells given
// as the 5-point cross; returns the number of cells that needed the exact
// glibc hypot (guard band hits)
int64_t pcth_fast_cells(const float *cross /* n x 5: e l r u d */, const float *ceil, int64_t n,
                        double r_g, const double *pv, float *enc_out, uint8_t *gentle_out) {
  EvalConsts K{};
  K.d_min = pv[0];
  K.d_ref = pv[1];
  K.theta_b = pv[2];
  K.theta_s = pv[3];
  K.c_barrier = pv[5];
  K.alpha_d = pv[6];
  K.alpha_b = pv[7];
  K.alpha_s = pv[8];
  K.rg = r_g;
  K.inv_rg = 1.0 / r_g;
  K.two_rg = 2.0 * r_g;
  K.inv_two_rg = 1.0 / K.two_rg;
  K.inv_theta_b = 1.0 / K.theta_b;
  K.inv_theta_s = 1.0 / K.theta_s;
  K.ts2_lo = K.theta_s * K.theta_s * (1.0 - 0x1p-40);
  K.ts2_hi = K.theta_s * K.theta_s * (1.0 + 0x1p-40);
  int64_t exact = 0;
  for (int64_t i = 0; i < n; ++i) {
    const float *p = cross + 5 * i;
    Cross c{p[0], p[1], p[2], p[3], p[4]};
    FastCell t = fast_terrain(c, K);
    enc_out[i] = fast_cinit(c.e, ceil[i], t, K);
    gentle_out[i] = t.gentle;
    if (t.valid && t.gentle && !t.isolated && !(t.m_xy > K.theta_b) && t.s != 0.0) {
      double cd;
      float f = gentle_cost_from(sqrt(t.s), K, &cd);
      if (!(t.s > 0x1p-900 && (float)(cd * (1.0 + 0x1p-44)) == f &&
            (float)(cd * (1.0 - 0x1p-44)) == f))
        ++exact;
    }
    if (t.valid && t.s >= K.ts2_lo && t.s <= K.ts2_hi) ++exact;
  }
  return exact;
}

// reference-order per-cell path (terrain_cell + cinit_encoded) on the same arrays
void pcth_ref_cells(const float *cross, const float *ceil, int64_t n, double r_g,
                    const double *pv, float *enc_out, uint8_t *gentle_out) {
  EvalConsts K{};
  K.d_min = pv[0];
  K.d_ref = pv[1];
  K.theta_b = pv[2];
  K.theta_s = pv[3];
  K.c_barrier = pv[5];
  K.alpha_d = pv[6];
  K.alpha_b = pv[7];
  K.alpha_s = pv[8];
  K.rg = r_g;
  K.inv_rg = 1.0 / r_g;
  K.two_rg = 2.0 * r_g;
  K.inv_two_rg = 1.0 / K.two_rg;
  K.inv_theta_b = 1.0 / K.theta_b;
  K.inv_theta_s = 1.0 / K.theta_s;
  for (int64_t i = 0; i < n; ++i) {
    const float *p = cross + 5 * i;
    Cross c{p[0], p[1], p[2], p[3], p[4]};
    TerrainCell t = terrain_cell(c, K);
    enc_out[i] = cinit_encoded(c.e, ceil[i], t, K);
    gentle_out[i] = t.gentle;
  }
}

void pcth_cinit(const float *g, const float *c, int rows, int cols, double r_g,
                const double *pv /* d_min d_ref theta_b theta_s theta_p c_barrier alpha_d
                                    alpha_b alpha_s */,
                int patch_radius, int ps_min_count, float *out) {
  EvalConsts K{};
  K.d_min = pv[0];
  K.d_ref = pv[1];
  K.theta_b = pv[2];
  K.theta_s = pv[3];
  K.c_barrier = pv[5];
  K.alpha_d = pv[6];
  K.alpha_b = pv[7];
  K.alpha_s = pv[8];
  K.rg = r_g;
  K.inv_rg = 1.0 / r_g;
  K.two_rg = 2.0 * r_g;
  K.inv_two_rg = 1.0 / K.two_rg;
  K.inv_theta_b = 1.0 / K.theta_b;
  K.inv_theta_s = 1.0 / K.theta_s;
  K.patch_radius = patch_radius;
  K.ps_min_count = ps_min_count;
  const float nanf_ = bits_f32(kNaNBits);
  auto at = [&](int i, int j) -> float {
    return (i >= 0 && i < rows && j >= 0 && j < cols) ? g[(int64_t)i * cols + j] : nanf_;
  };
  std::vector<uint8_t> gentle((size_t)rows * cols);
  std::vector<float> enc((size_t)rows * cols);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) {
      Cross x{at(i, j), at(i, j - 1), at(i, j + 1), at(i - 1, j), at(i + 1, j)};
      TerrainCell t = terrain_cell(x, K);
      gentle[(size_t)i * cols + j] = t.gentle;
      enc[(size_t)i * cols + j] = cinit_encoded(x.e, c[(int64_t)i * cols + j], t, K);
    }
  const int r = patch_radius;
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) {
      int cnt = 0;
      for (int a = i - r; a <= i + r; ++a)
        for (int b = j - r; b <= j + r; ++b)
          if (a >= 0 && a < rows && b >= 0 && b < cols) cnt += gentle[(size_t)a * cols + b];
      out[(size_t)i * cols + j] = cinit_resolve(enc[(size_t)i * cols + j], cnt, K);
    }
}

}  // extern "C"
