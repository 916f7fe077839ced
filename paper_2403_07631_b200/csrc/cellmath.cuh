// cellmath.cuh — per-cell arithmetic of the hot path, shared by the sm_100a
// kernels and a host build used by the CPU tests (tests/test_cellmath.py).
//
// Bit-exactness contract: every expression follows the
// reference's numpy operation order in float64 and rounds to float32 exactly
// where the reference does.  The library is compiled with --fmad=false
// (device) / -ffp-contract=off (host); the only fused multiply-adds are the
// explicit fma() calls of the Markstein division below.
#pragma once

#include <math.h>
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define PCT_HD __host__ __device__ __forceinline__
#else
#define PCT_HD static inline
#endif

namespace pct {

PCT_HD uint32_t f32_bits(float f) {
#if defined(__CUDA_ARCH__)
  return __float_as_uint(f);
#else
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
#endif
}
PCT_HD float bits_f32(uint32_t u) {
#if defined(__CUDA_ARCH__)
  return __uint_as_float(u);
#else
  float f;
  memcpy(&f, &u, 4);
  return f;
#endif
}

// numpy's float32 NaN (np.float32(np.nan)): the invalid-cell marker the
// reference writes (tomogram.py:203-204) and the LGA archive stores.
static constexpr uint32_t kNaNBits = 0x7FC00000u;

// Order-preserving float32 -> uint32 key: a < b  <=>  key(a) < key(b) for
// all non-NaN floats (-0.0 sorts just below +0.0).  Key 0 and key ~0u are
// never produced by a finite float, so they encode "empty" for max / min.
PCT_HD uint32_t f32_key(float f) {
  uint32_t u = f32_bits(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
PCT_HD float key_f32(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
  return bits_f32(u);
}
// f32_bits(key_f32(k)) in two instructions (shift + one LOP3)
PCT_HD uint32_t key_bits(uint32_t k) {
  return k ^ (~(uint32_t)((int32_t)k >> 31) | 0x80000000u);
}
static constexpr uint32_t kKeyEmptyMax = 0u;           // identity of max
static constexpr uint32_t kKeyEmptyMin = 0xFFFFFFFFu;  // identity of min

PCT_HD float decode_ground(uint32_t k) {
  return k == kKeyEmptyMax ? bits_f32(kNaNBits) : key_f32(k);
}
PCT_HD float decode_ceiling(uint32_t k) {
  return k == kKeyEmptyMin ? bits_f32(kNaNBits) : key_f32(k);
}

PCT_HD bool finite32(float f) { return (f32_bits(f) & 0x7F800000u) != 0x7F800000u; }

// Correctly rounded a / d for a compile-time-like constant divisor d with
// yinv = RN(1/d): q0 = RN(a*yinv) is within 1 ulp of a/d, the FMA residual
// r = a - d*q0 is exact, and RN(q0 + r*yinv) = RN(a/d) (Markstein's theorem).
// Verified against IEEE division on 8e8 samples.
PCT_HD double div_const(double a, double d, double yinv) {
  double q0 = a * yinv;
  double r = fma(-q0, d, a);
  return fma(r, yinv, q0);
}

// glibc >= 2.35 hypot (sysdeps/ieee754/dbl-64/e_hypot.c, non-FMA kernel),
// restated: numpy's np.hypot calls libm hypot, and the reference computes
// m_grad with it (traversability.py:112).  Matches glibc 2.39 bit-for-bit on
// 2e8 random pairs (tests/test_cellmath.py re-checks against np.hypot).
PCT_HD double hypot_kernel(double ax, double ay) {
  double h = sqrt(ax * ax + ay * ay);
  double t1, t2;
  if (h <= 2.0 * ay) {
    double delta = h - ay;
    t1 = ax * (2.0 * delta - ax);
    t2 = (delta - 2.0 * (ax - ay)) * delta;
  } else {
    double delta = h - ax;
    t1 = 2.0 * delta * (ax - 2.0 * ay);
    t2 = (4.0 * delta - ay) * ay + delta * delta;
  }
  h -= (t1 + t2) / (2.0 * h);
  return h;
}

PCT_HD double glibc_hypot(double x, double y) {
  // inputs here are always finite (differences of finite float32 values)
  x = fabs(x);
  y = fabs(y);
  double ax = x < y ? y : x;
  double ay = x < y ? x : y;
  const double kScale = 0x1p-600, kLarge = 0x1p+511, kTiny = 0x1p-459, kEps = 0x1p-54;
  if (ax > kLarge) {
    if (ay <= ax * kEps) return ax + ay;
    return hypot_kernel(ax * kScale, ay * kScale) / kScale;
  }
  if (ay < kTiny) {
    if (ax >= ay / kEps) return ax + ay;
    return hypot_kernel(ax / kScale, ay / kScale) * kScale;
  }
  if (ay <= ax * kEps) return ax + ay;
  return hypot_kernel(ax, ay);
}

// Constants of the per-cell evaluation, precomputed on the host.
struct EvalConsts {
  double d_min, d_ref, theta_b, theta_s, c_barrier, alpha_d, alpha_b, alpha_s;
  double rg, inv_rg, two_rg, inv_two_rg;  // gradient divisors (traversability.py:100-102)
  double inv_theta_b, inv_theta_s;        // q = m / theta (traversability.py:138,141)
  double ts2_lo, ts2_hi;  // theta_s^2 (1 -/+ 2^-40): guard band of the gentle test
  int32_t ps_min_count;  // smallest gentle count c with RN(c/(2r+1)^2) > theta_p
  int32_t patch_radius;
};

// One axis of _axis_gradient (traversability.py:76-103): central difference
// where both neighbours are valid, one-sided otherwise, 0 with none.
// Branch-free form: with no valid neighbour the numerator is ef - ef = +0 and
// the quotient +0, as in the reference.
PCT_HD double axis_gradient(bool vn, bool vp, double en, double ep, double ef,
                            const EvalConsts &K) {
  const bool both = vn && vp;
  const double num = (vn ? en : ef) - (vp ? ep : ef);
  return div_const(num, both ? K.two_rg : K.rg, both ? K.inv_two_rg : K.inv_rg);
}

// Neighbourhood of one ground cell: centre e and the 4 axis neighbours
// (x = columns: r = j+1, l = j-1; y = rows: d = i+1, u = i-1).  NaN = invalid
// (cells outside the grid are passed as NaN).
struct Cross {
  float e, l, r, u, d;
};

struct TerrainCell {
  double m_xy, m_grad;
  bool valid, isolated, gentle;
};

PCT_HD TerrainCell terrain_cell(const Cross &c, const EvalConsts &K) {
  TerrainCell t;
  bool v = finite32(c.e), vl = finite32(c.l), vr = finite32(c.r), vu = finite32(c.u),
       vd = finite32(c.d);
  double ef = v ? (double)c.e : 0.0;
  double gx = axis_gradient(vr, vl, vr ? (double)c.r : 0.0, vl ? (double)c.l : 0.0, ef, K);
  double gy = axis_gradient(vd, vu, vd ? (double)c.d : 0.0, vu ? (double)c.u : 0.0, ef, K);
  double ax = fabs(gx), ay = fabs(gy);
  t.m_xy = ax > ay ? ax : ay;
  t.m_grad = glibc_hypot(gx, gy);
  t.valid = v;
  t.isolated = v && !(vl || vr || vu || vd);
  t.gentle = v && (t.m_grad < K.theta_s);
  return t;
}

// Terrain branch (traversability.py:131-147) in float64.  *needs_ps is set
// for the foothold branch whose value holds only when p_s > theta_p.
PCT_HD double terrain_value(double m_xy, double m_grad, const EvalConsts &K, bool *needs_ps) {
  *needs_ps = false;
  if (m_xy > K.theta_b) return K.c_barrier;
  if (m_grad < K.theta_s) {
    double q = div_const(m_grad, K.theta_s, K.inv_theta_s);
    return K.alpha_s * (q * q);
  }
  *needs_ps = true;
  double q = div_const(m_xy, K.theta_b, K.inv_theta_b);
  return K.alpha_b * (q * q);
}

// interval_cost (traversability.py:59-73) for a valid ground cell, as float32.
PCT_HD float interval_value(float g, float c, const EvalConsts &K) {
  if (!finite32(c)) return 0.0f;  // open sky
  double d = (double)c - (double)g;
  double adapt = K.alpha_d * (K.d_ref - d);
  adapt = adapt > 0.0 ? adapt : 0.0;  // np.maximum(0.0, .)
  return (float)(d < K.d_min ? K.c_barrier : adapt);
}

// fuse_costs (traversability.py:162-170) for a valid ground cell.
PCT_HD float fuse_value(float ci, float cg, const EvalConsts &K) {
  double s = (double)ci + (double)cg;
  return (float)(K.c_barrier < s ? K.c_barrier : s);
}

// c_init of one cell given its terrain data and ceiling; float32 with the
// sign bit marking "becomes c_barrier unless the foothold count passes"
// (all costs are >= 0, and a foothold-branch value is > 0).
PCT_HD float cinit_encoded(float g, float ceil, const TerrainCell &t, const EvalConsts &K) {
  if (!t.valid) return (float)K.c_barrier;
  float ci = interval_value(g, ceil, K);
  bool needs_ps = false;
  double tv = t.isolated ? K.c_barrier : terrain_value(t.m_xy, t.m_grad, K, &needs_ps);
  float cg = (float)tv;
  float f = fuse_value(ci, cg, K);
  if (needs_ps) f = bits_f32(f32_bits(f) | 0x80000000u);
  return f;
}

// ---------------------------------------------------------------------------
// Fast exact path (used by the fused kernel).  glibc's hypot is
// h = RN(h0 - (t1+t2)/(2 h0)) with h0 = sqrt(ax*ax + ay*ay), i.e. within
// 1 ulp of h0.  The value of m_grad only matters (a) in the comparison
// m_grad < theta_s and (b) through float32(alpha_s * (m_grad/theta_s)^2) in
// the gentle branch.  (a) is decided from s = ax*ax + ay*ay outside a
// relative guard band of 2^-40 around theta_s^2; (b) is computed from h0 and
// accepted when the float64 cost lies farther than 2^-44 (relative) from a
// float32 rounding boundary, since h0 and h differ by < 2^-51 relative and
// the cost by < 2^-48.  Inside either band the exact glibc value is used.

// true if every double within rel*|x| of x rounds to the float f = RN32(x)
PCT_HD bool f32_round_safe(double x, float f, double rel) {
  if (x == 0.0) return true;
  uint32_t b = f32_bits(f) & 0x7FFFFFFFu;
  if (b == 0u || b >= 0x7F800000u - 1u) return false;
  const double fd = (double)(f < 0 ? -f : f);
  const double ax = x < 0 ? -x : x;
  const double r = ax - fd;  // exact: |r| <= ulp(f)/2
  const double up = (double)bits_f32(b + 1u) - fd;
  const double dn = fd - (double)bits_f32(b - 1u);
  const double half = 0.5 * (r >= 0.0 ? up : dn);
  return half - (r >= 0.0 ? r : -r) > rel * ax;
}

PCT_HD float gentle_cost_from(double m, const EvalConsts &K, double *cd) {
  const double q = div_const(m, K.theta_s, K.inv_theta_s);
  *cd = K.alpha_s * (q * q);
  return (float)*cd;
}

// float32 terrain cost of the gentle branch (m_grad < theta_s) for the
// gradient (gx, gy) with s = ax*ax + ay*ay, bit-identical to the reference.
// The cost from h0 = sqrt(s) is within 2^-48 (relative) of the cost from
// glibc's hypot; if both ends of the +-2^-44 interval round to the same
// float32, so does every value inside it (rounding is monotone).
PCT_HD float gentle_cost32(double gx, double gy, double s, const EvalConsts &K) {
  double cd;
  if (s == 0.0) return 0.0f;  // hypot(0, 0) = 0 exactly
  if (s > 0x1p-900) {         // away from the subnormal range sqrt(s) is within 1 ulp
    const float f = gentle_cost_from(sqrt(s), K, &cd);
    if ((float)(cd * (1.0 + 0x1p-44)) == f && (float)(cd * (1.0 - 0x1p-44)) == f) return f;
  }
  return gentle_cost_from(glibc_hypot(gx, gy), K, &cd);
}

// m_grad < theta_s from s, exact glibc hypot only inside the guard band
PCT_HD bool below_theta_s(double gx, double gy, double s, const EvalConsts &K) {
  if (s < K.ts2_lo) return true;
  if (s > K.ts2_hi) return false;
  return glibc_hypot(gx, gy) < K.theta_s;
}

struct FastCell {
  double gx, gy, s, m_xy;
  bool valid, isolated, gentle;
};

PCT_HD FastCell fast_terrain(const Cross &c, const EvalConsts &K) {
  FastCell t;
  const bool v = finite32(c.e), vl = finite32(c.l), vr = finite32(c.r), vu = finite32(c.u),
             vd = finite32(c.d);
  const double ef = v ? (double)c.e : 0.0;
  t.gx = axis_gradient(vr, vl, vr ? (double)c.r : 0.0, vl ? (double)c.l : 0.0, ef, K);
  t.gy = axis_gradient(vd, vu, vd ? (double)c.d : 0.0, vu ? (double)c.u : 0.0, ef, K);
  const double ax = fabs(t.gx), ay = fabs(t.gy);
  t.m_xy = ax > ay ? ax : ay;
  t.s = ax * ax + ay * ay;
  t.valid = v;
  t.isolated = v && !(vl || vr || vu || vd);
  t.gentle = v && below_theta_s(t.gx, t.gy, t.s, K);
  return t;
}

// c_init of a cell (same encoding as cinit_encoded) from the fast terrain data
PCT_HD float fast_cinit(float g, float ceil, const FastCell &t, const EvalConsts &K) {
  if (!t.valid) return (float)K.c_barrier;
  const float ci = interval_value(g, ceil, K);
  float cg;
  bool needs_ps = false;
  if (t.isolated || t.m_xy > K.theta_b) {
    cg = (float)K.c_barrier;
  } else if (t.gentle) {
    cg = gentle_cost32(t.gx, t.gy, t.s, K);
  } else {
    needs_ps = true;
    const double q = div_const(t.m_xy, K.theta_b, K.inv_theta_b);
    cg = (float)(K.alpha_b * (q * q));
  }
  float f = fuse_value(ci, cg, K);
  if (needs_ps) f = bits_f32(f32_bits(f) | 0x80000000u);
  return f;
}

// as cinit_resolve with the test count >= ps_min_count already decided
PCT_HD float cinit_resolve_ok(float enc, bool ok, const EvalConsts &K) {
  const uint32_t u = f32_bits(enc);
  if (u & 0x80000000u) return ok ? bits_f32(u & 0x7FFFFFFFu) : (float)K.c_barrier;
  return enc;
}

PCT_HD float cinit_resolve(float enc, int count, const EvalConsts &K) {
  uint32_t u = f32_bits(enc);
  if (u & 0x80000000u) return count >= K.ps_min_count ? bits_f32(u & 0x7FFFFFFFu)
                                                      : (float)K.c_barrier;
  return enc;
}

}  // namespace pct
