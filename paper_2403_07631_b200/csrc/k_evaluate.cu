// k_evaluate.cu — K4+K5: fused traversability stencil + inflation per slice.
// Replaces traversability.py:59-236 (interval_cost, slope_magnitudes,
// gentle_fraction, terrain_cost_values, ground_cost, fuse_costs, inflate,
// evaluate_slice / evaluate_tomogram).
//
// One CTA computes a TH x TW tile of c_T for one slice entirely on chip
// (DESIGN.md §4.2):
//   A  ground tile + halo (R + r + 1 cells) -> smem (NaN outside the grid)
//   B  per cell of the (TH+2R+2r)^2 "gentle" region: gradients, gentle flag
//      (exact glibc m_grad only inside a 2^-40 guard band); for the
//      (TH+2R)^2 c_init region also the interval cost and the fused cost,
//      the foothold branch marked in the sign bit
//   C  gentle flags packed to bits, one row of words per region row
//   D  foothold count over the (2r+1)^2 window by popcount -> p_s test as an
//      integer threshold -> final c_init
//   E  weighted max over the (2R+1)^2 kernel taps with zero padding:
//      max_t fl32(w_t * c_init) (== the reference's per-class max filter,
//      since x -> fl32(w*x) is monotone for w > 0).  8-fold symmetric
//      kernels with R <= 4 use a register sliding window of horizontal pair
//      maxima P_b(i,j) = max(c(i,j-b), c(i,j+b)); others loop over taps.
// eval_fast_kernel has the whole geometry as template constants (the common
// parameter sets); eval_generic_kernel takes it at run time and also serves
// the per-operation entry points.
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

constexpr int kMaxTaps = 125 * 125;
__constant__ float c_wfull[kMaxTaps];  // generic path: kside x kside weights
__constant__ float c_wsym[9 * 9];      // symmetric path: w[a][b], a,b in [0, R], stride 9
__constant__ EvalConsts c_K;

// ------------------------------------------------ stage E, symmetric, R<=4
// Thread = one output column x of a strip of V rows; register ring of the
// horizontal pair maxima of 2R+1 consecutive c_init rows.
// max of n values by a balanced tree of 3-input maxima (FMNMX3); exact and
// order-independent for non-NaN inputs
template <int N>
__device__ __forceinline__ float max_tree(const float (&v)[N]) {
  if constexpr (N == 1) {
    return v[0];
  } else if constexpr (N == 2) {
    return fmaxf(v[0], v[1]);
  } else {
    constexpr int M = (N + 2) / 3;
    float u[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const int a = 3 * i;
      u[i] = a + 2 < N ? fmaxf(fmaxf(v[a], v[a + 1]), v[a + 2])
                       : (a + 1 < N ? fmaxf(v[a], v[a + 1]) : v[a]);
    }
    return max_tree<M>(u);
  }
}

// The weighted max for output (c) of a strip from the pair-maxima ring: one
// product per tap group (a, b), a >= b.  Groups with weight <= 0 give a
// product <= 0, which cannot exceed the accumulator's start value 0 (the
// reference skips them; all c_init >= 0), so no group needs a branch and the
// whole reduction is a compile-time tree.
template <int R, int ROWS>
__device__ __forceinline__ float weighted_max(const float (&P)[ROWS][R + 1], int c) {
  constexpr int NP = (R + 1) * (R + 2) / 2 + 1;
  float v[NP];
  int n = 0;
#pragma unroll
  for (int a = 0; a <= R; ++a) {
#pragma unroll
    for (int b = 0; b <= a; ++b) {
      float m;
      if (a == 0) {
        m = P[c][0];
      } else if (b == 0) {
        m = fmaxf(fmaxf(P[c - a][0], P[c + a][0]), P[c][a]);
      } else if (a == b) {
        m = fmaxf(P[c - a][a], P[c + a][a]);
      } else {
        m = fmaxf(fmaxf(P[c - a][b], P[c + a][b]), fmaxf(P[c - b][a], P[c + b][a]));
      }
      v[n++] = c_wsym[a * 9 + b] * m;
    }
  }
  v[n] = 0.0f;
  return max_tree<NP>(v);
}

template <int R, int V>
__device__ __forceinline__ void inflate_sym_strip(const float *__restrict__ cinit, int CW,
                                                  int x, int ys, float *__restrict__ out,
                                                  int64_t out_stride, int orow0, int ocol,
                                                  int rows, int cols) {
  float P[V + 2 * R][R + 1];
#pragma unroll
  for (int t = 0; t < V + 2 * R; ++t) {
    const float *rowp = cinit + (ys + t) * CW + x;  // CI columns x .. x+2R
    P[t][0] = rowp[R];
#pragma unroll
    for (int b = 1; b <= R; ++b) P[t][b] = fmaxf(rowp[R - b], rowp[R + b]);
    if (t >= 2 * R) {
      const int o = t - 2 * R;  // output row in strip; centre P row = o + R
      const float acc = weighted_max<R, V + 2 * R>(P, o + R);
      const int gi = orow0 + o;
      if (gi < rows && ocol < cols) out[(int64_t)gi * out_stride + ocol] = acc;
    }
  }
}

// --------------------------------------- stage E, symmetric, 4 < R <= 8
// A (2R+1) x (R+1) ring does not fit in registers; the pair maxima P_b are
// split between two warp roles: LO owns b in [0, B0], HI owns b in
// [B0+1, R].  Every tap group (a, b) contributes w_ab * max(P_b(i+-a)) from
// the owner of b and w_ab * max(P_a(i+-b)) from the owner of a; since
// x -> fl32(w x) is monotone, max over both partials is the full result.
// The row loop is unrolled by template recursion (nvcc's #pragma unroll gives
// up on this body size and would move the ring to local memory).
template <int R, int BL, int NB, int V, int T>
__device__ __forceinline__ void half_step(float (&P)[V + 2 * R][NB], const float *__restrict__ cinit,
                                          int CW, int x, int ys, float *__restrict__ part,
                                          int pstride) {
  if constexpr (T < V + 2 * R) {
    const float *rowp = cinit + (ys + T) * CW + x;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int b = BL + j;
      P[T][j] = b == 0 ? rowp[R] : fmaxf(rowp[R - b], rowp[R + b]);
    }
    if constexpr (T >= 2 * R) {
      constexpr int o = T - 2 * R, c = o + R;
      float acc = 0.0f;
#pragma unroll
      for (int a = 0; a <= R; ++a) {
#pragma unroll
        for (int b = 0; b <= a; ++b) {
          const float w = c_wsym[a * 9 + b];
          if (w > 0.0f) {
            const bool own_b = b >= BL && b < BL + NB;
            const bool own_a = a >= BL && a < BL + NB;
            const int jb = own_b ? b - BL : 0, ja = own_a ? a - BL : 0;  // in-range indices
            float m = 0.0f;
            bool any = false;
            if (a == 0) {
              if (own_b) { m = P[c][jb]; any = true; }
            } else if (b == 0) {
              if (own_b) { m = fmaxf(P[c - a][jb], P[c + a][jb]); any = true; }
              if (own_a) { m = any ? fmaxf(m, P[c][ja]) : P[c][ja]; any = true; }
            } else if (a == b) {
              if (own_a) { m = fmaxf(P[c - a][ja], P[c + a][ja]); any = true; }
            } else {
              if (own_b) { m = fmaxf(P[c - a][jb], P[c + a][jb]); any = true; }
              if (own_a) {
                const float q = fmaxf(P[c - b][ja], P[c + b][ja]);
                m = any ? fmaxf(m, q) : q;
                any = true;
              }
            }
            if (any) acc = fmaxf(acc, w * m);
          }
        }
      }
      part[(ys + o) * pstride + x] = acc;
    }
    half_step<R, BL, NB, V, T + 1>(P, cinit, CW, x, ys, part, pstride);
  }
}

template <int R, int B0, int V, bool HI>
__device__ __forceinline__ void inflate_half_strip(const float *__restrict__ cinit, int CW, int x,
                                                   int ys, float *__restrict__ part, int pstride) {
  constexpr int BL = HI ? B0 + 1 : 0;
  constexpr int NB = HI ? R - B0 : B0 + 1;
  float P[V + 2 * R][NB];
  half_step<R, BL, NB, V, 0>(P, cinit, CW, x, ys, part, pstride);
}

// ------------------------------------------------------------- fast kernel
template <int R, int PR, int TH, int TW>
struct FastGeom {
  static constexpr int CH = TH + 2 * R, CW = TW + 2 * R;      // c_init region
  static constexpr int GH = CH + 2 * PR, GW = CW + 2 * PR;    // gentle region
  static constexpr int LH = GH + 2, LW = GW + 2;              // loaded ground
  static constexpr int H = R + PR + 1;                        // ground halo
  static constexpr int WORDS = (GW + 31) / 32 + 1;            // bit words per row (+1 pad)
  static constexpr int GWP = WORDS * 32;                      // padded u8 row
  static constexpr int OFF_GEN = LH * LW * 4;
  static constexpr int OFF_BITS = OFF_GEN + GH * GWP;
  static constexpr int OFF_FLIST = OFF_BITS + GH * WORDS * 4;  // u16 list of CI cells
  static constexpr int OFF_CINIT = (OFF_FLIST + CH * CW * 2 + 15) / 16 * 16;
  static constexpr int SMEM = OFF_CINIT + CH * CW * 4;
};

template <int R, int PR, int TH, int TW, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) eval_fast_kernel(const float *__restrict__ ground,
                                                       const float *__restrict__ ceiling,
                                                       int rows, int cols,
                                                       float *__restrict__ cost) {
  using G = FastGeom<R, PR, TH, TW>;
  extern __shared__ __align__(16) unsigned char smem[];
  float *grd = reinterpret_cast<float *>(smem);
  unsigned char *gen = smem + G::OFF_GEN;
  uint32_t *bits = reinterpret_cast<uint32_t *>(smem + G::OFF_BITS);
  float *cinit = reinterpret_cast<float *>(smem + G::OFF_CINIT);
  const int64_t plane = (int64_t)rows * cols;
  const int k = blockIdx.z;
  const int i0 = blockIdx.y * TH, j0 = blockIdx.x * TW;
  const float *gk = ground + k * plane;
  const float *ck = ceiling + k * plane;
  const float nanf_ = bits_f32(kNaNBits);
  const int tid = threadIdx.x;

  __shared__ int n_flagged;
  if (tid == 0) n_flagged = 0;
  // interior tiles (the common case) skip every grid-bounds test
  const bool interior = i0 - G::H >= 0 && j0 - G::H >= 0 && i0 + TH + G::H <= rows &&
                        j0 + TW + G::H <= cols;

  // A: ground tile + halo (NaN outside the grid); incremental 2D index
  {
    int y = tid / G::LW, x = tid - (tid / G::LW) * G::LW;
    const float *src = gk + (int64_t)(i0 - G::H) * cols + (j0 - G::H);
    for (int idx = tid; idx < G::LH * G::LW; idx += NT) {
      float v;
      if (interior) {
        v = __ldg(src + (int64_t)y * cols + x);
      } else {
        const int gi = i0 - G::H + y, gj = j0 - G::H + x;
        v = (gi >= 0 && gi < rows && gj >= 0 && gj < cols) ? __ldg(src + (int64_t)y * cols + x)
                                                           : nanf_;
      }
      grd[idx] = v;
      x += NT % G::LW;
      y += NT / G::LW;
      if (x >= G::LW) {
        x -= G::LW;
        ++y;
      }
    }
  }
  __syncthreads();

  // B: gentle flags over the gentle region, encoded c_init over the inner
  // region; foothold-branch cells are appended to a list for stage D
  uint16_t *flist = reinterpret_cast<uint16_t *>(bits + G::GH * G::WORDS);
  {
    int y = tid / G::GW, x = tid - (tid / G::GW) * G::GW;
    const float *crow = ck + (int64_t)(i0 - R) * cols + (j0 - R);  // CI origin
    for (int idx = tid; idx < G::GH * G::GW; idx += NT) {
      const int gi = i0 - R - PR + y, gj = j0 - R - PR + x;
      const bool in_grid = interior || (gi >= 0 && gi < rows && gj >= 0 && gj < cols);
      const bool in_ci = y >= PR && y < PR + G::CH && x >= PR && x < PR + G::CW;
      unsigned char gflag = 0;
      float enc = 0.0f;  // zero padding outside the map (inflate cval=0)
      if (in_grid) {
        const float *p = grd + (y + 1) * G::LW + (x + 1);
        const Cross c{p[0], p[-1], p[1], p[-G::LW], p[G::LW]};
        const FastCell t = fast_terrain(c, c_K);
        gflag = t.gentle ? 1 : 0;
        if (in_ci) {
          const float cv =
              t.valid ? __ldg(crow + (int64_t)(y - PR) * cols + (x - PR)) : nanf_;
          enc = fast_cinit(c.e, cv, t, c_K);
        }
      }
      gen[y * G::GWP + x] = gflag;
      const int ci_idx = (y - PR) * G::CW + (x - PR);
      const bool flagged = in_ci && (f32_bits(enc) & 0x80000000u);
      const unsigned act = __activemask();
      const unsigned fm = __ballot_sync(act, flagged);
      if (fm) {
        const int lane = tid & 31;
        const int leader = __ffs(fm) - 1;
        int base = 0;
        if (lane == leader) base = atomicAdd(&n_flagged, __popc(fm));
        base = __shfl_sync(act, base, leader);
        if (flagged) flist[base + __popc(fm & ((1u << lane) - 1u))] = (uint16_t)ci_idx;
      }
      if (in_ci) cinit[ci_idx] = enc;
      x += NT % G::GW;
      y += NT / G::GW;
      if (x >= G::GW) {
        x -= G::GW;
        ++y;
      }
    }
  }
  __syncthreads();

  // C: pack the flags, 32 cells per word (bytes past GW are masked off)
  for (int idx = tid; idx < G::GH * G::WORDS; idx += NT) {
    const int y = idx / G::WORDS, w = idx - y * G::WORDS;
    const int valid_bits = G::GW - w * 32;
    uint32_t word = 0;
    if (valid_bits > 0) {
      const uint32_t *src = reinterpret_cast<const uint32_t *>(gen + y * G::GWP + w * 32);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t v = src[q];  // 4 flags, one per byte
        word |= ((v & 1u) | ((v >> 7) & 2u) | ((v >> 14) & 4u) | ((v >> 21) & 8u)) << (4 * q);
      }
      if (valid_bits < 32) word &= (1u << valid_bits) - 1u;
    }
    bits[idx] = word;
  }
  __syncthreads();

  // D: foothold test p_s > theta_p  <=>  count >= ps_min_count, flagged cells only
  constexpr int SIDE = 2 * PR + 1;
  constexpr uint64_t MASK = (SIDE >= 64) ? ~0ull : ((1ull << SIDE) - 1ull);
  const int nf = n_flagged;
  for (int i = tid; i < nf; i += NT) {
    const int idx = flist[i];
    const int y = idx / G::CW, x = idx - y * G::CW;  // window rows y..y+2r, cols x..x+2r
    const int w = x >> 5, sh = x & 31;
    int cnt = 0;
#pragma unroll
    for (int d = 0; d < SIDE; ++d) {
      const uint32_t *rw = bits + (y + d) * G::WORDS + w;
      const uint64_t v = (uint64_t)rw[0] | ((uint64_t)rw[1] << 32);
      cnt += __popcll((v >> sh) & MASK);
    }
    cinit[idx] = cinit_resolve(cinit[idx], cnt, c_K);
  }
  __syncthreads();

  // E: inflation
  if constexpr (R <= 4) {
    constexpr int STRIPS = NT / TW;
    constexpr int V = TH / STRIPS;
    const int x = tid % TW, s = tid / TW;
    inflate_sym_strip<R, V>(cinit, G::CW, x, s * V, cost + k * plane, cols, i0 + s * V, j0 + x,
                            rows, cols);
  } else {
    // warps: [strip][role][column half]; partial maxima of both roles go to
    // the (now dead) ground region, then are merged and stored coalesced
    static_assert(TW == 64 && NT == 256, "split inflation layout");
    constexpr int V = TH / 2;
    const int warp = tid >> 5, lane = tid & 31;
    const int x = (warp & 1) * 32 + lane;
    const bool hi = (warp >> 1) & 1;
    const int s = warp >> 2;
    float *part_lo = grd;
    float *part_hi = grd + TH * TW;
    // two sub-strips of V/2 rows keep the fully unrolled ring in registers
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      if (hi)
        inflate_half_strip<R, R / 2, V / 2, true>(cinit, G::CW, x, s * V + h * (V / 2), part_hi,
                                                  TW);
      else
        inflate_half_strip<R, R / 2, V / 2, false>(cinit, G::CW, x, s * V + h * (V / 2), part_lo,
                                                   TW);
    }
    __syncthreads();
    float *out = cost + k * plane;
    for (int idx = tid; idx < TH * TW; idx += NT) {
      const int oy = idx / TW, ox = idx - oy * TW;
      const int gi = i0 + oy, gj = j0 + ox;
      if (gi < rows && gj < cols) out[(int64_t)gi * cols + gj] = fmaxf(part_lo[idx], part_hi[idx]);
    }
  }
}

// slices of DRAM -> L2 prefetch ahead of the terrain walk's register loads
// (prefetch.global.L2 holds no registers; the walk keeps one slice in
// registers): 4 measured best (cfg1 walk 96 -> 90 us, cfg2 524 -> 481 us;
// 2 and 8 close); PCT_WALK_L2PF=0 turns it off
int walk_l2_ahead_host() {
  const char *e = getenv("PCT_WALK_L2PF");
  return e ? atoi(e) : 4;
}

#include "k_eval_incr.cuh"
#include "k_eval_split.cuh"
#include "k_eval_bnb.cuh"

// ---------------------------------------------------------- generic kernel
struct TileGeom {
  int R, r;            // inflation radius, patch radius
  int TH, TW;          // output tile
  int CH, CW;          // c_init region = tile + R halo
  int GH, GW;          // gentle region = c_init region + r halo
  int LH, LW;          // loaded ground region = gentle region + 1
  int off_gen, off_hsum, off_cinit, smem;  // byte offsets
};

TileGeom make_geom(int R, int r, int TH, int TW) {
  TileGeom g;
  g.R = R;
  g.r = r;
  g.TH = TH;
  g.TW = TW;
  g.CH = TH + 2 * R;
  g.CW = TW + 2 * R;
  g.GH = g.CH + 2 * r;
  g.GW = g.CW + 2 * r;
  g.LH = g.GH + 2;
  g.LW = g.GW + 2;
  size_t o = (size_t)g.LH * g.LW * 4;
  g.off_gen = (int)o;
  o += ((size_t)g.GH * g.GW + 15) & ~(size_t)15;
  g.off_hsum = (int)o;
  o += (((size_t)g.GH * g.CW * 2) + 15) & ~(size_t)15;
  g.off_cinit = (int)o;
  o += (size_t)g.CH * g.CW * 4;
  g.smem = (int)o;
  return g;
}

// mode: kEvalFull (c_T), kEvalCinit (fused cost before inflation),
// kEvalGroundCost (ground_cost only), kEvalInterval (interval_cost only).
template <int NT>
__device__ __forceinline__ void stages_abcd(const TileGeom &G, const float *__restrict__ ground,
                                            const float *__restrict__ ceiling, int rows, int cols,
                                            int i0, int j0, int mode, unsigned char *smem) {
  float *grd = reinterpret_cast<float *>(smem);
  unsigned char *gen = smem + G.off_gen;
  uint16_t *hsum = reinterpret_cast<uint16_t *>(smem + G.off_hsum);
  float *cinit = reinterpret_cast<float *>(smem + G.off_cinit);
  const float nanf_ = bits_f32(kNaNBits);
  const int H = G.R + G.r + 1;
  const int tid = threadIdx.x;

  for (int idx = tid; idx < G.LH * G.LW; idx += NT) {
    const int y = idx / G.LW, x = idx - y * G.LW;
    const int gi = i0 - H + y, gj = j0 - H + x;
    float v = nanf_;
    if (gi >= 0 && gi < rows && gj >= 0 && gj < cols) v = __ldg(ground + (int64_t)gi * cols + gj);
    grd[idx] = v;
  }
  __syncthreads();

  const int rr = G.r;
  for (int idx = tid; idx < G.GH * G.GW; idx += NT) {
    const int y = idx / G.GW, x = idx - y * G.GW;
    const int gi = i0 - G.R - rr + y, gj = j0 - G.R - rr + x;
    const bool in_grid = gi >= 0 && gi < rows && gj >= 0 && gj < cols;
    const bool in_ci = y >= rr && y < rr + G.CH && x >= rr && x < rr + G.CW;
    unsigned char gflag = 0;
    float enc = 0.0f;
    if (in_grid) {
      const float *p = grd + (y + 1) * G.LW + (x + 1);
      Cross c{p[0], p[-1], p[1], p[-G.LW], p[G.LW]};
      TerrainCell t = terrain_cell(c, c_K);
      gflag = t.gentle ? 1 : 0;
      if (in_ci) {
        if (mode == kEvalInterval) {
          enc = t.valid ? interval_value(c.e, __ldg(ceiling + (int64_t)gi * cols + gj), c_K)
                        : (float)c_K.c_barrier;
        } else if (mode == kEvalGroundCost) {
          bool needs_ps = false;
          if (t.valid) {
            double tv = t.isolated ? c_K.c_barrier
                                   : terrain_value(t.m_xy, t.m_grad, c_K, &needs_ps);
            enc = (float)tv;
            if (needs_ps) enc = bits_f32(f32_bits(enc) | 0x80000000u);
          }
        } else {
          const float ceil_v = t.valid ? __ldg(ceiling + (int64_t)gi * cols + gj) : nanf_;
          enc = cinit_encoded(c.e, ceil_v, t, c_K);
        }
      }
    }
    gen[idx] = gflag;
    if (in_ci) cinit[(y - rr) * G.CW + (x - rr)] = enc;
  }
  __syncthreads();

  const int side = 2 * rr + 1;
  for (int idx = tid; idx < G.GH * G.CW; idx += NT) {
    const int y = idx / G.CW, x = idx - y * G.CW;
    const unsigned char *g = gen + y * G.GW + x;
    int s = 0;
    for (int d = 0; d < side; ++d) s += g[d];
    hsum[idx] = (uint16_t)s;
  }
  __syncthreads();

  for (int idx = tid; idx < G.CH * G.CW; idx += NT) {
    const float enc = cinit[idx];
    if (f32_bits(enc) & 0x80000000u) {
      const int y = idx / G.CW, x = idx - y * G.CW;
      int cnt = 0;
      for (int d = 0; d < side; ++d) cnt += hsum[(y + d) * G.CW + x];
      cinit[idx] = cinit_resolve(enc, cnt, c_K);
    }
  }
  __syncthreads();
}

template <int NT>
__device__ __forceinline__ void inflate_generic(const TileGeom &G, const float *__restrict__ cinit,
                                                int kside, float *__restrict__ out, int rows,
                                                int cols, int i0, int j0) {
  for (int idx = threadIdx.x; idx < G.TH * G.TW; idx += NT) {
    const int oy = idx / G.TW, ox = idx - oy * G.TW;
    const int gi = i0 + oy, gj = j0 + ox;
    if (gi >= rows || gj >= cols) continue;
    float acc = 0.0f;
    for (int m = 0; m < kside; ++m) {
      const float *rowp = cinit + (oy + m) * G.CW + ox;
      for (int n = 0; n < kside; ++n) {
        const float w = c_wfull[m * kside + n];
        if (w > 0.0f) acc = fmaxf(acc, w * rowp[n]);
      }
    }
    out[(int64_t)gi * cols + gj] = acc;
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) eval_generic_kernel(TileGeom G,
                                                          const float *__restrict__ ground,
                                                          const float *__restrict__ ceiling,
                                                          int rows, int cols, int kside, int mode,
                                                          float *__restrict__ cost) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int64_t plane = (int64_t)rows * cols;
  const int k = blockIdx.z;
  const int i0 = blockIdx.y * G.TH, j0 = blockIdx.x * G.TW;
  stages_abcd<NT>(G, ground + k * plane, ceiling ? ceiling + k * plane : nullptr, rows, cols, i0,
                  j0, mode, smem);
  const float *cinit = reinterpret_cast<const float *>(smem + G.off_cinit);
  float *out = cost + k * plane;
  if (mode == kEvalFull) {
    inflate_generic<NT>(G, cinit, kside, out, rows, cols, i0, j0);
  } else {
    for (int idx = threadIdx.x; idx < G.TH * G.TW; idx += NT) {
      const int oy = idx / G.TW, ox = idx - oy * G.TW;
      const int gi = i0 + oy, gj = j0 + ox;
      if (gi < rows && gj < cols) out[(int64_t)gi * cols + gj] = cinit[(oy + G.R) * G.CW + ox + G.R];
    }
  }
}

// standalone inflate (traversability.py:205-213) for the per-op API
template <int NT>
__global__ void __launch_bounds__(NT) inflate_kernel(TileGeom G, const float *__restrict__ in,
                                                     int rows, int cols, int kside,
                                                     float *__restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  float *cinit = reinterpret_cast<float *>(smem + G.off_cinit);
  const int i0 = blockIdx.y * G.TH, j0 = blockIdx.x * G.TW;
  for (int idx = threadIdx.x; idx < G.CH * G.CW; idx += NT) {
    const int y = idx / G.CW, x = idx - y * G.CW;
    const int gi = i0 - G.R + y, gj = j0 - G.R + x;
    cinit[idx] = (gi >= 0 && gi < rows && gj >= 0 && gj < cols) ? __ldg(in + (int64_t)gi * cols + gj)
                                                                 : 0.0f;
  }
  __syncthreads();
  inflate_generic<NT>(G, cinit, kside, out, rows, cols, i0, j0);
}

// ---------------------------------------------------------------- host side
bool symmetric_kernel(const float *w, int kside, int R, float wsym[81]) {
  if (R > 8) return false;
  for (int i = 0; i < 81; ++i) wsym[i] = 0.0f;
  for (int a = 0; a <= R; ++a)
    for (int b = 0; b <= a; ++b) wsym[a * 9 + b] = w[(R + a) * kside + (R + b)];
  for (int m = 0; m < kside; ++m)
    for (int n = 0; n < kside; ++n) {
      int a = std::abs(m - R), b = std::abs(n - R);
      if (a < b) std::swap(a, b);
      const float v = w[m * kside + n];
      if (std::memcmp(&v, &wsym[a * 9 + b], 4) != 0) return false;
    }
  return true;
}

int ps_min_count(double theta_p, int radius) {
  const int side = 2 * radius + 1;
  const double div = (double)(side * side);
  for (int c = 0; c <= side * side; ++c)
    if ((double)c / div > theta_p) return c;
  return side * side + 1;
}

constexpr int kNT = 256;

// slice-incremental kernel: runs of consecutive slices per CTA, run length
// chosen so the grid still fills ~2 waves of 2 CTAs per SM
template <int R, int PR, int TH, int TW, int NT, int MINB>
int launch_incr_t(pct_ctx *ctx, const float *ground, const float *ceiling, int S, int rows,
                  int cols, float *cost) {
  auto kern = eval_incr_kernel<R, PR, TH, TW, NT, MINB>;
  constexpr int smem = IncrGeom<R, PR, TH, TW>::SMEM;
  PCT_CUDA(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int tx = (cols + TW - 1) / TW, ty = (rows + TH - 1) / TH;
  const int64_t tiles = (int64_t)tx * ty;
  int per_sm = 0;
  PCT_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
  const int64_t slots = (int64_t)std::max(1, per_sm) * ctx->num_sms;  // resident CTAs
  // runs of 12 slices (measured best on cfg1), shorter if the grid would
  // otherwise not get ~2 work items per resident CTA
  int run = 12;
  while (run > 4 && tiles * ((S + run - 1) / run) < 2 * slots) run /= 2;
  if (const char *e = getenv("PCT_EVAL_RUN")) run = std::max(1, atoi(e));
  run = std::min(run, S);
  const int64_t items = tiles * ((S + run - 1) / run);
  if (items > INT32_MAX || tiles > INT32_MAX) return fail(ctx, PCT_E_INVALID, "grid too large");
  int *counter = reinterpret_cast<int *>(static_cast<char *>(ctx->dsmall) + 65536 - 64);
  PCT_CUDA(ctx, cudaMemsetAsync(counter, 0, sizeof(int), ctx->stream));
  const unsigned grid = (unsigned)std::min<int64_t>(items, slots);
  kern<<<grid, NT, smem, ctx->stream>>>(ground, ceiling, rows, cols, S, run, tx, (int)tiles,
                                        (int)items, counter, cost);
  return check_launch(ctx, "eval_incr_kernel");
}

// two-kernel evaluation (k_eval_split.cuh): per-cell slice walk, then tiled
// foothold resolution + inflation; intermediates in the context scratch.
// Inflation: the branch-and-bound kernel (k_eval_bnb.cuh) when the kernel's
// weight classes fit its compiled disk (PCT_INFL=sym keeps the full-tap TMA
// kernel for R <= 4), else the full-tap TMA kernel (R <= 4 only).
// resident CTAs the bnb kernel is compiled for (caps its registers): R = 4
// tiles need ~34 KB of shared memory (6 CTAs fit), R = 8 ~47 KB (4 fit)
template <int R>
constexpr int kBnbMinBlocks() {
  return R <= 4 ? 6 : 4;
}
// the sparse-merge instantiation: its shared memory allows 5 CTAs per SM at
// R = 4, so it may use the registers of 5 (the change-map prefetch lives in
// them)
#ifndef PCT_BNB_TH
#define PCT_BNB_TH 24  // output tile rows of the R = 4 bnb evaluation
#endif
#ifndef PCT_BNB_SP_MINB
#define PCT_BNB_SP_MINB 5
#endif
template <int R>
constexpr int kBnbMinBlocksSp() {
  return R <= 4 ? PCT_BNB_SP_MINB : 4;
}

template <int R, int PR, int TH, int TW, int BNT = 256>
int launch_split(pct_ctx *ctx, const float *ground, const float *ceiling, int S, int rows,
                 int cols, const float *kernel_w, int kside, float *cost, bool bnb) {
  ConstBank cb(ctx);  // nested in launch_evaluate's scope: c_bw joins its constants
  const int64_t cells = (int64_t)rows * cols;
  const int wpr = (cols + 31) / 32;
  const int64_t words = (int64_t)rows * wpr;  // gentle bitmap words per slice
  std::vector<float> bw;
  if constexpr (R == 4 || R == 8) {
    if (bnb && !bnb_tables<R>(kernel_w, kside, bw)) bnb = false;
  } else {
    bnb = false;
  }
  if (!bnb && R > 4) return fail(ctx, PCT_E_INVALID, "split evaluation needs the bnb tables for R > 4");
  EncLayout L;
  L.padr = R;
  L.padc = R;
  L.prows = (rows + TH - 1) / TH * TH + 2 * R;
  L.pitch = ((int64_t)((cols + TW - 1) / TW * TW + 2 * R) + 3) / 4 * 4;
  L.sstride = (int64_t)L.prows * L.pitch;
  const size_t enc_bytes = (size_t)S * L.sstride * 4;
  // gentle bitmap | (bnb) descriptor of a batch of one | walk change map
  const size_t cm_off = (((size_t)S * words * 4 + 255) / 256) * 256 + ((sizeof(EvalMap) + 128 + 255) / 256) * 256;
  const size_t cm_bytes = (size_t)S * ((rows + 7) / 8) * wpr;
  // then the walk's input-change masks (2 x 8 B per cell, S <= 64) and its
  // fresh map (sparse output: one byte per slice, row and bitmap word)
  const size_t m_off = ((cm_off + cm_bytes + 64 + 255) / 256) * 256;
  const int fpitch = (wpr + 15) & ~15;
  const size_t f_off = m_off + (S <= 64 ? 2 * (size_t)cells * 8 : 0);
  const size_t f_bytes = S <= 64 ? (size_t)S * rows * fpitch : 0;
  if (int rc = ensure_scratch(ctx, f_off + f_bytes)) return rc;
  uint32_t *bits = static_cast<uint32_t *>(ctx->scratch);
  // tiles whose window saw no change skip the resolve/inflate work: cfg2
  // (R = 8) bnb 798 -> 473 us, cfg3 (R = 4, open campus) 3.22 -> 2.00 ms;
  // cfg1 about neutral (the change map costs the walk ~5 us).  PCT_BNB_SKIP=0
  // turns it off.
  const char *skv = getenv("PCT_BNB_SKIP");
  const bool use_skip = skv ? skv[0] == '1' : true;
  unsigned char *chgmap = use_skip ? static_cast<unsigned char *>(ctx->scratch) + cm_off : nullptr;
  if (chgmap) PCT_CUDA(ctx, cudaMemsetAsync(chgmap, 0, cm_bytes, ctx->stream));
  if (ctx->enc_bytes < enc_bytes) {
    if (ctx->enc) {
      cudaStreamSynchronize(ctx->stream);
      cudaFree(ctx->enc);
      ctx->enc = nullptr;
      ctx->enc_bytes = 0;
    }
    PCT_CUDA(ctx, cudaMalloc(&ctx->enc, enc_bytes));
    ctx->enc_bytes = enc_bytes;
    ctx->enc_tag[0] = -1;
  }
  float *enc = static_cast<float *>(ctx->enc);
  const int64_t tag[6] = {S, rows, cols, R, TH, TW};
  if (!std::equal(tag, tag + 6, ctx->enc_tag)) {  // new layout: clear its padding once
    zero_pads_kernel<<<dim3((unsigned)L.prows, S), 128, 0, ctx->stream>>>(enc, L, rows, cols);
    if (int rc = check_launch(ctx, "zero_pads_kernel")) return rc;
    std::copy(tag, tag + 6, ctx->enc_tag);
  }
  const int64_t walk_threads = (int64_t)rows * wpr * 32;
  const unsigned g1 = (unsigned)((walk_threads + kWalkNT - 1) / kWalkNT);
  const char *pf = getenv("PCT_WALK_PF");
  const int l2d = walk_l2_ahead_host();
  // slice chunks: a small map gets ~2 waves of threads by walking its slices
  // in up to 4 independent chunks (each chunk's first slice in full); large
  // maps fill the GPU with one chunk (PCT_WALK_CHUNKS overrides)
  int chunks = 1;
  {
    const int64_t resident = (int64_t)ctx->num_sms * 2048;
    const int64_t threads = (int64_t)g1 * kWalkNT;
    while (chunks < 4 && threads * chunks * 2 <= 2 * resident && S >= 6 * (chunks * 2)) chunks *= 2;
    if (const char *e = getenv("PCT_WALK_CHUNKS")) chunks = std::max(1, std::min(S, atoi(e)));
  }
  // the resolve / inflate kernel's slices per work item: long runs reuse the
  // previous slice (only the first slice of a run is computed in full); the
  // longest run that still gives every resident CTA ~3 items (small maps:
  // down to one slice per item; cfg0 evaluate 44 -> 36 us, cfg1 unchanged at 5)
  int bnb_run = 1, bnb_slots = 1;
  bool sparse = false;
  const char *wk = getenv("PCT_WALK");
  const bool skip_walk = S <= 64 && !(wk && wk[0] == '1');
  if constexpr (R == 4 || R == 8) {
    if (bnb) {
      auto plan = [&](auto kb, int bsmem) -> int {
        PCT_CUDA(ctx, cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, bsmem));
        int per_sm = 0;
        PCT_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kb, BNT, bsmem));
        bnb_slots = (int)std::max(1, per_sm) * ctx->num_sms;
        const int64_t tiles = (int64_t)((cols + TW - 1) / TW) * ((rows + TH - 1) / TH);
        const int64_t runs_per_tile =
            std::min<int64_t>(S, (3 * (int64_t)bnb_slots + tiles - 1) / tiles);
        bnb_run = (int)((S + runs_per_tile - 1) / runs_per_tile);
        if (const char *e = getenv("PCT_INFL_RUN")) bnb_run = std::max(1, atoi(e));
        bnb_run = std::min(std::min(bnb_run, S), 64);  // per-item skip mask: 64 slices
        return PCT_OK;
      };
      if (int rc = plan(resolve_inflate_bnb_kernel<R, PR, TH, TW, BNT, kBnbMinBlocks<R>()>,
                        BnbGeom<R, PR, TH, TW>::SMEM))
        return rc;
      // sparse walk output (merged by the bnb kernel) pays off when the
      // kernel's items are long runs of slices and its merge buffers cost no
      // more than one resident CTA: R = 4 (cfg3 evaluate 3.32 -> 2.88 ms);
      // short runs re-write every run start anyway (cfg1: 0.179 dense vs
      // 0.193 ms); at R = 8 the buffers drop the kernel from 4 to 3 CTAs per
      // SM (cfg2: 0.74 dense vs 0.84 ms)
      const char *spv = getenv("PCT_WALK_SPARSE");
      sparse = skip_walk && chgmap && (spv ? spv[0] == '1' : (R == 4 && bnb_run >= 16));
      if (sparse)
        if (int rc = plan(resolve_inflate_bnb_kernel<R, PR, TH, TW, BNT, kBnbMinBlocksSp<R>(), true>,
                          BnbGeom<R, PR, TH, TW, true>::SMEM))
          return rc;
    }
  }
  unsigned char *fresh = nullptr;
  if (skip_walk) {
    if (sparse) {
      fresh = static_cast<unsigned char *>(ctx->scratch) + f_off;
      PCT_CUDA(ctx, cudaMemsetAsync(fresh, 0, f_bytes, ctx->stream));
    }
    // input-change masks, then the walk that skips the slices where none of
    // a warp's inputs changed
    const unsigned long long *gm = ctx->eval_masks, *cmk = nullptr;
    if (gm) {  // written by the build of these stacks
      cmk = gm + cells;
    } else {
      unsigned long long *m = reinterpret_cast<unsigned long long *>(
          static_cast<char *>(ctx->scratch) + m_off);
      change_mask_kernel<<<(unsigned)((cells + kMaskNT - 1) / kMaskNT), kMaskNT, 0, ctx->stream>>>(
          ground, ceiling, S, cells, m, m + cells);
      if (int rc = check_launch(ctx, "change_mask_kernel")) return rc;
      gm = m;
      cmk = m + cells;
    }
    unsigned long long runmask = 0ull;  // slices k with k % bnb_run == 0 (S <= 64 here)
    if (bnb_run > 0)
      for (int k = 0; k < S && k < 64; k += bnb_run) runmask |= 1ull << k;
    if (chunks > 1)
      terrain_walk_skip_kernel<true><<<dim3(g1, chunks), kWalkNT, 0, ctx->stream>>>(
          ground, ceiling, S, rows, cols, enc, L, bits, wpr, chgmap, gm, cmk, fresh, fpitch,
          runmask);
    else
      terrain_walk_skip_kernel<false><<<g1, kWalkNT, 0, ctx->stream>>>(
          ground, ceiling, S, rows, cols, enc, L, bits, wpr, chgmap, gm, cmk, fresh, fpitch,
          runmask);
  } else
  // one slice of look-ahead measured fastest (cfg1 85 us vs 105 / 132 for
  // 2 / 4; deeper prefetch costs occupancy)
  if (pf && pf[0] == '2')
    terrain_walk_kernel<2><<<g1, kWalkNT, 0, ctx->stream>>>(ground, ceiling, S, rows, cols, enc, L,
                                                           bits, wpr, chgmap, l2d);
  else
    if (chunks > 1)
      terrain_walk_kernel<1, true><<<dim3(g1, chunks), kWalkNT, 0, ctx->stream>>>(
          ground, ceiling, S, rows, cols, enc, L, bits, wpr, chgmap, l2d);
    else
      terrain_walk_kernel<1><<<g1, kWalkNT, 0, ctx->stream>>>(ground, ceiling, S, rows, cols, enc,
                                                             L, bits, wpr, chgmap, l2d);
  if (int rc = check_launch(ctx, "terrain_walk_kernel")) return rc;
  const char *tma = getenv("PCT_TMA");
  if (bnb || (!(tma && tma[0] == '0') && R % 4 == 0)) {
    // persistent TMA-pipelined resolve + inflate: a 3-D tensor map over the
    // padded stacks, box = one c_init tile + halo
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
      void *fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      PCT_CUDA(ctx, cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
      if (!fn || q != cudaDriverEntryPointSuccess)
        return fail(ctx, PCT_E_CUDA, "cuTensorMapEncodeTiled unavailable");
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    constexpr int CH = TH + 2 * R, CW = TW + 2 * R;
    CUtensorMap map;
    const cuuint64_t dims[3] = {(cuuint64_t)L.pitch, (cuuint64_t)L.prows, (cuuint64_t)S};
    const cuuint64_t strides[2] = {(cuuint64_t)L.pitch * 4, (cuuint64_t)L.sstride * 4};
    const cuuint32_t box[3] = {(cuuint32_t)CW, (cuuint32_t)CH, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    if (encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, enc, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return fail(ctx, PCT_E_CUDA, "cuTensorMapEncodeTiled failed");
    const int64_t items = (int64_t)((cols + TW - 1) / TW) * ((rows + TH - 1) / TH) * S;
    if (items > INT32_MAX) return fail(ctx, PCT_E_INVALID, "grid too large");
    if constexpr (R == 4 || R == 8) {
     if (bnb) {
      PCT_CUDA(ctx, cb.set_symbol(c_bw, bw.data(), bw.size() * sizeof(float)));
      auto kb = sparse ? resolve_inflate_bnb_kernel<R, PR, TH, TW, BNT, kBnbMinBlocksSp<R>(), true>
                       : resolve_inflate_bnb_kernel<R, PR, TH, TW, BNT, kBnbMinBlocks<R>()>;
      const int bsmem = sparse ? BnbGeom<R, PR, TH, TW, true>::SMEM : BnbGeom<R, PR, TH, TW>::SMEM;
      const int64_t slots = bnb_slots;
      const int64_t tiles = (int64_t)((cols + TW - 1) / TW) * ((rows + TH - 1) / TH);
      const int run = bnb_run;
      const int64_t nitems = tiles * ((S + run - 1) / run);
      if (nitems > INT32_MAX) return fail(ctx, PCT_E_INVALID, "grid too large");
      const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nitems, slots));
      // a batch of one: the descriptor (with its tensor map) and the item
      // offsets behind the gentle bitmap in the scratch (64-byte aligned)
      const size_t boff = (((size_t)S * words * 4 + 255) / 256) * 256;
      EvalMap hm;
      std::memset(&hm, 0, sizeof(hm));
      hm.tmap = map;
      hm.ground = ground;
      hm.ceiling = ceiling;
      hm.enc = enc;
      hm.cost = cost;
      hm.bits = bits;
      hm.L = L;
      hm.S = S;
      hm.rows = rows;
      hm.cols = cols;
      hm.wpr = wpr;
      hm.run = run;
      hm.words = words;
      hm.chg = chgmap;
      hm.fresh = fresh;
      hm.fpitch = fpitch;
      if (ctx->eval_tcm && S <= 64) {  // per-tile cost-change masks for the simplify window
        PCT_CUDA(ctx, cudaMemsetAsync(ctx->eval_tcm, 0, (size_t)tiles * 8, ctx->stream));
        hm.tcm = ctx->eval_tcm;
        ctx->eval_tcm_written = true;
        ctx->tcm_th = TH;
        ctx->tcm_tw = TW;
      }
      // output tiles by TMA bulk stores when the cost rows are 16-byte pitched
      const char *tsv = getenv("PCT_BNB_TMA_STORE");
      if ((cols & 3) == 0 && (reinterpret_cast<uintptr_t>(cost) & 15) == 0 &&
          !(tsv && tsv[0] == '0')) {
        const cuuint64_t odims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)S};
        const cuuint64_t ostr[2] = {(cuuint64_t)cols * 4, (cuuint64_t)cols * rows * 4};
        const cuuint32_t obox[3] = {(cuuint32_t)TW, (cuuint32_t)TH, 1};
        if (encode(&hm.omap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, cost, odims, ostr, obox, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
          hm.ostore = 1;
      }
      struct {
        EvalMap m;
        int off[2];
        int work;  // dynamic item counter (PCT_BNB_DYNAMIC=0: static round robin)
      } desc;
      static_assert(offsetof(decltype(desc), m) == 0, "descriptor layout");
      desc.m = hm;
      desc.off[0] = 0;
      desc.off[1] = (int)nitems;
      desc.work = 0;
      const char *dyv = getenv("PCT_BNB_DYNAMIC");
      const bool dyn = !(dyv && dyv[0] == '0');
      char *dptr = static_cast<char *>(ctx->scratch) + boff;
      PCT_CUDA(ctx, upload_async(ctx, dptr, &desc, sizeof(desc)));
      const EvalMap *dm = reinterpret_cast<const EvalMap *>(dptr);
      const int *doff = reinterpret_cast<const int *>(dptr + offsetof(decltype(desc), off));
      int *dwork = reinterpret_cast<int *>(dptr + offsetof(decltype(desc), work));
      kb<<<grid, BNT, bsmem, ctx->stream>>>(dm, doff, 1, dyn ? dwork : nullptr);
      return check_launch(ctx, "resolve_inflate_bnb_kernel");
     }
    }
    if constexpr (R <= 4 && R % 4 == 0) {
      using TG = TmaGeom<R, PR, TH, TW>;
      auto kt = resolve_inflate_tma_kernel<R, PR, TH, TW, kNT, 3>;
      constexpr int tsmem = TG::SMEM;
      PCT_CUDA(ctx, cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, tsmem));
      int per_sm = 0;
      PCT_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kt, kNT, tsmem));
      const unsigned grid = (unsigned)std::max<int64_t>(
          1, std::min<int64_t>(items, (int64_t)std::max(1, per_sm) * ctx->num_sms));
      kt<<<grid, kNT, tsmem, ctx->stream>>>(map, bits, rows, cols, S, words, cost);
      return check_launch(ctx, "resolve_inflate_tma_kernel");
    }
  }
  if constexpr (R <= 4) {
    auto kern = resolve_inflate_kernel<R, PR, TH, TW, kNT, 3>;
    constexpr int smem = SplitGeom<R, PR, TH, TW>::SMEM;
    PCT_CUDA(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    dim3 grid((cols + TW - 1) / TW, (rows + TH - 1) / TH, S);
    kern<<<grid, kNT, smem, ctx->stream>>>(enc, L, bits, rows, cols, words, cost);
    return check_launch(ctx, "resolve_inflate_kernel");
  }
  return fail(ctx, PCT_E_INVALID, "no resolve/inflate kernel for this radius");
}

// Kernel choice for symmetric kernels with compiled geometry: the two-kernel
// split by default (R = 8 only when the bnb tables fit); PCT_EVAL_KERNEL=fast
// selects the fused per-slice kernel and =incr (R <= 4) the slice-incremental
// CTA kernel (kept as measured alternatives; PCT_EVAL_TILE /
// PCT_EVAL_RUN tune it).
template <int R, int PR>
int launch_fast(pct_ctx *ctx, const float *ground, const float *ceiling, int S, int rows,
                int cols, const float *kernel_w, int kside, float *cost) {
  const char *m = getenv("PCT_EVAL_KERNEL");
  const char *infl = getenv("PCT_INFL");
  const char *tile = getenv("PCT_BNB_TILE");
  const bool alt = tile && tile[0] == '1';
  std::vector<float> bw;
  bool bnb = false;
  if constexpr (R == 4 || R == 8) bnb = !(infl && infl[0] == 's') && bnb_tables<R>(kernel_w, kside, bw);
  if (!m || m[0] == 's') {
    // default: the two-kernel split (terrain walk + resolve/inflate)
    if constexpr (R == 4) {
      if (bnb && alt)
        return launch_split<R, PR, 32, 64, 128>(ctx, ground, ceiling, S, rows, cols, kernel_w, kside, cost, true);
      // 24 x 32 output tiles (measured against 32 x 32: cfg3 evaluate 2.525 ->
      // 2.474 ms and simplify 0.682 -> 0.665 (finer tile change masks), cfg1
      // evaluate 0.172 -> 0.167 ms; 16 x 32 with 6 CTAs per SM: 2.525 / 0.657)
      if (bnb)
        return launch_split<R, PR, PCT_BNB_TH, 32, 128>(ctx, ground, ceiling, S, rows, cols, kernel_w, kside, cost, true);
    }
    if constexpr (R == 8) {
      if (bnb && alt)
        return launch_split<R, PR, 64, 32, 256>(ctx, ground, ceiling, S, rows, cols, kernel_w, kside, cost, true);
      if (bnb)
        return launch_split<R, PR, 32, 32, 128>(ctx, ground, ceiling, S, rows, cols, kernel_w, kside, cost, true);
    }
    if constexpr (R <= 4)
      return launch_split<R, PR, 64, 64>(ctx, ground, ceiling, S, rows, cols, kernel_w, kside, cost, false);
  }
  if constexpr (R <= 4) {
    if (m && m[0] == 'i' && S > 1) {
      const char *t = getenv("PCT_EVAL_TILE");
      if (t && atoi(t) == 64)
        return launch_incr_t<R, PR, 64, 64, 256, 2>(ctx, ground, ceiling, S, rows, cols, cost);
      if (t && atoi(t) == 16)
        return launch_incr_t<R, PR, 16, 32, 64, 8>(ctx, ground, ceiling, S, rows, cols, cost);
      return launch_incr_t<R, PR, 32, 32, 128, 4>(ctx, ground, ceiling, S, rows, cols, cost);
    }
  }
  constexpr int TH = 64, TW = 64;
  auto kern = eval_fast_kernel<R, PR, TH, TW, kNT, (R <= 4 ? 3 : 2)>;
  constexpr int smem = FastGeom<R, PR, TH, TW>::SMEM;
  PCT_CUDA(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  dim3 grid((cols + TW - 1) / TW, (rows + TH - 1) / TH, S);
  kern<<<grid, kNT, smem, ctx->stream>>>(ground, ceiling, rows, cols, cost);
  return check_launch(ctx, "eval_fast_kernel");
}

}  // namespace

EvalConsts make_consts(const pct_trav_params &p, double r_g) {
  EvalConsts K;
  K.d_min = p.d_min;
  K.d_ref = p.d_ref;
  K.theta_b = p.theta_b;
  K.theta_s = p.theta_s;
  K.c_barrier = p.c_barrier;
  K.alpha_d = p.alpha_d;
  K.alpha_b = p.alpha_b;
  K.alpha_s = p.alpha_s;
  K.rg = r_g;
  K.inv_rg = 1.0 / r_g;
  K.two_rg = 2.0 * r_g;
  K.inv_two_rg = 1.0 / K.two_rg;
  K.inv_theta_b = 1.0 / p.theta_b;
  K.inv_theta_s = 1.0 / p.theta_s;
  K.ts2_lo = p.theta_s * p.theta_s * (1.0 - 0x1p-40);
  K.ts2_hi = p.theta_s * p.theta_s * (1.0 + 0x1p-40);
  K.patch_radius = p.patch_radius;
  K.ps_min_count = ps_min_count(p.theta_p, p.patch_radius);
  return K;
}

int launch_evaluate(pct_ctx *ctx, const float *ground, const float *ceiling, int S, int rows,
                    int cols, double r_g, const pct_trav_params &p, const float *kernel_w,
                    int kside, float *cost, int mode) {
  if (S <= 0 || rows <= 0 || cols <= 0) return PCT_OK;
  if (p.patch_radius < 0 || p.patch_radius > 60)
    return fail(ctx, PCT_E_INVALID, "patch radius out of supported range [0, 60]");
  int R = 0;
  if (mode == kEvalFull) {
    if (kside <= 0 || (kside & 1) == 0 || kside * kside > kMaxTaps)
      return fail(ctx, PCT_E_INVALID, "inflation kernel side must be odd and <= 125");
    R = kside / 2;
  }
  ConstBank cb(ctx);
  EvalConsts K = make_consts(p, r_g);
  PCT_CUDA(ctx, cb.set_symbol(c_K, &K, sizeof(K)));
  float wsym[81];
  const bool sym = mode == kEvalFull && symmetric_kernel(kernel_w, kside, R, wsym);
  if (mode == kEvalFull) {
    if (sym)
      PCT_CUDA(ctx, cb.set_symbol(c_wsym, wsym, sizeof(wsym)));
    else
      PCT_CUDA(ctx, cb.set_symbol(c_wfull, kernel_w, sizeof(float) * kside * kside));
  }
  if (sym && R == 4 && p.patch_radius == 3)  // r_g = 0.1 with the Table-I radii
    return launch_fast<4, 3>(ctx, ground, ceiling, S, rows, cols, kernel_w, kside, cost);
  if (sym && R == 2 && p.patch_radius == 2)  // r_g = 0.2
    return launch_fast<2, 2>(ctx, ground, ceiling, S, rows, cols, kernel_w, kside, cost);
  if (sym && R == 3 && p.patch_radius == 3)
    return launch_fast<3, 3>(ctx, ground, ceiling, S, rows, cols, kernel_w, kside, cost);
  if (sym && R == 4 && p.patch_radius == 4)
    return launch_fast<4, 4>(ctx, ground, ceiling, S, rows, cols, kernel_w, kside, cost);
  if (sym && R == 8 && p.patch_radius == 6)  // r_g = 0.05 with the Table-I radii
    return launch_fast<8, 6>(ctx, ground, ceiling, S, rows, cols, kernel_w, kside, cost);
  // generic path: pick the largest square-ish tile that fits in shared memory
  int TH = 64, TW = 64;
  TileGeom G = make_geom(R, p.patch_radius, TH, TW);
  while (G.smem > 200 * 1024 && (TH > 8 || TW > 8)) {
    if (TH >= TW) TH /= 2; else TW /= 2;
    G = make_geom(R, p.patch_radius, TH, TW);
  }
  if (G.smem > 220 * 1024) return fail(ctx, PCT_E_INVALID, "stencil radius too large for one tile");
  auto kern = eval_generic_kernel<kNT>;
  PCT_CUDA(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G.smem));
  dim3 grid((cols + TW - 1) / TW, (rows + TH - 1) / TH, S);
  kern<<<grid, kNT, G.smem, ctx->stream>>>(G, ground, ceiling, rows, cols, kside, mode, cost);
  return check_launch(ctx, "eval_generic_kernel");
}

// Batched maps (config 4): one walk launch and one resolve/inflate launch for
// every map (blockIdx.y / flattened work items select the map's descriptor).
// Kernels whose weight classes the compiled tables cover (R = 4, r = 3: r_g
// 0.1 with the Table-I parameters); anything else evaluates map by map.
int launch_evaluate_batch(pct_ctx *ctx, int n_maps, float *const *ground, float *const *ceiling,
                          const pct_frame *frames, const pct_trav_params &p,
                          const float *kernel_w, int kside, float *const *cost) {
  if (n_maps <= 0) return PCT_OK;
#ifndef PCT_BNB_BATCH_TH
#define PCT_BNB_BATCH_TH 24  // (32: cfg4 5.438 vs 5.41 ms)
#endif
  constexpr int R = 4, PR = 3, TH = PCT_BNB_BATCH_TH, TW = 32, BNT = 128;
  std::vector<float> bw;
  const double r_g = frames[0].r_g;
  bool same_rg = true;
  for (int m = 1; m < n_maps; ++m) same_rg = same_rg && frames[m].r_g == r_g;
  if (!(kside == 2 * R + 1 && p.patch_radius == PR && same_rg && bnb_tables<R>(kernel_w, kside, bw))) {
    for (int m = 0; m < n_maps; ++m)
      if (int rc = launch_evaluate(ctx, ground[m], ceiling[m], frames[m].n_slices, frames[m].rows,
                                   frames[m].cols, frames[m].r_g, p, kernel_w, kside, cost[m],
                                   kEvalFull))
        return rc;
    return PCT_OK;
  }
  ConstBank cb(ctx);
  EvalConsts K = make_consts(p, r_g);
  PCT_CUDA(ctx, cb.set_symbol(c_K, &K, sizeof(K)));
  PCT_CUDA(ctx, cb.set_symbol(c_bw, bw.data(), bw.size() * sizeof(float)));
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    PCT_CUDA(ctx, cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess)
      return fail(ctx, PCT_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  auto kb = resolve_inflate_bnb_kernel<R, PR, TH, TW, BNT, kBnbMinBlocks<R>()>;
  constexpr int bsmem = BnbGeom<R, PR, TH, TW>::SMEM;
  PCT_CUDA(ctx, cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, bsmem));
  int per_sm = 0;
  PCT_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kb, BNT, bsmem));
  const int64_t slots = (int64_t)std::max(1, per_sm) * ctx->num_sms;
  // layouts, offsets, run length
  std::vector<EvalMap> hm(n_maps);
  std::vector<int> off(n_maps + 2, 0);  // item offsets, then the dynamic item counter (0)
  int64_t enc_floats = 0, bit_words = 0, total_tiles = 0, walk_blocks = 1;
  uint64_t tag = 1469598103934665603ull;
  for (int m = 0; m < n_maps; ++m) {
    const pct_frame &fr = frames[m];
    EvalMap &e = hm[m];
    std::memset(&e, 0, sizeof(EvalMap));
    e.S = fr.n_slices;
    e.rows = fr.rows;
    e.cols = fr.cols;
    e.wpr = (fr.cols + 31) / 32;
    e.words = (int64_t)fr.rows * e.wpr;
    e.L.padr = R;
    e.L.padc = R;
    e.L.prows = (fr.rows + TH - 1) / TH * TH + 2 * R;
    e.L.pitch = ((int64_t)((fr.cols + TW - 1) / TW * TW + 2 * R) + 3) / 4 * 4;
    e.L.sstride = (int64_t)e.L.prows * e.L.pitch;
    enc_floats += (int64_t)e.S * e.L.sstride;
    bit_words += (int64_t)e.S * e.words;
    total_tiles += (int64_t)((fr.cols + TW - 1) / TW) * ((fr.rows + TH - 1) / TH);
    walk_blocks = std::max<int64_t>(walk_blocks, (e.words * 32 + kWalkNT - 1) / kWalkNT);
    for (uint64_t v : {(uint64_t)e.S, (uint64_t)e.rows, (uint64_t)e.cols})
      tag = (tag ^ v) * 1099511628211ull;
  }
  // encoded c_init stacks of every map in the context's buffer; zeroed once
  // per batch layout (the walk rewrites the interiors, the pads stay 0)
  const size_t enc_bytes = (size_t)enc_floats * 4;
  if (ctx->enc_bytes < enc_bytes) {
    if (ctx->enc) {
      cudaStreamSynchronize(ctx->stream);
      cudaFree(ctx->enc);
      ctx->enc = nullptr;
      ctx->enc_bytes = 0;
    }
    PCT_CUDA(ctx, cudaMalloc(&ctx->enc, enc_bytes));
    ctx->enc_bytes = enc_bytes;
    ctx->enc_tag[0] = -1;
  }
  const int64_t tagi = (int64_t)(tag >> 1);
  if (ctx->enc_tag[0] != -2 || ctx->enc_tag[1] != tagi) {
    PCT_CUDA(ctx, cudaMemsetAsync(ctx->enc, 0, enc_bytes, ctx->stream));
    ctx->enc_tag[0] = -2;
    ctx->enc_tag[1] = tagi;
  }
  // scratch: gentle bitmaps | descriptors (64-byte aligned) | item offsets |
  // walk change maps
  const size_t bbytes = (((size_t)bit_words * 4 + 255) / 256) * 256;
  const size_t dbytes = (((size_t)n_maps * sizeof(EvalMap) + 255) / 256) * 256;
  const size_t obytes = (((size_t)(n_maps + 2) * 4 + 255) / 256) * 256;  // + work counter
  int64_t cm_total = 0;
  for (auto &e : hm) cm_total += (int64_t)e.S * ((e.rows + 7) / 8) * e.wpr;
  if (int rc = ensure_scratch(ctx, bbytes + dbytes + obytes + (size_t)cm_total + 64)) return rc;
  char *sb = static_cast<char *>(ctx->scratch);
  unsigned char *cmb = reinterpret_cast<unsigned char *>(sb + bbytes + dbytes + obytes);
  const char *skv = getenv("PCT_BNB_SKIP");  // on by default (see launch_split)
  const bool use_skip = skv ? skv[0] == '1' : true;
  if (use_skip) PCT_CUDA(ctx, cudaMemsetAsync(cmb, 0, (size_t)cm_total, ctx->stream));
  int run_all = 0;
  {
    int smax = 1;
    for (auto &e : hm) smax = std::max(smax, e.S);
    run_all = smax;
    int64_t all_tiles = 0;
    for (auto &e : hm) all_tiles += (int64_t)((e.cols + TW - 1) / TW) * ((e.rows + TH - 1) / TH);
    const int64_t runs = std::min<int64_t>(smax, (3 * slots + all_tiles - 1) / all_tiles);
    run_all = (int)((smax + runs - 1) / runs);  // as in launch_split
    if (const char *e = getenv("PCT_INFL_RUN")) run_all = std::max(1, atoi(e));
    run_all = std::min(run_all, 64);  // per-item skip mask: 64 slices
  }
  float *encb = static_cast<float *>(ctx->enc);
  int64_t eoff = 0, boffw = 0;
  for (int m = 0; m < n_maps; ++m) {
    EvalMap &e = hm[m];
    e.ground = ground[m];
    e.ceiling = ceiling[m];
    e.cost = cost[m];
    e.enc = encb + eoff;
    e.bits = reinterpret_cast<uint32_t *>(sb) + boffw;
    e.run = std::min(run_all, e.S);
    e.chg = use_skip ? cmb : nullptr;
    cmb += (int64_t)e.S * ((e.rows + 7) / 8) * e.wpr;
    const cuuint64_t dims[3] = {(cuuint64_t)e.L.pitch, (cuuint64_t)e.L.prows, (cuuint64_t)e.S};
    const cuuint64_t strides[2] = {(cuuint64_t)e.L.pitch * 4, (cuuint64_t)e.L.sstride * 4};
    const cuuint32_t box[3] = {(cuuint32_t)(TW + 2 * R), (cuuint32_t)(TH + 2 * R), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    if (encode(&e.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, e.enc, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return fail(ctx, PCT_E_CUDA, "cuTensorMapEncodeTiled failed");
    const int tiles = ((e.cols + TW - 1) / TW) * ((e.rows + TH - 1) / TH);
    off[m + 1] = off[m] + tiles * ((e.S + e.run - 1) / e.run);
    eoff += (int64_t)e.S * e.L.sstride;
    boffw += (int64_t)e.S * e.words;
  }
  EvalMap *dm = reinterpret_cast<EvalMap *>(sb + bbytes);
  int *doff = reinterpret_cast<int *>(sb + bbytes + dbytes);
  PCT_CUDA(ctx, upload_async(ctx, dm, hm.data(), sizeof(EvalMap) * n_maps));
  PCT_CUDA(ctx, upload_async(ctx, doff, off.data(), sizeof(int) * (n_maps + 2)));
  terrain_walk_batch_kernel<1><<<dim3((unsigned)walk_blocks, n_maps), kWalkNT, 0, ctx->stream>>>(dm);
  if (int rc = check_launch(ctx, "terrain_walk_batch_kernel")) return rc;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(off[n_maps], slots));
  const char *dyv = getenv("PCT_BNB_DYNAMIC");
  const bool dyn = !(dyv && dyv[0] == '0');
  kb<<<grid, BNT, bsmem, ctx->stream>>>(dm, doff, n_maps, dyn ? doff + n_maps + 1 : nullptr);
  return check_launch(ctx, "resolve_inflate_bnb_kernel");
}

int launch_inflate(pct_ctx *ctx, const float *in, int rows, int cols, const float *kernel_w,
                   int kside, float *out) {
  if (rows <= 0 || cols <= 0) return PCT_OK;
  if (kside <= 0 || (kside & 1) == 0 || kside * kside > kMaxTaps)
    return fail(ctx, PCT_E_INVALID, "inflation kernel side must be odd and <= 125");
  ConstBank cb(ctx);
  PCT_CUDA(ctx, cb.set_symbol(c_wfull, kernel_w, sizeof(float) * kside * kside));
  int TH = 32, TW = 32;
  TileGeom G = make_geom(kside / 2, 0, TH, TW);
  while (G.smem > 200 * 1024 && (TH > 8 || TW > 8)) {
    if (TH >= TW) TH /= 2; else TW /= 2;
    G = make_geom(kside / 2, 0, TH, TW);
  }
  auto kern = inflate_kernel<kNT>;
  PCT_CUDA(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G.smem));
  dim3 grid((cols + TW - 1) / TW, (rows + TH - 1) / TH, 1);
  kern<<<grid, kNT, G.smem, ctx->stream>>>(G, in, rows, cols, kside, out);
  return check_launch(ctx, "inflate_kernel");
}

}  // namespace pct
