// k_eval_incr.cuh — slice-incremental fused evaluation (included by
// k_evaluate.cu inside namespace pct::{anon}; uses its c_K / c_wsym).
//
// A CTA owns one TH x TW output tile and walks a run of consecutive slices
// k0..k1-1.  All per-cell state of the previous slice stays in shared memory
// (ground region, ceiling, terrain result, gentle bits, c_init) and, for the
// next slice, only what depends on changed inputs is recomputed:
//
//   gchg  ground cells whose value changed            (load region)
//   xchg  cells whose 5-point ground cross changed    -> terrain recomputed
//   gflip gentle flags that flipped                   -> foothold windows dirty
//   rset  c_init cells to re-derive: xchg | ceiling changed | gflip dilated by r
//   ichg  c_init cells whose value changed            -> outputs within R redone
//
// Every value is recomputed by the same arithmetic as the full kernel from the
// same inputs, so the result is bit-identical to recomputing everything; the
// first slice of a run is a full computation.  On the tomograms of the
// configs only 15-25 % of the cells of a slice differ from the slice below
// (ground and ceiling only change where a cutting plane passes a surface).

template <int R, int PR, int TH, int TW>
struct IncrGeom {
  static constexpr int CH = TH + 2 * R, CW = TW + 2 * R;    // c_init region
  static constexpr int GH = CH + 2 * PR, GW = CW + 2 * PR;  // gentle region
  static constexpr int LH = GH + 2, LW = GW + 2;            // loaded ground
  static constexpr int H = R + PR + 1;
  static constexpr int LWW = (LW + 31) / 32 + 1;  // words per bit row (+1 pad)
  static constexpr int GWW = (GW + 31) / 32 + 1;
  static constexpr int CWW = (CW + 31) / 32 + 1;
  // shared memory layout (bytes)
  static constexpr int O_GRD = 0;
  static constexpr int O_CEIL = O_GRD + LH * LW * 4;
  static constexpr int O_CG = O_CEIL + CH * CW * 4;
  static constexpr int O_CI = O_CG + CH * CW * 4;
  static constexpr int O_GBITS = O_CI + CH * CW * 4;
  static constexpr int O_GCHG = O_GBITS + GH * GWW * 4;
  static constexpr int O_XCHG = O_GCHG + LH * LWW * 4;
  static constexpr int O_GFLIP = O_XCHG + GH * GWW * 4;
  static constexpr int O_HDIL = O_GFLIP + GH * GWW * 4;
  static constexpr int O_CCHG = O_HDIL + GH * CWW * 4;
  static constexpr int O_RSET = O_CCHG + CH * CWW * 4;
  static constexpr int O_ICHG = O_RSET + CH * CWW * 4;
  static constexpr int O_LIST = O_ICHG + CH * CWW * 4;
  static constexpr int SMEM = O_LIST + ((GH * GW * 2 + 15) / 16) * 16;
};

// 32 bits of a bit row starting at column xs (row has >= (xs>>5)+2 words)
__device__ __forceinline__ uint32_t bits_at(const uint32_t *row, int xs) {
  const int w = xs >> 5, sh = xs & 31;
  const uint64_t v = (uint64_t)row[w] | ((uint64_t)row[w + 1] << 32);
  return (uint32_t)(v >> sh);
}

__device__ __forceinline__ uint32_t valid_mask(int width, int w) {
  const int n = width - 32 * w;
  return n >= 32 ? 0xFFFFFFFFu : (n <= 0 ? 0u : ((1u << n) - 1u));
}

// Append the set bits of a (rows x words) bit array to list (as y*width+x).
template <int NT>
__device__ __forceinline__ void compact_bits(const uint32_t *bitsarr, int nrows, int words,
                                             int width, uint16_t *list, int *count) {
  for (int idx = threadIdx.x; idx < nrows * words; idx += NT) {
    const int y = idx / words, w = idx - y * words;
    uint32_t m = bitsarr[idx] & valid_mask(width, w);
    if (!m) continue;
    int pos = atomicAdd(count, __popc(m));
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      list[pos++] = (uint16_t)(y * width + 32 * w + b);
    }
  }
}

// Inflation of one column strip into registers (same arithmetic as
// inflate_sym_strip).
template <int R, int V>
__device__ __forceinline__ void inflate_strip_regs(const float *__restrict__ cinit, int CW, int x,
                                                   int ys, float (&acc_out)[V]) {
  float P[V + 2 * R][R + 1];
#pragma unroll
  for (int t = 0; t < V + 2 * R; ++t) {
    const float *rowp = cinit + (ys + t) * CW + x;
    P[t][0] = rowp[R];
#pragma unroll
    for (int b = 1; b <= R; ++b) P[t][b] = fmaxf(rowp[R - b], rowp[R + b]);
    if (t >= 2 * R) {
      const int o = t - 2 * R;
      const int c = o + R;
      float acc = 0.0f;
#pragma unroll
      for (int a = 0; a <= R; ++a) {
#pragma unroll
        for (int b = 0; b <= a; ++b) {
          const float w = c_wsym[a * 9 + b];
          if (w > 0.0f) {
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
            acc = fmaxf(acc, w * m);
          }
        }
      }
      acc_out[o] = acc;
    }
  }
}

template <int R, int PR, int TH, int TW, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) eval_incr_kernel(const float *__restrict__ ground,
                                                          const float *__restrict__ ceiling,
                                                          int rows, int cols, int S, int run,
                                                          int tiles_x, int n_tiles, int n_items,
                                                          int *__restrict__ next_item,
                                                          float *__restrict__ cost) {
  using G = IncrGeom<R, PR, TH, TW>;
  extern __shared__ __align__(16) unsigned char smem[];
  float *grd = reinterpret_cast<float *>(smem + G::O_GRD);
  float *ceil_s = reinterpret_cast<float *>(smem + G::O_CEIL);
  float *cgenc = reinterpret_cast<float *>(smem + G::O_CG);
  float *cinit = reinterpret_cast<float *>(smem + G::O_CI);
  uint32_t *gbits = reinterpret_cast<uint32_t *>(smem + G::O_GBITS);
  uint32_t *gchg = reinterpret_cast<uint32_t *>(smem + G::O_GCHG);
  uint32_t *xchg = reinterpret_cast<uint32_t *>(smem + G::O_XCHG);
  uint32_t *gflip = reinterpret_cast<uint32_t *>(smem + G::O_GFLIP);
  uint32_t *hdil = reinterpret_cast<uint32_t *>(smem + G::O_HDIL);
  uint32_t *cchg = reinterpret_cast<uint32_t *>(smem + G::O_CCHG);
  uint32_t *rset = reinterpret_cast<uint32_t *>(smem + G::O_RSET);
  uint32_t *ichg = reinterpret_cast<uint32_t *>(smem + G::O_ICHG);
  uint16_t *list = reinterpret_cast<uint16_t *>(smem + G::O_LIST);
  __shared__ int cnt;
  __shared__ int item_s;

  const int tid = threadIdx.x;
  const int64_t plane = (int64_t)rows * cols;
  const float nanf_ = bits_f32(kNaNBits);
  const float cb32 = (float)c_K.c_barrier;
  constexpr int SIDE = 2 * PR + 1;
  constexpr uint32_t WMASK = (1u << SIDE) - 1u;  // SIDE <= 31
  constexpr int STRIPS = NT / TW;
  constexpr int V = TH / STRIPS;
  const int ox = tid % TW, strip = tid / TW;
  float outv[V];

  // persistent CTAs pull (tile, slice run) items; runs of one tile differ in
  // cost (first slice full, the rest incremental), so balance dynamically
  for (;;) {
  if (tid == 0) item_s = atomicAdd(next_item, 1);
  __syncthreads();
  const int item = item_s;
  if (item >= n_items) break;
  const int tile = item % n_tiles, chunk = item / n_tiles;
  const int i0 = (tile / tiles_x) * TH, j0 = (tile % tiles_x) * TW;
  const int k0 = chunk * run;
  const int k1 = min(S, k0 + run);

  // persistent state starts "unknown": force a full first slice
  for (int i = tid; i < G::LH * G::LW; i += NT) grd[i] = bits_f32(0x7FFFFFFFu);  // never loaded
  for (int i = tid; i < G::CH * G::CW; i += NT) {
    ceil_s[i] = bits_f32(0x7FFFFFFFu);
    cinit[i] = 0.0f;
    cgenc[i] = nanf_;
  }
  for (int i = tid; i < G::GH * G::GWW; i += NT) gbits[i] = 0u;
  __syncthreads();

  for (int k = k0; k < k1; ++k) {
    const bool first = (k == k0);
    const float *gk = ground + k * plane;
    const float *ck = ceiling + k * plane;
    // ---- clear change sets
    for (int i = tid; i < G::LH * G::LWW; i += NT) gchg[i] = 0u;
    for (int i = tid; i < G::GH * G::GWW; i += NT) gflip[i] = 0u;
    for (int i = tid; i < G::CH * G::CWW; i += NT) {
      cchg[i] = 0u;
      ichg[i] = 0u;
    }
    if (tid == 0) cnt = 0;
    __syncthreads();

    // ---- A: load ground region and CI ceiling (all loads of a thread in
    // flight together), note changed cells
    {
      constexpr int NA = (G::LH * G::LW + NT - 1) / NT;
      constexpr int NC = (G::CH * G::CW + NT - 1) / NT;
      float va[NA], vc[NC];
#pragma unroll
      for (int u = 0; u < NA; ++u) {
        const int idx = tid + u * NT;
        const int y = idx / G::LW, x = idx - y * G::LW;
        const int gi = i0 - G::H + y, gj = j0 - G::H + x;
        va[u] = (idx < G::LH * G::LW && gi >= 0 && gi < rows && gj >= 0 && gj < cols)
                    ? __ldg(gk + (int64_t)gi * cols + gj)
                    : nanf_;
      }
#pragma unroll
      for (int u = 0; u < NC; ++u) {
        const int idx = tid + u * NT;
        const int y = idx / G::CW, x = idx - y * G::CW;
        const int gi = i0 - R + y, gj = j0 - R + x;
        vc[u] = (idx < G::CH * G::CW && gi >= 0 && gi < rows && gj >= 0 && gj < cols)
                    ? __ldg(ck + (int64_t)gi * cols + gj)
                    : nanf_;
      }
#pragma unroll
      for (int u = 0; u < NA; ++u) {
        const int idx = tid + u * NT;
        if (idx < G::LH * G::LW && f32_bits(va[u]) != f32_bits(grd[idx])) {
          const int y = idx / G::LW, x = idx - y * G::LW;
          grd[idx] = va[u];
          atomicOr(&gchg[y * G::LWW + (x >> 5)], 1u << (x & 31));
        }
      }
#pragma unroll
      for (int u = 0; u < NC; ++u) {
        const int idx = tid + u * NT;
        if (idx < G::CH * G::CW && f32_bits(vc[u]) != f32_bits(ceil_s[idx])) {
          const int y = idx / G::CW, x = idx - y * G::CW;
          ceil_s[idx] = vc[u];
          atomicOr(&cchg[y * G::CWW + (x >> 5)], 1u << (x & 31));
        }
      }
    }
    __syncthreads();

    // ---- cross-changed set over the gentle region (GEN (y,x) = load (y+1,x+1))
    for (int idx = tid; idx < G::GH * G::GWW; idx += NT) {
      const int y = idx / G::GWW, w = idx - y * G::GWW;
      uint32_t m = 0;
      if (first) {
        m = 0xFFFFFFFFu;
      } else if (32 * w < G::GW) {
        const uint32_t *r0 = gchg + y * G::LWW, *r1 = r0 + G::LWW, *r2 = r1 + G::LWW;
        const int xs = 32 * w;
        m = bits_at(r0, xs + 1) | bits_at(r2, xs + 1) | bits_at(r1, xs) | bits_at(r1, xs + 1) |
            bits_at(r1, xs + 2);
      }
      xchg[idx] = m & valid_mask(G::GW, w);
    }
    __syncthreads();
    compact_bits<NT>(xchg, G::GH, G::GWW, G::GW, list, &cnt);
    __syncthreads();

    // ---- B: terrain for changed crosses; gentle flips; terrain part of c_init
    {
      const int n = cnt;
      for (int i = tid; i < n; i += NT) {
        const int gidx = list[i];
        const int y = gidx / G::GW, x = gidx - y * G::GW;
        const float *p = grd + (y + 1) * G::LW + (x + 1);
        const Cross c{p[0], p[-1], p[1], p[-G::LW], p[G::LW]};
        const FastCell t = fast_terrain(c, c_K);
        const uint32_t bit = 1u << (x & 31);
        uint32_t *gw = gbits + y * G::GWW + (x >> 5);
        const bool old = (*gw & bit) != 0;
        if (old != t.gentle) {
          atomicXor(gw, bit);
          atomicOr(gflip + y * G::GWW + (x >> 5), bit);
        }
        if (y >= PR && y < PR + G::CH && x >= PR && x < PR + G::CW) {
          float enc;
          if (!t.valid) {
            enc = nanf_;
          } else if (t.isolated || t.m_xy > c_K.theta_b) {
            enc = cb32;
          } else if (t.gentle) {
            enc = gentle_cost32(t.gx, t.gy, t.s, c_K);
          } else {
            const double q = div_const(t.m_xy, c_K.theta_b, c_K.inv_theta_b);
            enc = bits_f32(f32_bits((float)(c_K.alpha_b * (q * q))) | 0x80000000u);
          }
          cgenc[(y - PR) * G::CW + (x - PR)] = enc;
        }
      }
    }
    __syncthreads();

    // ---- c_init recompute set: crosses | ceilings | foothold windows of flips
    for (int idx = tid; idx < G::GH * G::CWW; idx += NT) {  // horizontal dilation by r
      const int y = idx / G::CWW, w = idx - y * G::CWW;
      uint32_t m = 0;
      if (!first && 32 * w < G::CW) {
        const uint32_t *row = gflip + y * G::GWW;
#pragma unroll
        for (int d = 0; d < SIDE; ++d) m |= bits_at(row, 32 * w + d);
      }
      hdil[idx] = m;
    }
    if (tid == 0) cnt = 0;
    __syncthreads();
    for (int idx = tid; idx < G::CH * G::CWW; idx += NT) {
      const int y = idx / G::CWW, w = idx - y * G::CWW;
      uint32_t m;
      if (first) {
        m = 0xFFFFFFFFu;
      } else if (32 * w < G::CW) {
        m = cchg[idx] | bits_at(xchg + (y + PR) * G::GWW, 32 * w + PR);
#pragma unroll
        for (int d = 0; d < SIDE; ++d) m |= hdil[(y + d) * G::CWW + w];
      } else {
        m = 0u;
      }
      rset[idx] = m & valid_mask(G::CW, w);
    }
    __syncthreads();
    compact_bits<NT>(rset, G::CH, G::CWW, G::CW, list, &cnt);
    __syncthreads();

    // ---- C: re-derive c_init for the set; note changed values
    {
      const int n = cnt;
      for (int i = tid; i < n; i += NT) {
        const int ci = list[i];
        const int y = ci / G::CW, x = ci - y * G::CW;
        const int gi = i0 - R + y, gj = j0 - R + x;
        if (!(gi >= 0 && gi < rows && gj >= 0 && gj < cols)) continue;  // zero padding stays 0
        const float enc = cgenc[ci];
        float cnew;
        if (!finite32(enc)) {
          cnew = cb32;  // no ground: barrier (fuse_costs :169)
        } else {
          float cg = enc;
          if (f32_bits(enc) & 0x80000000u) {
            const int w = x >> 5, sh = x & 31;  // window GEN rows y..y+2r, cols x..x+2r
            int c = 0;
#pragma unroll
            for (int d = 0; d < SIDE; ++d) {
              const uint32_t *rw = gbits + (y + d) * G::GWW + w;
              const uint64_t v = (uint64_t)rw[0] | ((uint64_t)rw[1] << 32);
              c += __popc((uint32_t)(v >> sh) & WMASK);
            }
            cg = c >= c_K.ps_min_count ? bits_f32(f32_bits(enc) & 0x7FFFFFFFu) : cb32;
          }
          const float g = grd[(y + PR + 1) * G::LW + (x + PR + 1)];
          cnew = fuse_value(interval_value(g, ceil_s[ci], c_K), cg, c_K);
        }
        if (f32_bits(cnew) != f32_bits(cinit[ci])) {
          cinit[ci] = cnew;
          atomicOr(&ichg[y * G::CWW + (x >> 5)], 1u << (x & 31));
        }
      }
    }
    __syncthreads();

    // ---- E: inflation of the output strips that see a changed c_init
    bool dirty = first;
    if (!dirty) {
      uint32_t any = 0;
#pragma unroll 4
      for (int t = 0; t < V + 2 * R; ++t) any |= bits_at(ichg + (strip * V + t) * G::CWW, ox);
      dirty = (any & ((1u << (2 * R + 1)) - 1u)) != 0;
    }
    if (__any_sync(0xFFFFFFFFu, dirty)) inflate_strip_regs<R, V>(cinit, G::CW, ox, strip * V, outv);
    {
      float *out = cost + k * plane;
      const int gj = j0 + ox;
#pragma unroll
      for (int o = 0; o < V; ++o) {
        const int gi = i0 + strip * V + o;
        if (gi < rows && gj < cols) out[(int64_t)gi * cols + gj] = outv[o];
      }
    }
    __syncthreads();
  }
  }  // work items
}
