// k_eval_split.cuh — two-kernel evaluation (included by k_evaluate.cu inside
// namespace pct::{anon}; uses its c_K / c_wsym and the inflation helpers).
//
//  T  terrain_walk_kernel: one thread per cell walks the slices bottom-up.
//     The float64 terrain arithmetic (gradients, guarded glibc hypot, costs)
//     runs only when the cell's 5-point ground cross differs from the slice
//     below, the interval/fuse step only when the cross or the ceiling
//     differs; otherwise the previous slice's values are reused (they are a
//     function of exactly those inputs, so the result is bit-identical).  On
//     the config maps ground and ceiling change in < 25 % of the cells per
//     slice (a cutting plane passes a surface).  Writes the encoded c_init
//     (float32, sign bit = foothold branch pending) and the gentle flags as a
//     row-major bitmap per slice (one __ballot_sync word per 32 cells).
//  I  resolve_inflate_kernel: per 64x64 tile and slice, the encoded c_init
//     tile + R halo and the gentle bits of the foothold window are staged in
//     shared memory, the pending cells are resolved by popcount over
//     (2r+1)^2 bits, and the weighted max of the inflation kernel is taken
//     from a register ring of pair maxima (as eval_fast_kernel stage E).
// No cell is computed twice for a halo, and T needs no block barrier.

constexpr int kWalkNT = 256;

// Encoded c_init stacks live in a zero-padded layout: every tile + halo the
// inflation kernel stages is in bounds and reads 0 outside the map
// (inflate's cval=0), and row starts are 16-byte aligned for float4 loads.
struct EncLayout {
  int padr, padc;        // rows / columns of zeros before the map
  int64_t pitch;         // floats per padded row (multiple of 4)
  int64_t sstride;       // floats per padded slice
  int prows;             // padded rows
  __host__ __device__ int64_t at(int k, int i, int j) const {
    return (int64_t)k * sstride + (int64_t)(i + padr) * pitch + (j + padc);
  }
};

// zero every padded cell outside the map (interior cells are written by T):
// one block per padded row; pad rows are cleared whole, map rows only at
// their left / right margins
__global__ void __launch_bounds__(128) zero_pads_kernel(float *__restrict__ enc, EncLayout L,
                                                        int rows, int cols) {
  const int k = blockIdx.y, r = blockIdx.x;  // padded row
  float *row = enc + (int64_t)k * L.sstride + (int64_t)r * L.pitch;
  const int i = r - L.padr;
  if (i < 0 || i >= rows) {
    for (int c = threadIdx.x; c < L.pitch; c += blockDim.x) row[c] = 0.0f;
  } else {
    for (int c = threadIdx.x; c < L.padc; c += blockDim.x) row[c] = 0.0f;
    for (int c = L.padc + cols + threadIdx.x; c < L.pitch; c += blockDim.x) row[c] = 0.0f;
  }
}

// Gentle bitmap layout: per slice, rows of wpr = ceil(cols / 32) words; bit
// b of word w of row i = cell (i, 32 w + b).  gentle_word returns the 32 bits
// of row gi starting at column gj (any gj; 0 outside the map).
__device__ __forceinline__ uint32_t gentle_word(const uint32_t *__restrict__ bk, int wpr, int gi,
                                                int gj, int rows, int cols) {
  if (gi < 0 || gi >= rows || gj >= cols || gj + 32 <= 0) return 0u;
  const uint32_t *row = bk + (int64_t)gi * wpr;
  const int w = gj >> 5, sh = gj & 31;  // floor division: w >= -1
  const uint32_t lo = w >= 0 ? __ldg(row + w) : 0u;
  const uint32_t hi = (sh != 0 && w + 1 < wpr) ? __ldg(row + w + 1) : 0u;
  return sh ? __funnelshift_r(lo, hi, sh) : lo;  // bits past cols are 0 in the map
}

// Per-cell state of a terrain walk between slices, and one slice of it: the
// terrain part runs only when the 5-point cross changed since the slice
// below, the interval / fuse part only when the cross or the ceiling did.
struct WalkState {
  uint32_t xe = 0, xl = 0, xr = 0, xu = 0, xd = 0, xc = 0;  // previous slice's input bits
  float tenc;  // terrain part: NaN = no ground, sign bit = foothold branch
  float enc = 0.0f;
  bool gentle = false;
};

__device__ __forceinline__ void walk_step(WalkState &st, int k, bool live, float e, float l,
                                          float r, float u, float d, float c, float nanf_,
                                          float cb32) {
  const bool xch = k == 0 || f32_bits(e) != st.xe || f32_bits(l) != st.xl ||
                   f32_bits(r) != st.xr || f32_bits(u) != st.xu || f32_bits(d) != st.xd;
  if (xch && live) {
    const FastCell t = fast_terrain(Cross{e, l, r, u, d}, c_K);
    st.gentle = t.gentle;
    if (!t.valid) {
      st.tenc = nanf_;
    } else if (t.isolated || t.m_xy > c_K.theta_b) {
      st.tenc = cb32;
    } else if (t.gentle) {
      st.tenc = gentle_cost32(t.gx, t.gy, t.s, c_K);
    } else {
      const double q = div_const(t.m_xy, c_K.theta_b, c_K.inv_theta_b);
      st.tenc = bits_f32(f32_bits((float)(c_K.alpha_b * (q * q))) | 0x80000000u);
    }
  }
  if ((xch || f32_bits(c) != st.xc) && live) {
    if (!finite32(st.tenc)) {
      st.enc = cb32;  // no ground: barrier (fuse_costs :169)
    } else {
      const uint32_t tb = f32_bits(st.tenc);
      st.enc = fuse_value(interval_value(e, c, c_K), bits_f32(tb & 0x7FFFFFFFu), c_K);
      if (tb & 0x80000000u) st.enc = bits_f32(f32_bits(st.enc) | 0x80000000u);
    }
  }
  st.xe = f32_bits(e); st.xl = f32_bits(l); st.xr = f32_bits(r); st.xu = f32_bits(u);
  st.xd = f32_bits(d); st.xc = f32_bits(c);
}

// Terrain walk: one thread per cell (flat row-major index, so a warp is 32
// consecutive cells) walks the slices bottom-up.  The float64 terrain
// arithmetic runs only when the cell's 5-point cross changed since the slice
// below, the interval / fuse step only when the cross or the ceiling did.
// Loads run PF slices ahead; left / right neighbours come from the adjacent
// lanes (lanes 0 and 31 load the cell beyond), grid borders read NaN.
template <int PF>
__device__ __forceinline__ void walk_body(const float *__restrict__ ground,
                                          const float *__restrict__ ceiling, int S, int rows,
                                          int cols, float *__restrict__ enc_out,
                                          const EncLayout &L, uint32_t *__restrict__ bits_out,
                                          int wpr, unsigned char *__restrict__ chgmap,
                                          int l2d, int kb, int ke) {
  // slices kb .. ke-1 (a chunk: its first slice is computed in full)
  const int64_t cells = (int64_t)rows * cols;
  // threads index row-padded columns: warp = one gentle-bitmap word of one row
  const int64_t pidx = (int64_t)blockIdx.x * kWalkNT + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int pcols = wpr * 32;
  // (32-bit division when the padded grid has < 2^32 cells: a 64-bit
  // division by a run-time value is a ~100-instruction subroutine)
  const int i0_ = (int64_t)rows * pcols <= 0xFFFFFFFFll
                      ? (int)((uint32_t)pidx / (uint32_t)pcols)
                      : (int)(pidx / pcols);
  const int j0_ = (int)(pidx - (int64_t)i0_ * pcols);
  const bool live = i0_ < rows && j0_ < cols;
  const int i = i0_ < rows ? i0_ : rows - 1;
  const int j = j0_ < cols ? j0_ : cols - 1;  // clamped: address formation only
  const bool wlead = lane == 0 && i0_ < rows;
  const bool hl = live && j > 0, hr = live && j + 1 < cols, hu = live && i > 0,
             hd = live && i + 1 < rows;
  const bool edge_l = lane == 0 && hl, edge_r = lane == 31 && hr;
  const float nanf_ = bits_f32(kNaNBits);
  const float cb32 = (float)c_K.c_barrier;
  const int64_t base = (int64_t)i * cols + j;
  const float *pg = ground + base + (int64_t)kb * cells;
  const float *pc = ceiling + base + (int64_t)kb * cells;
  float *pe = enc_out + L.at(kb, i, j);
  uint32_t *pb = bits_out + (int64_t)kb * rows * wpr + (int64_t)i * wpr + (j0_ >> 5);

  float qe[PF], qu[PF], qd[PF], qc[PF], ql[PF], qr[PF];
  auto fetch = [&](const float *g, const float *c, int s) {
    qe[s] = live ? __ldg(g) : nanf_;
    qu[s] = hu ? __ldg(g - cols) : nanf_;
    qd[s] = hd ? __ldg(g + cols) : nanf_;
    qc[s] = live ? __ldg(c) : nanf_;
    ql[s] = edge_l ? __ldg(g - 1) : nanf_;
    qr[s] = edge_r ? __ldg(g + 1) : nanf_;
  };
#pragma unroll
  for (int s = 0; s < PF; ++s)
    if (kb + s < ke) fetch(pg + s * cells, pc + s * cells, s);
  const float *ng = pg + PF * cells, *nc = pc + PF * cells;

  WalkState st;
  st.tenc = nanf_;
  // change map: one byte per (slice, 8-row block, bitmap word) set when any
  // cell's encoded c_init or gentle flag differs from the slice below (the
  // resolve/inflate kernel skips tiles whose window saw no change)
  const int64_t cmstride = (int64_t)((rows + 7) >> 3) * wpr;
  unsigned char *pcm = chgmap + (int64_t)kb * cmstride + (int64_t)(i >> 3) * wpr + (j0_ >> 5);
  uint32_t prev_enc = 0u;
  unsigned prev_word = 0u;
  for (int k0 = kb; k0 < ke; k0 += PF) {
#pragma unroll
    for (int s = 0; s < PF; ++s) {
      const int k = k0 + s;
      if (k >= ke) break;
      const float e = qe[s], u = qu[s], d = qd[s], c = qc[s];
      float l = __shfl_up_sync(0xFFFFFFFFu, e, 1);
      float r = __shfl_down_sync(0xFFFFFFFFu, e, 1);
      if (lane == 0) l = ql[s];
      if (lane == 31) r = qr[s];
      if (!hl) l = nanf_;
      if (!hr) r = nanf_;
      if (k + PF < ke) {
        fetch(ng, nc, s);
        if (l2d > 0 && live && k + PF + l2d < ke) {  // DRAM -> L2 ahead, no registers held
          asm volatile("prefetch.global.L2 [%0];" ::"l"(ng + (int64_t)l2d * cells));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(nc + (int64_t)l2d * cells));
        }
        ng += cells;
        nc += cells;
      }
      walk_step(st, k - kb, live, e, l, r, u, d, c, nanf_, cb32);
      const float enc = st.enc;
      const bool gentle = st.gentle;
      if (live) *pe = enc;
      pe += L.sstride;
      const unsigned word = __ballot_sync(0xFFFFFFFFu, live && gentle);
      if (chgmap) {  // uniform
        const bool enc_changed = __any_sync(0xFFFFFFFFu, live && f32_bits(enc) != prev_enc);
        if (wlead && (k == kb || word != prev_word || enc_changed)) *pcm = 1;
        prev_word = word;
        prev_enc = f32_bits(enc);
      }
      if (wlead) *pb = word;
      pb += (int64_t)rows * wpr;
      pcm += cmstride;
    }
  }
}

template <int PF, bool CHUNKED = false>
__global__ void __launch_bounds__(kWalkNT) terrain_walk_kernel(
    const float *__restrict__ ground, const float *__restrict__ ceiling, int S, int rows,
    int cols, float *__restrict__ enc_out, EncLayout L, uint32_t *__restrict__ bits_out,
    int wpr, unsigned char *__restrict__ chgmap, int l2d) {
  if constexpr (CHUNKED) {  // blockIdx.y = chunk of slices (small maps: more threads in flight)
    const int kb = (int)((int64_t)S * blockIdx.y / gridDim.y);
    const int ke = (int)((int64_t)S * (blockIdx.y + 1) / gridDim.y);
    walk_body<PF>(ground, ceiling, S, rows, cols, enc_out, L, bits_out, wpr, chgmap, l2d, kb, ke);
  } else {
    walk_body<PF>(ground, ceiling, S, rows, cols, enc_out, L, bits_out, wpr, chgmap, l2d, 0, S);
  }
}

// ---------------------------------------------------------------------------
// Change masks + skipping walk.  A cell's encoded c_init and gentle flag at
// slice k are functions of its 5-point ground cross and its ceiling at k
// (walk_step recomputes only when those inputs change), and a plane cuts a
// surface in few cells: on the campus map 5.4 % of the cells' inputs change
// from one slice to the next, and only 7.3 % of the 32-cell warps see any
// change at a slice.  So:
//   change_mask_kernel: one streaming pass over ground / ceiling -> per cell
//     gm bit k = ground[k] differs (bitwise) from ground[k-1], cm the same
//     for the ceiling (bit 0 set), S <= 64;
//   terrain_walk_skip_kernel: as terrain_walk_kernel, but a warp ORs its
//     cells' input-change masks (own ground and ceiling, the 4 neighbours'
//     ground) and loads / computes only at the slices where some lane's
//     inputs changed; at the other slices every lane's encoded c_init and
//     gentle flag are the previous slice's, which are stored again (the
//     resolve / inflate kernel reads whole slices) -- no loads, no arithmetic.
// The per-lane "changed" tests are the masks themselves (no bit compares).
constexpr int kMaskNT = 256;

__global__ void __launch_bounds__(kMaskNT) change_mask_kernel(
    const float *__restrict__ ground, const float *__restrict__ ceiling, int S, int64_t cells,
    unsigned long long *__restrict__ gm, unsigned long long *__restrict__ cm) {
  const int64_t c = (int64_t)blockIdx.x * kMaskNT + threadIdx.x;
  if (c >= cells) return;
  constexpr int U = 8;  // independent loads in flight per array
  unsigned long long g = 1ull, m = 1ull;
  uint32_t pg = f32_bits(__ldcs(ground + c)), pc = f32_bits(__ldcs(ceiling + c));
  int k = 1;
  for (; k + U <= S; k += U) {
    uint32_t vg[U], vc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      vg[u] = f32_bits(__ldcs(ground + (int64_t)(k + u) * cells + c));
      vc[u] = f32_bits(__ldcs(ceiling + (int64_t)(k + u) * cells + c));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      g |= (unsigned long long)(vg[u] != pg) << (k + u);
      m |= (unsigned long long)(vc[u] != pc) << (k + u);
      pg = vg[u];
      pc = vc[u];
    }
  }
  for (; k < S; ++k) {
    const uint32_t vg = f32_bits(__ldcs(ground + (int64_t)k * cells + c));
    const uint32_t vc = f32_bits(__ldcs(ceiling + (int64_t)k * cells + c));
    g |= (unsigned long long)(vg != pg) << k;
    m |= (unsigned long long)(vc != pc) << k;
    pg = vg;
    pc = vc;
  }
  gm[c] = g;
  cm[c] = m;
}

__device__ __forceinline__ unsigned long long warp_or64(unsigned long long v) {
  const unsigned lo = __reduce_or_sync(0xFFFFFFFFu, (unsigned)v);
  const unsigned hi = __reduce_or_sync(0xFFFFFFFFu, (unsigned)(v >> 32));
  return ((unsigned long long)hi << 32) | lo;
}

// Sparse output (fresh != NULL): a warp writes its encoded c_init, gentle
// word and fresh byte (1 per slice, row and bitmap word) only at the slices
// it recomputed, plus every run-start slice of the resolve / inflate kernel
// (k % run == 0, loaded without a previous tile); that kernel takes the other
// cells of a loaded tile from its previous slice.  At the campus map this
// drops 93 % of the walk's stores.
template <bool CHUNKED>
#ifdef PCT_WALK_MINB
#define PCT_WALK_BOUNDS __launch_bounds__(kWalkNT, PCT_WALK_MINB)
#else
#define PCT_WALK_BOUNDS __launch_bounds__(kWalkNT)
#endif
__global__ void PCT_WALK_BOUNDS terrain_walk_skip_kernel(
    const float *__restrict__ ground, const float *__restrict__ ceiling, int S, int rows,
    int cols, float *__restrict__ enc_out, EncLayout L, uint32_t *__restrict__ bits_out,
    int wpr, unsigned char *__restrict__ chgmap, const unsigned long long *__restrict__ gmask,
    const unsigned long long *__restrict__ cmask, unsigned char *__restrict__ fresh, int fpitch,
    unsigned long long runmask) {
  int kb = 0, ke = S;
  if constexpr (CHUNKED) {  // blockIdx.y = chunk of slices (small maps: more threads in flight)
    kb = (int)((int64_t)S * blockIdx.y / gridDim.y);
    ke = (int)((int64_t)S * (blockIdx.y + 1) / gridDim.y);
  }
  const int64_t cells = (int64_t)rows * cols;
  const int64_t pidx = (int64_t)blockIdx.x * kWalkNT + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int pcols = wpr * 32;
  // (32-bit division when the padded grid has < 2^32 cells: a 64-bit
  // division by a run-time value is a ~100-instruction subroutine)
  const int i0_ = (int64_t)rows * pcols <= 0xFFFFFFFFll
                      ? (int)((uint32_t)pidx / (uint32_t)pcols)
                      : (int)(pidx / pcols);
  const int j0_ = (int)(pidx - (int64_t)i0_ * pcols);
  const bool live = i0_ < rows && j0_ < cols;
  const int i = i0_ < rows ? i0_ : rows - 1;
  const int j = j0_ < cols ? j0_ : cols - 1;  // clamped: address formation only
  const bool wlead = lane == 0 && i0_ < rows;
  const bool hl = live && j > 0, hr = live && j + 1 < cols, hu = live && i > 0,
             hd = live && i + 1 < rows;
  const bool edge_l = lane == 0 && hl, edge_r = lane == 31 && hr;
  const float nanf_ = bits_f32(kNaNBits);
  const float cb32 = (float)c_K.c_barrier;
  const int64_t base = (int64_t)i * cols + j;
  // input-change masks: cross (own + 4 neighbours' ground) and interval (+ ceiling)
  unsigned long long g_own = live ? __ldg(gmask + base) : 0ull;
  unsigned long long xm = g_own;
  if (hu) xm |= __ldg(gmask + base - cols);
  if (hd) xm |= __ldg(gmask + base + cols);
  unsigned long long gl = __shfl_up_sync(0xFFFFFFFFu, g_own, 1);
  unsigned long long gr = __shfl_down_sync(0xFFFFFFFFu, g_own, 1);
  if (lane == 0) gl = edge_l ? __ldg(gmask + base - 1) : 0ull;
  if (lane == 31) gr = edge_r ? __ldg(gmask + base + 1) : 0ull;
  if (hl) xm |= gl;
  if (hr) xm |= gr;
  const unsigned long long first = 1ull << kb;  // a chunk's first slice is computed in full
  xm |= first;
  const unsigned long long im = xm | (live ? __ldg(cmask + base) : 0ull);
  const unsigned long long W = warp_or64(live ? im : first);  // warp-uniform
  const unsigned long long kmask = ke >= 64 ? ~0ull : ((1ull << ke) - 1ull);
  unsigned long long todo = W & kmask & ~((1ull << kb) - 1ull);

  float *pe = enc_out + L.at(kb, i, j);
  const int64_t bstride = (int64_t)rows * wpr;
  uint32_t *pb = bits_out + (int64_t)kb * bstride + (int64_t)i * wpr + (j0_ >> 5);
  const int64_t cmstride = (int64_t)((rows + 7) >> 3) * wpr;
  unsigned char *pcm = chgmap ? chgmap + (int64_t)(i >> 3) * wpr + (j0_ >> 5) : nullptr;

  // loads of one slice (grid borders read NaN)
  float qe, qu, qd, qc, ql, qr;
  auto fetch = [&](int k) {
    const float *g = ground + base + (int64_t)k * cells;
    qe = live ? __ldg(g) : nanf_;
    qu = hu ? __ldg(g - cols) : nanf_;
    qd = hd ? __ldg(g + cols) : nanf_;
    qc = live ? __ldg(ceiling + base + (int64_t)k * cells) : nanf_;
    ql = edge_l ? __ldg(g - 1) : nanf_;
    qr = edge_r ? __ldg(g + 1) : nanf_;
  };
  int knext = todo ? __ffsll((long long)todo) - 1 : ke;  // next slice with a change
  if (knext < ke) fetch(knext);
  WalkState st;
  st.tenc = nanf_;
  uint32_t prev_enc = 0u;
  unsigned word = 0u, prev_word = 0u;
  // one slice where some lane's inputs changed: loads (the next such slice's
  // issued before the arithmetic), walk_step, gentle word, change-map byte
  auto compute = [&](int k) {
    const float e = qe, u = qu, d = qd, c = qc;
    float l = __shfl_up_sync(0xFFFFFFFFu, e, 1);
    float r = __shfl_down_sync(0xFFFFFFFFu, e, 1);
    if (lane == 0) l = ql;
    if (lane == 31) r = qr;
    if (!hl) l = nanf_;
    if (!hr) r = nanf_;
    todo &= todo - 1ull;
    knext = todo ? __ffsll((long long)todo) - 1 : ke;
    if (knext < ke) fetch(knext);  // in flight while this slice computes
    const bool xch = (xm >> k) & 1ull, ich = (im >> k) & 1ull;
    if (xch && live && !finite32(e)) {  // no ground: nothing to grade (fast_terrain's result)
      st.gentle = false;
      st.tenc = nanf_;
    } else if (xch && live) {
      const FastCell t = fast_terrain(Cross{e, l, r, u, d}, c_K);
      st.gentle = t.gentle;
      if (!t.valid) {
        st.tenc = nanf_;
      } else if (t.isolated || t.m_xy > c_K.theta_b) {
        st.tenc = cb32;
      } else if (t.gentle) {
        st.tenc = gentle_cost32(t.gx, t.gy, t.s, c_K);
      } else {
        const double q = div_const(t.m_xy, c_K.theta_b, c_K.inv_theta_b);
        st.tenc = bits_f32(f32_bits((float)(c_K.alpha_b * (q * q))) | 0x80000000u);
      }
    }
    if (ich && live) {
      if (!finite32(st.tenc)) {
        st.enc = cb32;  // no ground: barrier (fuse_costs :169)
      } else {
        const uint32_t tb = f32_bits(st.tenc);
        st.enc = fuse_value(interval_value(e, c, c_K), bits_f32(tb & 0x7FFFFFFFu), c_K);
        if (tb & 0x80000000u) st.enc = bits_f32(f32_bits(st.enc) | 0x80000000u);
      }
    }
    word = __ballot_sync(0xFFFFFFFFu, live && st.gentle);
    if (pcm) {
      const bool enc_changed = __any_sync(0xFFFFFFFFu, live && f32_bits(st.enc) != prev_enc);
      if (wlead && (k == kb || word != prev_word || enc_changed)) pcm[(int64_t)k * cmstride] = 1;
    }
    prev_word = word;
    prev_enc = f32_bits(st.enc);
  };
  if (!fresh) {  // dense output: every slice written
    // runs of slices without an event repeat the current values (a tight
    // store loop); an event slice computes first
    int k = kb;
    while (true) {
      const int kstop = knext < ke ? knext : ke;  // uniform
#pragma unroll 2
      for (; k < kstop; ++k) {
        if (live) *pe = st.enc;
        pe += L.sstride;
        if (wlead) *pb = word;
        pb += bstride;
      }
      if (k >= ke) break;
      compute(k);
      if (live) *pe = st.enc;
      pe += L.sstride;
      if (wlead) *pb = word;
      pb += bstride;
      ++k;
    }
    return;
  }
  // sparse output: only the slices this warp recomputed, and the run starts
  // of the resolve / inflate kernel (loaded whole, without a previous slice)
  unsigned long long ev = todo;
  ev |= runmask & kmask & ~((1ull << kb) - 1ull);  // run starts (host-built bits k % run == 0)
  float *pe0 = enc_out + L.at(0, i, j);
  uint32_t *pb0 = bits_out + (int64_t)i * wpr + (j0_ >> 5);
  unsigned char *pf0 = fresh + (int64_t)i * fpitch + (j0_ >> 5);
  while (ev) {
    const int k = __ffsll((long long)ev) - 1;
    ev &= ev - 1ull;
    if (k == knext) compute(k);  // uniform
    if (live) pe0[(int64_t)k * L.sstride] = st.enc;
    if (wlead) {
      pb0[(int64_t)k * bstride] = word;
      pf0[(int64_t)k * rows * fpitch] = 1;
    }
  }
}

// per-map arguments of the split evaluation (a single map is a batch of one)
struct EvalMap {
  CUtensorMap tmap;  // encoded c_init stack (TMA), 64-byte aligned first member
  CUtensorMap omap;  // cost stack (TMA store of output tiles), valid when ostore
  const float *ground, *ceiling;
  float *enc, *cost;
  uint32_t *bits;
  EncLayout L;
  int S, rows, cols, wpr, run;
  int64_t words;  // gentle bitmap words per slice
  unsigned char *chg;  // change map of the walk ((rows + 7) / 8 x wpr bytes per slice)
  // sparse walk output: fresh[(k * rows + i) * fpitch + w] = 1 where the walk
  // wrote slice k's c_init / gentle word w of row i (NULL: every slice written)
  const unsigned char *fresh;
  int fpitch;
  int ostore;  // output tiles leave by TMA bulk tensor stores (omap)
  // per output tile (S <= 64): bit k = the tile's outputs may differ from
  // slice k-1 (NULL: not recorded); read by the simplify window
  unsigned long long *tcm;
};

// walk over a batch: blockIdx.y = map; blocks past the map's extent leave
template <int PF>
__global__ void __launch_bounds__(kWalkNT) terrain_walk_batch_kernel(const EvalMap *__restrict__ maps) {
  const EvalMap &m = maps[blockIdx.y];
  if ((int64_t)blockIdx.x * kWalkNT >= (int64_t)m.rows * m.wpr * 32) return;  // whole block
  // no L2 look-ahead for batches of small maps (measured slower: cfg4
  // evaluate 1.97 -> 2.07 ms)
  walk_body<PF>(m.ground, m.ceiling, m.S, m.rows, m.cols, m.enc, m.L, m.bits, m.wpr, m.chg, 0, 0,
                m.S);
}

template <int R, int PR, int TH, int TW>
struct SplitGeom {
  static constexpr int CH = TH + 2 * R, CW = TW + 2 * R;
  static constexpr int GH = CH + 2 * PR, GW = CW + 2 * PR;
  static constexpr int GWW = (GW + 31) / 32 + 1;
  static constexpr int O_CI = 0;
  static constexpr int O_BITS = O_CI + CH * CW * 4;
  static constexpr int O_LIST = O_BITS + GH * GWW * 4;
  static constexpr int SMEM = O_LIST + ((CH * CW * 2 + 15) / 16) * 16;
};

template <int R, int PR, int TH, int TW, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) resolve_inflate_kernel(
    const float *__restrict__ enc, EncLayout L, const uint32_t *__restrict__ bits_in, int rows,
    int cols, int64_t words, float *__restrict__ cost) {
  using G = SplitGeom<R, PR, TH, TW>;
  extern __shared__ __align__(16) unsigned char smem[];
  float *cinit = reinterpret_cast<float *>(smem + G::O_CI);
  uint32_t *bits = reinterpret_cast<uint32_t *>(smem + G::O_BITS);
  uint16_t *flist = reinterpret_cast<uint16_t *>(smem + G::O_LIST);
  __shared__ int n_flagged;
  const int tid = threadIdx.x;
  const int64_t cells = (int64_t)rows * cols;
  const int k = blockIdx.z;
  const int i0 = blockIdx.y * TH, j0 = blockIdx.x * TW;
  const uint32_t *bk = bits_in + (int64_t)k * words;
  const int wpr = (cols + 31) / 32;
  if (tid == 0) n_flagged = 0;
  __syncthreads();

  // encoded c_init of the tile + R halo from the zero-padded layout (no bounds
  // tests; float4 when the padding keeps rows aligned); foothold-branch cells
  // go to a list
  const float *ek = enc + L.at(k, i0 - R, j0 - R);
  auto note = [&](int idx, float v) {
    const bool flagged = (f32_bits(v) & 0x80000000u) != 0;
    const unsigned act = __activemask();
    const unsigned fm = __ballot_sync(act, flagged);
    if (fm) {
      const int lane = tid & 31, leader = __ffs(fm) - 1;
      int base = 0;
      if (lane == leader) base = atomicAdd(&n_flagged, __popc(fm));
      base = __shfl_sync(act, base, leader);
      if (flagged) flist[base + __popc(fm & ((1u << lane) - 1u))] = (uint16_t)idx;
    }
  };
  if constexpr (G::CW % 4 == 0 && R % 4 == 0) {
    constexpr int CW4 = G::CW / 4;
    for (int q = tid; q < G::CH * CW4; q += NT) {
      const int y = q / CW4, x4 = q - y * CW4;
      const float4 v = __ldg(reinterpret_cast<const float4 *>(ek + (int64_t)y * L.pitch) + x4);
      const int idx = y * G::CW + 4 * x4;
      reinterpret_cast<float4 *>(cinit)[q] = v;
      if ((f32_bits(v.x) | f32_bits(v.y) | f32_bits(v.z) | f32_bits(v.w)) & 0x80000000u) {
        if (f32_bits(v.x) & 0x80000000u) note(idx, v.x);
        if (f32_bits(v.y) & 0x80000000u) note(idx + 1, v.y);
        if (f32_bits(v.z) & 0x80000000u) note(idx + 2, v.z);
        if (f32_bits(v.w) & 0x80000000u) note(idx + 3, v.w);
      }
    }
  } else {
    for (int idx = tid; idx < G::CH * G::CW; idx += NT) {
      const int y = idx / G::CW, x = idx - y * G::CW;
      const float v = __ldg(ek + (int64_t)y * L.pitch + x);
      cinit[idx] = v;
      if (f32_bits(v) & 0x80000000u) note(idx, v);
    }
  }
  // gentle bits of the window region (rows i0-R-r .., cols j0-R-r ..), cut
  // out of the row-major bitmap; columns outside the map read as 0
  for (int idx = tid; idx < G::GH * G::GWW; idx += NT) {
    const int y = idx / G::GWW, w = idx - y * G::GWW;
    const int gi = i0 - R - PR + y;
    const int gj = j0 - R - PR + 32 * w;  // column of bit 0 of this word
    uint32_t word = gentle_word(bk, wpr, gi, gj, rows, cols);
    if (32 * w >= G::GW) word = 0;
    else if (G::GW - 32 * w < 32) word &= (1u << (G::GW - 32 * w)) - 1u;
    bits[idx] = word;
  }
  __syncthreads();

  constexpr int SIDE = 2 * PR + 1;
  constexpr uint32_t WMASK = (1u << SIDE) - 1u;
  const int nf = n_flagged;
  for (int t = tid; t < nf; t += NT) {
    const int idx = flist[t];
    const int y = idx / G::CW, x = idx - y * G::CW;
    const int w = x >> 5, sh = x & 31;
    int cnt = 0;
#pragma unroll
    for (int d = 0; d < SIDE; ++d) {
      const uint32_t *rw = bits + (y + d) * G::GWW + w;
      const uint64_t v = (uint64_t)rw[0] | ((uint64_t)rw[1] << 32);
      cnt += __popc((uint32_t)(v >> sh) & WMASK);
    }
    cinit[idx] = cinit_resolve(cinit[idx], cnt, c_K);
  }
  __syncthreads();

  float *out = cost + (int64_t)k * cells;
  if constexpr (R <= 4) {
    constexpr int STRIPS = NT / TW;
    constexpr int V = TH / STRIPS;
    const int x = tid % TW, s = tid / TW;
    inflate_sym_strip<R, V>(cinit, G::CW, x, s * V, out, cols, i0 + s * V, j0 + x, rows, cols);
  }
}

// ---------------------------------------------------------------------------
// I, TMA version: persistent CTAs; the encoded c_init tile + halo of the next
// work item is fetched by the Tensor Memory Accelerator
// (cp.async.bulk.tensor.3d, completion on an mbarrier) into the second of
// two shared-memory buffers while the current item is resolved and inflated.
#include "bulk.cuh"  // smem_u32, mbarrier helpers
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar, int x,
                                            int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// shared -> global bulk tensor store (async proxy; the caller fences the
// shared-memory writes it covers and waits before overwriting the source)
__device__ __forceinline__ void tma_store_3d(const CUtensorMap *map, const void *src, int x, int y,
                                             int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(map),
      "r"(x), "r"(y), "r"(z), "r"(smem_u32(src))
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int R, int PR, int TH, int TW>
struct TmaGeom {
  static constexpr int CH = TH + 2 * R, CW = TW + 2 * R;
  static constexpr int GH = CH + 2 * PR, GW = CW + 2 * PR;
  static constexpr int GWW = (GW + 31) / 32 + 1;
  static constexpr int BUF = ((CH * CW * 4) + 127) / 128 * 128;  // one TMA box, 128 B aligned
  static constexpr int O_BUF = 0;                                 // 2 buffers
  static constexpr int O_BITS = 2 * BUF;
  static constexpr int O_LIST = O_BITS + GH * GWW * 4;
  static constexpr int O_BAR = O_LIST + ((CH * CW * 2 + 15) / 16) * 16;  // 2 mbarriers + counter
  static constexpr int SMEM = O_BAR + 32;
};

template <int R, int PR, int TH, int TW, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) resolve_inflate_tma_kernel(
    const __grid_constant__ CUtensorMap enc_map, const uint32_t *__restrict__ bits_in, int rows,
    int cols, int S, int64_t words, float *__restrict__ cost) {
  using G = TmaGeom<R, PR, TH, TW>;
  // everything lives in the dynamic region (no static __shared__), whose base
  // is 128-byte aligned as the TMA destination requires; constant offsets
  // keep the compiler on the shared address space (LDS/STS, not generic LD)
  extern __shared__ __align__(128) unsigned char smem[];
  uint32_t *bits = reinterpret_cast<uint32_t *>(smem + G::O_BITS);
  uint16_t *flist = reinterpret_cast<uint16_t *>(smem + G::O_LIST);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + G::O_BAR);
  int &n_flagged = *reinterpret_cast<int *>(smem + G::O_BAR + 16);
  const int tid = threadIdx.x;
  if (tid == 0 && (smem_u32(smem) & 127u) != 0u) __trap();  // TMA box alignment
  const int tx = (cols + TW - 1) / TW, ty = (rows + TH - 1) / TH;
  const int tiles = tx * ty;
  const int n_items = tiles * S;
  const int64_t cells = (int64_t)rows * cols;
  constexpr uint32_t BOX_BYTES = G::CH * G::CW * 4;
  auto coords = [&](int item, int &i0, int &j0, int &k) {
    k = item / tiles;
    const int t = item - k * tiles;
    i0 = (t / tx) * TH;
    j0 = (t % tx) * TW;
  };
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int item = blockIdx.x;
  if (tid == 0 && item < n_items) {
    int i0, j0, k;
    coords(item, i0, j0, k);
    mbar_expect_tx(&bar[0], BOX_BYTES);
    tma_load_3d(smem + G::O_BUF, &enc_map, &bar[0], j0, i0, k);  // padded coords
  }
  uint32_t phase[2] = {0u, 0u};
  for (int it = 0; item < n_items; ++it, item += gridDim.x) {
    const int cur = it & 1;
    float *cinit = reinterpret_cast<float *>(smem + G::O_BUF + cur * G::BUF);
    int i0, j0, k;
    coords(item, i0, j0, k);
    // prefetch the next item into the other buffer (freed by the barrier that
    // ended the previous iteration)
    const int nxt = item + gridDim.x;
    if (tid == 0 && nxt < n_items) {
      int ni0, nj0, nk;
      coords(nxt, ni0, nj0, nk);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&bar[cur ^ 1], BOX_BYTES);
      tma_load_3d(smem + G::O_BUF + (cur ^ 1) * G::BUF, &enc_map, &bar[cur ^ 1], nj0, ni0, nk);
    }
    if (tid == 0) n_flagged = 0;
    // gentle bits of the window region (global bitmap -> smem), overlapping the TMA
    const uint32_t *bk = bits_in + (int64_t)k * words;
    const int wpr = (cols + 31) / 32;
    for (int idx = tid; idx < G::GH * G::GWW; idx += NT) {
      const int y = idx / G::GWW, w = idx - y * G::GWW;
      const int gi = i0 - R - PR + y;
      const int gj = j0 - R - PR + 32 * w;
      uint32_t word = gentle_word(bk, wpr, gi, gj, rows, cols);
      if (32 * w >= G::GW) word = 0;
      else if (G::GW - 32 * w < 32) word &= (1u << (G::GW - 32 * w)) - 1u;
      bits[idx] = word;
    }
    mbar_wait(&bar[cur], phase[cur]);
    phase[cur] ^= 1u;
    __syncthreads();  // bits + n_flagged visible, TMA data landed
    // foothold-branch cells of the tile + halo
    for (int idx = tid; idx < G::CH * G::CW; idx += NT) {
      const bool flagged = (f32_bits(cinit[idx]) & 0x80000000u) != 0;
      const unsigned act = __activemask();
      const unsigned fm = __ballot_sync(act, flagged);
      if (fm) {
        const int lane = tid & 31, leader = __ffs(fm) - 1;
        int base = 0;
        if (lane == leader) base = atomicAdd(&n_flagged, __popc(fm));
        base = __shfl_sync(act, base, leader);
        if (flagged) flist[base + __popc(fm & ((1u << lane) - 1u))] = (uint16_t)idx;
      }
    }
    __syncthreads();
    constexpr int SIDE = 2 * PR + 1;
    constexpr uint32_t WMASK = (1u << SIDE) - 1u;
    const int nf = n_flagged;
    for (int t = tid; t < nf; t += NT) {
      const int idx = flist[t];
      const int y = idx / G::CW, x = idx - y * G::CW;
      const int w = x >> 5, sh = x & 31;
      int cnt = 0;
#pragma unroll
      for (int d = 0; d < SIDE; ++d) {
        const uint32_t *rw = bits + (y + d) * G::GWW + w;
        const uint64_t v = (uint64_t)rw[0] | ((uint64_t)rw[1] << 32);
        cnt += __popc((uint32_t)(v >> sh) & WMASK);
      }
      cinit[idx] = cinit_resolve(cinit[idx], cnt, c_K);
    }
    __syncthreads();
    float *out = cost + (int64_t)k * cells;
    if constexpr (R <= 4) {
      constexpr int STRIPS = NT / TW;
      constexpr int V = TH / STRIPS;
      const int x = tid % TW, s = tid / TW;
      inflate_sym_strip<R, V>(cinit, G::CW, x, s * V, out, cols, i0 + s * V, j0 + x, rows, cols);
    }
    __syncthreads();  // buffer `cur` and the bit rows are free again
  }
}
