// k_eval_bnb.cuh — resolve + branch-and-bound inflation (included by
// k_evaluate.cu inside namespace pct::{anon}, after k_eval_split.cuh whose TMA
// helpers, EncLayout and terrain walk it shares).
//
// inflate (traversability.py:205-213) is out = max_k fl32(w_k * M_k), M_k the
// max of c_init over the taps of weight class k (w_1 > w_2 > ... > 0).  All
// c_init >= 0 and x -> fl32(w x) is monotone, so with U >= every M_k:
//   * once acc >= fl32(w_k * U), no class k' >= k can raise acc (branch and
//     bound over the classes in weight order);
//   * class 1 (weight 1 for Table-I parameters: the disk d <= d_inf) is a
//     small disk whose max D1 is a separable max filter.
// Per tile and slice:
//   P0  gentle bits of the foothold window (global bitmap -> smem), TMA'd
//       encoded c_init tile + halo; vertical gentle counts of the (2r+1)-row
//       window, bit-sliced (one plane per count bit, 32 columns per word);
//       foothold-branch cells resolved in place (3-4 funnel-shift popcounts)
//   P1  maxima of aligned R x R blocks of c_init, and the horizontal maxima
//       planes H_h(y, x) = max c(y, x-h .. x+h) the disk needs
//   P2  U(output block) = max of its 3 x 3 neighbouring blocks (covers every
//       tap of the (2R+1)^2 window); D1 per output from the planes; outputs
//       with fl32(w_1 D1) >= fl32(w_2 U) are final (~80 % on the config maps),
//       the rest go to a list
//   P3  listed outputs walk the remaining classes (compiled ring offsets,
//       bnb_rings.h) until the bound stops them
// The class structure is compiled per R (R=4: r_g 0.1, R=8: r_g 0.05 with the
// Table-I d_inf / d_sm); the host checks the caller's kernel against it and
// otherwise keeps the full-tap kernels.

#include "bnb_rings.h"

constexpr int kBnbMaxClasses = 64;
__constant__ float c_bw[kBnbMaxClasses + 1];  // class weights, descending; c_bw[n] = 0

// half-widths of the class-1 disk per row offset |a|
template <int R>
struct DiskShape;
template <>
struct DiskShape<4> {  // a^2 + b^2 <= 4: 13 taps
  static constexpr int A = 2;
  static constexpr int h[3] = {2, 1, 0};
};
template <>
struct DiskShape<8> {  // a^2 + b^2 <= 16: 49 taps
  static constexpr int A = 4;
  static constexpr int h[5] = {4, 3, 3, 2, 0};
};

constexpr int count_bits(int n) { return n < 2 ? 1 : 1 + count_bits(n / 2); }

template <int R, int PR, int TH, int TW, bool SP = false>
struct BnbGeom {
  static constexpr int CH = TH + 2 * R, CW = TW + 2 * R;  // c_init tile + halo
  static constexpr int GH = CH + 2 * PR, GW = CW + 2 * PR;
  static constexpr int GWW = (GW + 31) / 32 + 1;
  static constexpr int CWW = (CW + 31) / 32;            // words of one foothold-ok row
  static constexpr int SIDE = 2 * PR + 1;
  static constexpr int NVP = count_bits(SIDE);          // bit planes of a column count
  static constexpr int NSB = count_bits(SIDE * SIDE);   // bit planes of a window count
  static constexpr int BUF = ((CH * CW * 4) + 127) / 128 * 128;
  static constexpr int NBUF = 3;              // previous, current, prefetched slice
  static constexpr int NPL = R == 4 ? 1 : 2;  // planes: R=4 H1; R=8 H3, H2
  static constexpr int PLANE = CH * TW;       // floats per plane
  static constexpr int NBY = CH / R, NBX = CW / R;  // c_init blocks (upper bound)
  static constexpr int QY = TH / R, QX = TW / R;    // output blocks (upper bound)
  static constexpr int CBY = CH / 4, CBX = CW / 4;  // 4x4 c_init change blocks
  static constexpr int DBY = TH / 4, DBX = TW / 4;  // 4x4 output dirty blocks
  static constexpr int SPAN = (3 + 2 * R) / 4 + 1;  // change blocks under one dirty block
  // regions (no aliasing: without a barrier at the end of a slice, P0 of the
  // next slice overlaps P3 / P4 of this one)
  static constexpr int O_BUF = 0;
  static constexpr int O_PL = NBUF * BUF;
  static constexpr int O_BITS = O_PL + NPL * PLANE * 4;
  static constexpr int O_OK = O_BITS + ((GH * GWW * 4 + 15) / 16) * 16;
  static constexpr int O_OT = ((O_OK + CH * CWW * 4 + 127) / 128) * 128;  // output tile (TMA store source)
  static constexpr int O_SL = O_OT + TH * TW * 4;                      // u16 list
  // list capacity: every warp's P2 outputs, i.e. TH x TW/4 groups rounded up
  // to whole passes of the CTA (up to 256 threads) x 4 outputs
  static constexpr int SLN = (TH * (TW / 4) + 255) / 256 * 256 * 4;
  static constexpr int O_BM = O_SL + ((SLN * 2 + 15) / 16) * 16;
  static constexpr int O_U = O_BM + ((NBY * NBX * 4 + 15) / 16) * 16;
  static constexpr int O_CB = O_U + ((QY * QX * 4 + 15) / 16) * 16;     // u8 change blocks
  static constexpr int O_DB = O_CB + ((CBY * CBX + 15) / 16) * 16;      // u8 dirty blocks
  // sparse walk output: the tile + halo's encoded c_init and the raw gentle
  // source words of the window as of the last loaded slice, and the fresh
  // flags of the current slice (one per row and source word)
  // (only the sparse instantiation, SP, has them: the others keep the
  // occupancy of the plain kernel)
  static constexpr int NSW = GWW + 1;
  static constexpr int O_RAWC = O_DB + ((DBY * DBX + 15) / 16) * 16;
  static constexpr int O_RAWW = O_RAWC + (SP ? BUF : 0);
  static constexpr int O_FRB = O_RAWW + (SP ? ((GH * NSW * 4 + 15) / 16) * 16 : 0);
  static constexpr int O_BAR = O_FRB + (SP ? ((GH * NSW + 15) / 16) * 16 : 0);
  static constexpr int SMEM = O_BAR + 128;  // 3 mbarriers, 3 x 2 coordinate slots, warp counts
  static_assert(TH % R == 0 && TW % R == 0 && CW % 4 == 0 && R % 4 == 0, "bnb tile geometry");
  static_assert(TW % 32 == 0, "sparse merge: 4-cell groups never straddle a bitmap word");
  static_assert(O_OT % 128 == 0, "TMA store source alignment");
  static_assert(TH * TW <= 65536, "u16 output indices");
  static_assert((TH * (TW / 4)) % 32 == 0, "warp-uniform output loop (ballots)");
  static_assert(SIDE <= 31 && NSB <= 10, "foothold window");
};

__device__ __forceinline__ float fmax3(float a, float b, float c) { return fmaxf(fmaxf(a, b), c); }
__device__ __forceinline__ float4 lds4(const float *p) { return *reinterpret_cast<const float4 *>(p); }

// full adder on 32 bit-slices: s = a ^ b ^ c, k = majority(a, b, c)
__device__ __forceinline__ void fadd(uint32_t a, uint32_t b, uint32_t c, uint32_t &s,
                                     uint32_t &k) {
  s = a ^ b ^ c;
  k = (a & b) | (c & (a ^ b));
}

// per-column counts of N one-bit rows, bit-sliced into NB planes
template <int N, int NB>
__device__ __forceinline__ void column_count(const uint32_t (&x)[N], uint32_t (&o)[NB]) {
  if constexpr (N == 7 && NB == 3) {
    uint32_t s1, c1, s2, c2, c3;
    fadd(x[0], x[1], x[2], s1, c1);
    fadd(x[3], x[4], x[5], s2, c2);
    fadd(s1, s2, x[6], o[0], c3);
    fadd(c1, c2, c3, o[1], o[2]);
  } else if constexpr (N == 13 && NB == 4) {
    uint32_t s1, c1, s2, c2, s3, c3, s4, c4, t1, d1, d2, u1, e1, u2, e2;
    fadd(x[0], x[1], x[2], s1, c1);
    fadd(x[3], x[4], x[5], s2, c2);
    fadd(x[6], x[7], x[8], s3, c3);
    fadd(x[9], x[10], x[11], s4, c4);
    fadd(s1, s2, s3, t1, d1);
    fadd(t1, s4, x[12], o[0], d2);
    fadd(c1, c2, c3, u1, e1);
    fadd(c4, d1, d2, u2, e2);
    o[1] = u1 ^ u2;
    fadd(e1, e2, u1 & u2, o[2], o[3]);
  } else {  // ripple accumulation
#pragma unroll
    for (int p = 0; p < NB; ++p) o[p] = 0u;
#pragma unroll
    for (int d = 0; d < N; ++d) {
      uint32_t c = x[d];
#pragma unroll
      for (int p = 0; p < NB; ++p) {
        const uint32_t t = o[p] & c;
        o[p] ^= c;
        c = t;
      }
    }
  }
}

// a += b << sh on bit-sliced numbers (NA planes, result truncated to NA)
template <int NA, int NB>
__device__ __forceinline__ void bs_add(uint32_t (&a)[NA], const uint32_t (&b)[NB], int sh) {
  uint32_t c = 0u;
#pragma unroll
  for (int p = 0; p < NA; ++p) {
    const int q = p - sh;
    const uint32_t y = (q >= 0 && q < NB) ? b[q] : 0u;
    const uint32_t s = a[p] ^ y ^ c;
    c = (a[p] & y) | (c & (a[p] ^ y));
    a[p] = s;
  }
}

// 32 lanes of "a >= t" for a bit-sliced a (NA planes) and a scalar t
template <int NA>
__device__ __forceinline__ uint32_t bs_ge(const uint32_t (&a)[NA], int t) {
  if (t <= 0) return 0xFFFFFFFFu;
  if (t >= (1 << NA)) return 0u;
  uint32_t borrow = 0u;  // a - t, from bit 0 up
#pragma unroll
  for (int p = 0; p < NA; ++p) {
    const uint32_t tb = ((t >> p) & 1) ? 0xFFFFFFFFu : 0u;
    borrow = (~a[p] & tb) | (~(a[p] ^ tb) & borrow);
  }
  return ~borrow;
}

// max over the ring taps T .. E-1 (compile-time offsets)
template <int R, int CW, int T, int E>
__device__ __forceinline__ float ring_max(const float *__restrict__ ctr, float m) {
  using RG = BnbRings<R>;
  if constexpr (T + 1 < E) {
    constexpr int o0 = RG::dy(T) * CW + RG::dx(T), o1 = RG::dy(T + 1) * CW + RG::dx(T + 1);
    return ring_max<R, CW, T + 2, E>(ctr, fmax3(m, ctr[o0], ctr[o1]));
  } else if constexpr (T < E) {
    constexpr int o0 = RG::dy(T) * CW + RG::dx(T);
    return fmaxf(m, ctr[o0]);
  } else {
    return m;
  }
}

// remaining classes K.. of the listed output at ctr under the bound U
template <int R, int CW, int K>
__device__ __forceinline__ void slow_classes(const float *__restrict__ ctr, float U, bool live,
                                             float &acc) {
  using RG = BnbRings<R>;
  if constexpr (K < RG::NCLS) {
    const float wk = c_bw[K];
    live = live && acc < wk * U;
    if (!__any_sync(0xFFFFFFFFu, live)) return;
    if (live) acc = fmaxf(acc, wk * ring_max<R, CW, RG::start(K), RG::start(K + 1)>(ctr, 0.0f));
    slow_classes<R, CW, K + 1>(ctr, U, live, acc);
  }
}

// Persistent CTAs over work items = (tile, run of consecutive slices).  The
// first slice of a run computes every output; later slices compare the
// resolved c_init tile + halo with the previous slice's (kept in the third
// TMA buffer) per 4 x 4 block and recompute only the 4 x 4 output blocks
// whose (2R+1)^2 windows touch a changed block: an output is a function of
// the resolved c_init in its window alone, so the others keep their values
// (the output tile lives in shared memory and is stored every slice).
template <int R, int PR, int TH, int TW, int NT, int MINB, bool SP = false>
__global__ void __launch_bounds__(NT, MINB) resolve_inflate_bnb_kernel(
    const EvalMap *__restrict__ maps, const int *__restrict__ item_off, int n_maps,
    int *__restrict__ work = nullptr) {
  using G = BnbGeom<R, PR, TH, TW, SP>;
  constexpr int NWARP = NT / 32;
  // list entries per warp: its P2 outputs (4 per thread per pass over the
  // TH x TW/4 output groups)
  constexpr int WSEG = (TH * (TW / 4) + NT - 1) / NT * 32 * 4;
  static_assert(NWARP * WSEG <= G::SLN, "bnb output list capacity");
  static_assert((TH * TW) % NWARP == 0 && NWARP <= 32, "warp list segments");
  extern __shared__ __align__(128) unsigned char smem[];
  uint32_t *bits = reinterpret_cast<uint32_t *>(smem + G::O_BITS);
  uint32_t *okb = reinterpret_cast<uint32_t *>(smem + G::O_OK);   // [CH][CWW]
  float *planes = reinterpret_cast<float *>(smem + G::O_PL);
  float *ot = reinterpret_cast<float *>(smem + G::O_OT);
  uint16_t *slist = reinterpret_cast<uint16_t *>(smem + G::O_SL);
  uint32_t *bm = reinterpret_cast<uint32_t *>(smem + G::O_BM);    // block maxima (float bits)
  float *ub = reinterpret_cast<float *>(smem + G::O_U);
  unsigned char *chg = smem + G::O_CB;
  unsigned char *dirty = smem + G::O_DB;
  float *rawc = reinterpret_cast<float *>(smem + G::O_RAWC);
  uint32_t *raww = reinterpret_cast<uint32_t *>(smem + G::O_RAWW);
  unsigned char *frb = smem + G::O_FRB;
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + G::O_BAR);  // [3]
  int *slot = reinterpret_cast<int *>(smem + G::O_BAR + 32);      // [3][3]
  int *wcnt = reinterpret_cast<int *>(smem + G::O_BAR + 72);      // [NWARP]
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  uint16_t *wlist = slist + warp * WSEG;
  if (tid == 0 && (smem_u32(smem) & 127u) != 0u) __trap();
  // work items: (map, run of slices, tile), maps concatenated (item_off:
  // first item of each map); a single map is a batch of one
  const int n_items = item_off[n_maps];
  auto decode = [&](int g, int &m, int &r, int &t) {
    int lo = 0, hi = n_maps - 1;  // last m with item_off[m] <= g
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (item_off[mid] <= g) lo = mid;
      else hi = mid - 1;
    }
    m = lo;
    const EvalMap &M = maps[m];
    const int tiles = ((M.cols + TW - 1) / TW) * ((M.rows + TH - 1) / TH);
    const int local = g - item_off[m];
    r = local / tiles;
    t = local - r * tiles;
  };
  auto origin = [&](const EvalMap &M, int t, int &i0, int &j0) {
    const int tx = (M.cols + TW - 1) / TW;
    const int ti = t / tx;
    i0 = ti * TH;
    j0 = (t - ti * tx) * TW;
  };
  constexpr uint32_t BOX_BYTES = G::CH * G::CW * 4;
  // the output tile of one slice from shared memory: float4 stores when the
  // rows are 16-byte aligned (cols % 4 == 0) and the tile is whole in x
  auto store_tile = [&](float *plane, int rows, int cols, int i0, int j0, int tid) {
    static_assert(NT % TW == 0 && TW % 4 == 0 && NT % (TW / 4) == 0, "store layout");
    const int imax = min(TH, rows - i0);
    if ((cols & 3) == 0 && j0 + TW <= cols) {
      constexpr int Q = TW / 4, RPS = NT / Q;
      const int q = tid % Q, r0 = tid / Q;
      for (int i = r0; i < imax; i += RPS)
        reinterpret_cast<float4 *>(plane + (int64_t)(i0 + i) * cols + j0)[q] =
            reinterpret_cast<const float4 *>(ot + i * TW)[q];
    } else {
      constexpr int RPS = NT / TW;  // rows per pass
      const int x = tid % TW, r0 = tid / TW;
      if (j0 + x < cols) {
        float *o = plane + (int64_t)(i0 + r0) * cols + (j0 + x);
        for (int i = r0; i < imax; i += RPS, o += (int64_t)RPS * cols) *o = ot[i * TW + x];
      }
    }
  };
  const float w0 = c_bw[0], w1 = c_bw[1];
  const uint32_t cb_bits = f32_bits((float)c_K.c_barrier);
  // Loads: only steps that are not skipped load their tile (TMA into buffer
  // (#loads issued) % 3); a step consumes the loads in issue order, so its
  // buffer is (#loads consumed) % 3 and the previous loaded tile is the one
  // before.  Thread 0 keeps one load in flight, for the next step to load.
  int acq_m = -1, ld = 0;  // thread 0
  bool pending = false;    // thread 0
  auto issue = [&](int m, int t, int k) {
    const EvalMap &M = maps[m];
    int i0, j0;
    origin(M, t, i0, j0);
    const int buf = ld % 3;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    // the tensor map lives in global memory and is rewritten between launches
    // (possibly at the same address): acquire it for the tensor-map proxy once
    // per map, so a stale descriptor-cache copy is not used
    if (m != acq_m) {
      asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(&M.tmap)
                   : "memory");
      acq_m = m;
    }
    mbar_expect_tx(&bar[buf], BOX_BYTES);
    tma_load_3d(smem + G::O_BUF + buf * G::BUF, &M.tmap, &bar[buf], j0, i0, k);
    ++ld;
    pending = true;
  };
  uint64_t *skipmask = reinterpret_cast<uint64_t *>(slot);  // per item: slice j skippable
  if (tid == 0) {
#pragma unroll
    for (int b = 0; b < G::NBUF; ++b) mbar_init(&bar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (blockIdx.x < n_items) {
      int m, r, t;
      decode(blockIdx.x, m, r, t);
      issue(m, t, r * maps[m].run);
    }
  }
  if (tid < 2) {  // the first item's mask words (parity 0)
    unsigned *w = reinterpret_cast<unsigned *>(skipmask);
    bool c0 = false;
    if (blockIdx.x < n_items) {
      int m, r, t;
      decode(blockIdx.x, m, r, t);
      c0 = maps[m].chg != nullptr;
    }
    w[tid] = c0 ? 0u : 0xFFFFFFFFu;
  }
  __syncthreads();
  int ip = 0;  // parity of the item's mask words
  // change-map bytes of the next item, prefetched into registers
  constexpr int kChgPf = 8;
  unsigned char cpf[kChgPf];
  int cpf_item = -1, cpf_j0 = 0, cpf_js = 1;
  uint32_t phase_bits = 0u;
  int lc = 0;  // loads consumed
  // Items: the CTA's first is blockIdx.x; with a work counter the next one
  // is claimed dynamically at each item's start (thread 0, published through
  // shared memory at the item's mask barrier), else item + gridDim.x.  Any
  // assignment gives the same outputs (items are independent).
  int *nxt_s = slot + 5;
  int nxt = 0;  // the item after this one (every thread, after the mask barrier)
  for (int item = blockIdx.x; item < n_items; item = nxt) {
    if (tid == 0) *nxt_s = work ? atomicAdd(work, 1) + (int)gridDim.x : item + (int)gridDim.x;
    int m, r, t;
    decode(item, m, r, t);
    const EvalMap &M = maps[m];
    int i0, j0;
    origin(M, t, i0, j0);
    const int k0 = r * M.run, k1 = min(M.S, k0 + M.run);  // run <= 64
    const int rows = M.rows, cols = M.cols;
    const int64_t cells = (int64_t)rows * cols, words = M.words;
    const uint32_t *bits_in = M.bits;
    float *cost = M.cost;
    const bool sparse = SP && M.fresh != nullptr;  // uniform (compile-time false without SP)
    const bool tstore = M.ostore != 0;       // uniform
    // the output tile of slice k to global memory: one TMA bulk tensor store
    // issued by thread 0 (the copy engine reads `ot`), else the threads' stores
    auto put_tile = [&](int k, int i0, int j0) {
      if (tstore) {
        if (tid == 0) tma_store_3d(&M.omap, ot, j0, i0, k);
      } else {
        store_tile(cost + (int64_t)k * cells, rows, cols, i0, j0, tid);
      }
    };
    // skippable slices of this item: no change of encoded c_init or gentle
    // flag in the tile + R + r window since the slice below (walk change map).
    // Each thread ORs the bytes it checks into a register mask (its loads
    // batched, no atomic per byte), one shared atomic per warp; the shared
    // words alternate between items (parity ip), the pair of the next item
    // is cleared here, before this item's slice barriers, so one barrier per
    // item suffices.
    unsigned *chgw = reinterpret_cast<unsigned *>(skipmask) + 2 * ip;  // [2]: slices 0-31, 32-63
    if (M.chg) {
      uint64_t loc = 0ull;
      if (cpf_item == item) {  // this thread's bytes were loaded during the previous item
#pragma unroll
        for (int u = 0; u < kChgPf; ++u) {
          const int j = cpf_j0 + u * cpf_js;
          if (j < 64) loc |= (uint64_t)(cpf[u] != 0) << j;  // 0 beyond the item's slices
        }
      } else {
        const int nbr = (rows + 7) >> 3, wpr = M.wpr;
        const int br0 = max(0, (i0 - R - PR) >> 3), br1 = min(nbr - 1, (i0 + TH + R + PR - 1) >> 3);
        const int wc0 = max(0, (j0 - R - PR) >> 5), wc1 = min(wpr - 1, (j0 + TW + R + PR - 1) >> 5);
        const int nb = br1 - br0 + 1, nw = wc1 - wc0 + 1;
        const int per = nb * nw;
        const int64_t cms = (int64_t)nbr * wpr;
        for (int q = tid; q < (k1 - k0 - 1) * per; q += NT) {
          const int j = 1 + q / per, e = q - (j - 1) * per;
          const int br = br0 + e / nw, wc = wc0 + e - (e / nw) * nw;
          loc |= (uint64_t)(M.chg[(int64_t)(k0 + j) * cms + (int64_t)br * wpr + wc] != 0) << j;
        }
      }
      const unsigned lo = __reduce_or_sync(0xFFFFFFFFu, (unsigned)loc);
      const unsigned hi = __reduce_or_sync(0xFFFFFFFFu, (unsigned)(loc >> 32));
      if (lane == 0) {
        if (lo) atomicOr(&chgw[0], lo);
        if (hi) atomicOr(&chgw[1], hi);
      }
    }
    __syncthreads();
    const uint64_t changed = (uint64_t)chgw[0] | ((uint64_t)chgw[1] << 32);
    const uint64_t skm = ~changed;  // bit j: slice k0 + j is skippable (bit 0 unused: first)
    nxt = *nxt_s;
    // the next item's change-map bytes: loads issued now, consumed at its start
    // (thread: one (block, word) entry of the window, every jstep-th slice;
    // only when the entries fit kChgPf registers, else that item loads them
    // itself)
    cpf_item = -1;
    if (nxt < n_items) {
      const int it2 = nxt;
      int m2, r2, t2;
      decode(it2, m2, r2, t2);
      const EvalMap &M2 = maps[m2];
      if (M2.chg) {
        int a0, b0;
        origin(M2, t2, a0, b0);
        const int q0 = r2 * M2.run, q1 = min(M2.S, q0 + M2.run);
        const int nbr = (M2.rows + 7) >> 3, wpr = M2.wpr;
        const int br0 = max(0, (a0 - R - PR) >> 3), br1 = min(nbr - 1, (a0 + TH + R + PR - 1) >> 3);
        const int wc0 = max(0, (b0 - R - PR) >> 5), wc1 = min(wpr - 1, (b0 + TW + R + PR - 1) >> 5);
        const int nb = br1 - br0 + 1, nw = wc1 - wc0 + 1;
        const int per = nb * nw;
        const int js = per <= NT ? NT / per : 1;
        if (per <= NT && (q1 - q0 - 1 + js - 1) / js <= kChgPf) {  // uniform
          const int64_t cms = (int64_t)nbr * wpr;
          const bool mine = tid < js * per;
          const int e = tid % per;
          const int br = br0 + e / nw, wc = wc0 + e - (e / nw) * nw;
          const unsigned char *pc = M2.chg + (int64_t)q0 * cms + (int64_t)br * wpr + wc;
          cpf_j0 = 1 + tid / per;
          cpf_js = js;
#pragma unroll
          for (int u = 0; u < kChgPf; ++u) {
            const int j = cpf_j0 + u * js;
            cpf[u] = (mine && j < q1 - q0) ? pc[(int64_t)j * cms] : (unsigned char)0;
          }
          cpf_item = it2;
        }
      }
    }
    if (tid < 2) {  // the next item's pair (its last readers finished an item ago)
      unsigned *nx = reinterpret_cast<unsigned *>(skipmask) + 2 * (ip ^ 1);
      const int item2 = nxt;
      bool nchg = false;
      if (item2 < n_items) {
        int m2, r2, t2;
        decode(item2, m2, r2, t2);
        nchg = maps[m2].chg != nullptr;
      }
      nx[tid] = nchg ? 0u : 0xFFFFFFFFu;  // no change map: nothing skips
    }
    ip ^= 1;
    unsigned long long touched = 0ull;  // slices whose outputs may have changed (thread 0)
    // sparse P0a prefetch registers: fresh byte + bitmap word of this
    // thread's window entries for slice pf_k
    constexpr int kPfEnt = (G::GH * G::NSW + NT - 1) / NT;
    uint32_t pf_w[kPfEnt];
    unsigned char pf_f[kPfEnt];
    int pf_k = -1;
    auto pf_load = [&](int e, int kk, int gi, int ws) {
      pf_f[e] = M.fresh[((int64_t)kk * rows + gi) * M.fpitch + ws];
      pf_w[e] = __ldg(M.bits + (int64_t)kk * words + (int64_t)gi * M.wpr + ws);
    };
    for (int k = k0; k < k1; ++k) {
      const bool first = k == k0;
      const bool skip = !first && ((skm >> (k - k0)) & 1ull);
      if (tid == 0) {
        if (!skip) pending = false;  // this step consumes the load in flight
        if (!pending) {              // the next step that loads: this item, or the next one
          int kn = k + 1;
          while (kn < k1 && ((skm >> (kn - k0)) & 1ull)) ++kn;
          if (kn < k1) {
            issue(m, t, kn);
          } else if (nxt < n_items) {
            int m2, r2, t2;
            decode(nxt, m2, r2, t2);
            issue(m2, t2, r2 * maps[m2].run);
          }
        }
      }
      if (skip) {  // outputs equal the previous slice's: store the kept tile
        put_tile(k, i0, j0);
        continue;
      }
      const int cur = lc % 3, prv = (lc + 2) % 3;
      ++lc;
      float *ci = reinterpret_cast<float *>(smem + G::O_BUF + cur * G::BUF);
      const float *cp = reinterpret_cast<const float *>(smem + G::O_BUF + prv * G::BUF);
    // the output tile is rewritten below: bulk stores still reading it first
    if (tstore && tid == 0) tma_store_wait_read();
    // ---- P0a: gentle bits of the window region (bit x of word w = gentle
    // column 32w + x, gentle column 0 = c_init column -r); resets
    const uint32_t *bk = bits_in + (int64_t)k * words;
    const int wpr = M.wpr;
    const int gj0 = j0 - R - PR, ws0 = gj0 >> 5;  // first source word (floor)
    if (sparse) {
      // raw source words, the fresh ones of this slice from memory, the
      // others kept from the last loaded slice (first slice of an item: all).
      // This thread's entries (fresh byte + word) for this slice were
      // usually loaded into registers during the previous loaded slice of
      // the item (pf_k == k); the next loaded slice's are issued below.
#pragma unroll
      for (int e = 0; e < kPfEnt; ++e) {
        const int idx = tid + e * NT;
        if (idx >= G::GH * G::NSW) break;
        const int y = idx / G::NSW, sw = idx - y * G::NSW;
        const int gi = i0 - R - PR + y, ws = ws0 + sw;
        const bool inmap = gi >= 0 && gi < rows && ws >= 0 && ws < wpr;
        if (pf_k != k && inmap && !first) pf_load(e, k, gi, ws);
        const bool fr = !inmap || first || pf_f[e] != 0;
        frb[idx] = fr;
        if (fr) raww[idx] = inmap ? (first ? __ldg(bk + (int64_t)gi * wpr + ws) : pf_w[e]) : 0u;
      }
      // prefetch: the next loaded slice of this item (registers held across
      // the rest of this step and any skipped steps)
      {
        pf_k = -1;
        uint64_t rest = (k + 1 < k1) ? (~skm >> (k + 1 - k0)) : 0ull;
        if (k + 1 - k0 < 64 && rest) {
          const int kn = k + 1 + __ffsll((long long)rest) - 1;
          if (kn < k1) {
            pf_k = kn;
#pragma unroll
            for (int e = 0; e < kPfEnt; ++e) {
              const int idx = tid + e * NT;
              if (idx >= G::GH * G::NSW) break;
              const int y = idx / G::NSW, sw = idx - y * G::NSW;
              const int gi = i0 - R - PR + y, ws = ws0 + sw;
              if (gi >= 0 && gi < rows && ws >= 0 && ws < wpr) pf_load(e, kn, gi, ws);
            }
          }
        }
      }
      __syncthreads();
      const int sh = gj0 & 31;
      for (int idx = tid; idx < G::GH * G::GWW; idx += NT) {
        const int y = idx / G::GWW, w = idx - y * G::GWW;
        const uint32_t lo = raww[y * G::NSW + w], hi = raww[y * G::NSW + w + 1];
        uint32_t word = sh ? __funnelshift_r(lo, hi, sh) : lo;
        if (32 * w >= G::GW) word = 0;
        else if (G::GW - 32 * w < 32) word &= (1u << (G::GW - 32 * w)) - 1u;
        bits[idx] = word;
      }
    } else {
      for (int idx = tid; idx < G::GH * G::GWW; idx += NT) {
        const int y = idx / G::GWW, w = idx - y * G::GWW;
        const int gi = i0 - R - PR + y;
        const int gj = j0 - R - PR + 32 * w;
        uint32_t word = gentle_word(bk, wpr, gi, gj, rows, cols);
        if (32 * w >= G::GW) word = 0;
        else if (G::GW - 32 * w < 32) word &= (1u << (G::GW - 32 * w)) - 1u;
        bits[idx] = word;
      }
    }
    for (int idx = tid; idx < G::CBY * G::CBX; idx += NT) chg[idx] = first ? 1 : 0;
    __syncthreads();
    // ---- P0b: foothold test of every c_init cell, 32 cells per word:
    // vertical counts of the (2r+1)-row window (bit-sliced, this word and the
    // next), then the horizontal (2r+1)-column sum, then count >= ps_min
    for (int idx = tid; idx < G::CH * G::CWW; idx += NT) {
      const int y = idx / G::CWW, w = idx - y * G::CWW;
      uint32_t x0[G::SIDE], x1[G::SIDE], v0[G::NVP], v1[G::NVP];
#pragma unroll
      for (int d = 0; d < G::SIDE; ++d) {
        x0[d] = bits[(y + d) * G::GWW + w];
        x1[d] = bits[(y + d) * G::GWW + w + 1];
      }
      column_count<G::SIDE, G::NVP>(x0, v0);
      column_count<G::SIDE, G::NVP>(x1, v1);
      uint32_t sum[G::NSB];
#pragma unroll
      for (int p = 0; p < G::NSB; ++p) sum[p] = 0u;
#pragma unroll
      for (int p = 0; p < G::NVP; ++p) {
        uint32_t sh[G::SIDE], h[G::NVP];
#pragma unroll
        for (int d = 0; d < G::SIDE; ++d) sh[d] = __funnelshift_r(v0[p], v1[p], d);
        column_count<G::SIDE, G::NVP>(sh, h);
        bs_add<G::NSB, G::NVP>(sum, h, p);
      }
      okb[idx] = bs_ge<G::NSB>(sum, c_K.ps_min_count);
    }
    mbar_wait(&bar[cur], (phase_bits >> cur) & 1u);
    phase_bits ^= 1u << cur;
    __syncthreads();
    // ---- P0c: resolve the foothold-branch cells in place; maxima of the
    // aligned R x R blocks (c_init >= 0: float order = uint order); 4 x 4
    // blocks that differ from the previous slice
    constexpr int CW4 = G::CW / 4;
    bool changed = first;
    for (int q = tid; q < G::CH * CW4; q += NT) {
      float4 v = lds4(ci + 4 * q);
      const int y = q / CW4, x = 4 * (q - y * CW4);
      if (sparse) {  // cells the walk did not rewrite: the last loaded slice's value
        // (4 cells never straddle a bitmap word: R % 4 == 0, TW % 32 == 0)
        const int sw = ((j0 - R + x) >> 5) - ws0;
        if (!frb[(y + PR) * G::NSW + sw]) {
          v = lds4(rawc + 4 * q);
          *reinterpret_cast<float4 *>(ci + 4 * q) = v;
        } else {
          *reinterpret_cast<float4 *>(rawc + 4 * q) = v;
        }
      }
      const uint32_t sgn = (f32_bits(v.x) | f32_bits(v.y) | f32_bits(v.z) | f32_bits(v.w));
      if (sgn & 0x80000000u) {  // branch-free cinit_resolve of the 4 cells
        const uint32_t ok = okb[y * G::CWW + (x >> 5)] >> (x & 31);  // 4 cells, one word
        auto res = [&](float f, uint32_t okbit) {
          const uint32_t u = f32_bits(f);
          const uint32_t r = okbit ? (u & 0x7FFFFFFFu) : cb_bits;
          return bits_f32((u & 0x80000000u) ? r : u);
        };
        v.x = res(v.x, ok & 1u);
        v.y = res(v.y, ok & 2u);
        v.z = res(v.z, ok & 4u);
        v.w = res(v.w, ok & 8u);
        *reinterpret_cast<float4 *>(ci + 4 * q) = v;
      }
      if (!first) {
        const float4 u = lds4(cp + 4 * q);
        if (f32_bits(u.x) != f32_bits(v.x) || f32_bits(u.y) != f32_bits(v.y) ||
            f32_bits(u.z) != f32_bits(v.z) || f32_bits(u.w) != f32_bits(v.w)) {
          chg[(y >> 2) * G::CBX + (x >> 2)] = 1;
          changed = true;
        }
      }
    }
    // a tile whose resolved c_init equals the previous slice's keeps every
    // output: straight to the store
    const bool tile_changed = __syncthreads_or(changed);
    if (tile_changed) touched |= 1ull << (k & 63);
    if (tile_changed) {
    // ---- P1: dirty output blocks; horizontal maxima planes; upper bound per
    // output block (3 x 3 c_init blocks cover every tap of its outputs' windows)
    {
      constexpr int NG = TW / 4;
      constexpr int NQ = G::QY * G::QX;
      constexpr int ND = G::DBY * G::DBX;
      constexpr int NB = G::NBY * G::NBX;
      for (int q = tid; q < ND + NB + G::CH * NG; q += NT) {
        if (q < ND) {
          const int dy = q / G::DBX, dx = q - dy * G::DBX;
          bool d = false;
#pragma unroll
          for (int a = 0; a < G::SPAN; ++a)
#pragma unroll
            for (int b = 0; b < G::SPAN; ++b) d |= chg[(dy + a) * G::CBX + dx + b] != 0;
          dirty[q] = d;
        } else if (q < ND + NB) {  // maxima of the aligned R x R c_init blocks
          const int e = q - ND;
          const int by = e / G::NBX, bx = e - by * G::NBX;
          const float *p = ci + by * R * G::CW + bx * R;
          float m = 0.0f;
#pragma unroll
          for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c4 = 0; c4 < R; c4 += 4) {
              const float4 v = lds4(p + r * G::CW + c4);
              m = fmax3(m, fmaxf(v.x, v.y), fmaxf(v.z, v.w));
            }
          bm[e] = f32_bits(m);
        } else {
          const int e = q - ND - NB;
          const int y = e / NG, g = e - y * NG;
          // c_init columns 4g + R - 4 .. 4g + R + 7 (12 values, 16-byte aligned)
          const float *p = ci + y * G::CW + 4 * g + R - 4;
          const float4 a = lds4(p), b = lds4(p + 4), c = lds4(p + 8);
          const float v[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
          // output column 4g + t has its centre at v[4 + t]
          if constexpr (R == 4) {
            float4 h1;
            h1.x = fmax3(v[3], v[4], v[5]);
            h1.y = fmax3(v[4], v[5], v[6]);
            h1.z = fmax3(v[5], v[6], v[7]);
            h1.w = fmax3(v[6], v[7], v[8]);
            *reinterpret_cast<float4 *>(planes + y * TW + 4 * g) = h1;
          } else {
            float h2[4], h3[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              h2[t] = fmax3(fmax3(v[t + 2], v[t + 3], v[t + 4]), v[t + 5], v[t + 6]);
              h3[t] = fmax3(h2[t], v[t + 1], v[t + 7]);
            }
            *reinterpret_cast<float4 *>(planes + y * TW + 4 * g) = make_float4(h3[0], h3[1], h3[2], h3[3]);
            *reinterpret_cast<float4 *>(planes + G::PLANE + y * TW + 4 * g) =
                make_float4(h2[0], h2[1], h2[2], h2[3]);
          }
        }
      }
    }
    __syncthreads();
    // ---- P2: dirty outputs: disk max, bound test; the rest to this warp's list
    int nlist = 0;  // warp-uniform
    {
      constexpr int NG = TW / 4;
      for (int q = tid; q < TH * NG; q += NT) {
        const int i = q / NG, g = q - i * NG;
        const bool dq = dirty[(i >> 2) * G::DBX + g] != 0;
        if (!__any_sync(0xFFFFFFFFu, dq)) continue;
        const int yc = i + R;  // centre row in c_init / plane coordinates
        float d1[4];
        if constexpr (R == 4) {
          const float4 a = lds4(planes + (yc - 1) * TW + 4 * g);
          const float4 b = lds4(planes + yc * TW + 4 * g);
          const float4 c = lds4(planes + (yc + 1) * TW + 4 * g);
          const float *cr = ci + yc * G::CW + 4 * g;  // c_init cols 4g .. 4g+11
          const float4 r0 = lds4(cr), r1 = lds4(cr + 4), r2 = lds4(cr + 8);
          const float rv[12] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w, r2.x, r2.y, r2.z, r2.w};
          const float4 u2 = lds4(ci + (yc - 2) * G::CW + 4 * g + 4);
          const float4 d2 = lds4(ci + (yc + 2) * G::CW + 4 * g + 4);
          d1[0] = fmax3(fmax3(a.x, b.x, c.x), fmax3(rv[2], rv[6], u2.x), d2.x);
          d1[1] = fmax3(fmax3(a.y, b.y, c.y), fmax3(rv[3], rv[7], u2.y), d2.y);
          d1[2] = fmax3(fmax3(a.z, b.z, c.z), fmax3(rv[4], rv[8], u2.z), d2.z);
          d1[3] = fmax3(fmax3(a.w, b.w, c.w), fmax3(rv[5], rv[9], u2.w), d2.w);
        } else {
          const float *h3 = planes + 4 * g, *h2 = planes + G::PLANE + 4 * g;
          const float4 a0 = lds4(h3 + (yc - 2) * TW), a1 = lds4(h3 + (yc - 1) * TW),
                       a2 = lds4(h3 + yc * TW), a3 = lds4(h3 + (yc + 1) * TW),
                       a4 = lds4(h3 + (yc + 2) * TW);
          const float4 b0 = lds4(h2 + (yc - 3) * TW), b1 = lds4(h2 + (yc + 3) * TW);
          const float *cr = ci + yc * G::CW + 4 * g;  // centre of output 4g: col 4g + 8
          const float4 l4 = lds4(cr + 4), r4 = lds4(cr + 12);
          const float4 u4 = lds4(ci + (yc - 4) * G::CW + 4 * g + 8);
          const float4 d4 = lds4(ci + (yc + 4) * G::CW + 4 * g + 8);
          d1[0] = fmax3(fmax3(a0.x, a1.x, a2.x), fmax3(a3.x, a4.x, b0.x),
                        fmax3(fmax3(b1.x, l4.x, r4.x), u4.x, d4.x));
          d1[1] = fmax3(fmax3(a0.y, a1.y, a2.y), fmax3(a3.y, a4.y, b0.y),
                        fmax3(fmax3(b1.y, l4.y, r4.y), u4.y, d4.y));
          d1[2] = fmax3(fmax3(a0.z, a1.z, a2.z), fmax3(a3.z, a4.z, b0.z),
                        fmax3(fmax3(b1.z, l4.z, r4.z), u4.z, d4.z));
          d1[3] = fmax3(fmax3(a0.w, a1.w, a2.w), fmax3(a3.w, a4.w, b0.w),
                        fmax3(fmax3(b1.w, l4.w, r4.w), u4.w, d4.w));
        }
        const uint32_t *pq = bm + (i / R) * G::NBX + (4 * g) / R;  // 3 x 3 blocks under the window
        const float U = bits_f32(max(max(max(pq[0], pq[1]), max(pq[2], pq[G::NBX])),
                                     max(max(pq[G::NBX + 1], pq[G::NBX + 2]),
                                         max(max(pq[2 * G::NBX], pq[2 * G::NBX + 1]),
                                             pq[2 * G::NBX + 2]))));
        const float bound = w1 * U;
        float v[4];
        unsigned m = 0;  // outputs of this thread that need the class walk
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          v[t] = w0 * d1[t];
          if (dq && v[t] < bound) m |= 1u << t;
        }
        if (dq) *reinterpret_cast<float4 *>(ot + i * TW + 4 * g) = make_float4(v[0], v[1], v[2], v[3]);
        if (__any_sync(0xFFFFFFFFu, m != 0u)) {
          const unsigned lt = (1u << lane) - 1u;
          int pos = nlist;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const unsigned b = __ballot_sync(0xFFFFFFFFu, m & (1u << t));
            if (m & (1u << t)) wlist[pos + __popc(b & lt)] = (uint16_t)(i * TW + 4 * g + t);
            pos += __popc(b);
          }
          nlist = pos;
        }
      }
    }
    if (lane == 0) wcnt[warp] = nlist;
    __syncthreads();
    // ---- P3: the listed outputs (all warps' lists, shared out evenly) walk
    // the remaining classes under the bound
    {
      int pre[NWARP + 1];
      pre[0] = 0;
#pragma unroll
      for (int w = 0; w < NWARP; ++w) pre[w + 1] = pre[w] + wcnt[w];
      const int ns = pre[NWARP];
      for (int base = tid - lane; base < ns; base += NT) {
        const int s = base + lane;
        const bool in_list = s < ns;
        int at = s;  // position in the segmented list: skip the unused tails
#pragma unroll
        for (int w = 1; w < NWARP; ++w)
          if (s >= pre[w]) at += WSEG - (pre[w] - pre[w - 1]);
        const int idx = in_list ? slist[at] : 0;
        const int i = idx / TW, x = idx - i * TW;
        const int yc = i + R;
        float d1;  // the disk max again, from the planes (as P2)
        if constexpr (R == 4) {
          const float *cc = ci + yc * G::CW + x + R;
          d1 = fmax3(fmax3(planes[(yc - 1) * TW + x], planes[yc * TW + x], planes[(yc + 1) * TW + x]),
                     fmax3(cc[-2], cc[2], cc[-2 * G::CW]), cc[2 * G::CW]);
        } else {
          const float *h3 = planes + x, *h2 = planes + G::PLANE + x;
          const float *cc = ci + yc * G::CW + x + R;
          d1 = fmax3(fmax3(h3[(yc - 2) * TW], h3[(yc - 1) * TW], h3[yc * TW]),
                     fmax3(h3[(yc + 1) * TW], h3[(yc + 2) * TW], h2[(yc - 3) * TW]),
                     fmax3(fmax3(h2[(yc + 3) * TW], cc[-4], cc[4]), cc[-4 * G::CW], cc[4 * G::CW]));
        }
        float acc = w0 * d1;
        const uint32_t *pq = bm + (i / R) * G::NBX + x / R;
        const float U = bits_f32(max(max(max(pq[0], pq[1]), max(pq[2], pq[G::NBX])),
                                     max(max(pq[G::NBX + 1], pq[G::NBX + 2]),
                                         max(max(pq[2 * G::NBX], pq[2 * G::NBX + 1]),
                                             pq[2 * G::NBX + 2]))));
        slow_classes<R, G::CW, 1>(ci + yc * G::CW + (x + R), U, in_list, acc);
        if (in_list) ot[idx] = acc;
      }
    }
    if (tstore) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // ot -> TMA store
    __syncthreads();
    }  // tile changed
    // ---- P4: store the output tile (every output, every slice)
    put_tile(k, i0, j0);
    // the next step's first barrier orders P4's reads of `ot` before its P2
    }
    // per tile: the slices whose outputs may differ from the slice below
    // (the first slice of a run counts as changed), for the simplify window
    if (M.tcm && tid == 0 && touched) atomicOr(M.tcm + t, touched | (1ull << (k0 & 63)));
  }
  if (tid == 0) tma_store_wait_all();  // bulk stores done before the CTA leaves
}

// Host: the caller's kernel must have exactly the compiled class structure
// (class 0 = DiskShape<R>, classes 1.. = BnbRings<R>, strictly decreasing
// weights); on success cw = the class weights + a trailing 0.
template <int R>
bool bnb_tables(const float *w, int kside, std::vector<float> &cw) {
  using RG = BnbRings<R>;
  using D = DiskShape<R>;
  if (kside != 2 * R + 1) return false;
  std::vector<float> vals;
  for (int t = 0; t < kside * kside; ++t)
    if (w[t] > 0.0f) vals.push_back(w[t]);
  std::sort(vals.begin(), vals.end(), [](float a, float b) { return a > b; });
  vals.erase(std::unique(vals.begin(), vals.end()), vals.end());
  if ((int)vals.size() != RG::NCLS || RG::NCLS > kBnbMaxClasses) return false;
  std::vector<int> cls(kside * kside, -1);  // compiled class of every tap
  for (int m = 0; m < kside; ++m)
    for (int n = 0; n < kside; ++n) {
      const int a = std::abs(m - R), b = std::abs(n - R);
      if (a <= D::A && D::h[a] >= b) cls[m * kside + n] = 0;
    }
  for (int c = 1; c < RG::NCLS; ++c)
    for (int t = RG::start(c); t < RG::start(c + 1); ++t)
      cls[(RG::dy(t) + R) * kside + (RG::dx(t) + R)] = c;
  for (int t = 0; t < kside * kside; ++t) {
    const int want = w[t] > 0.0f ? (int)(std::find(vals.begin(), vals.end(), w[t]) - vals.begin()) : -1;
    if (cls[t] != want) return false;
  }
  cw.assign(vals.begin(), vals.end());
  cw.push_back(0.0f);
  return true;
}
