// k_simplify.cu — K6: redundant-slice simplification (simplify.py:18-73).
//
// The reference sweeps forward over the slice list, removing a slice when no
// cell is "unique" w.r.t. its current lower and upper neighbours, and repeats
// until a pass removes nothing.  The per-check work is an any() over all
// cells of (trav & side(below) & side(above)); the sweep order is inherently
// sequential, so the device computes the any()s in bulk and the host replays
// the exact sweep:
//
//  * window_kernel: one pass over every cell computes, for each slice k and
//    each lower neighbour a in {none, k-1, ..., k-16}, whether any cell is
//    unique for the triple (a, k, k+1) — every check of the first pass whose
//    removal chain is <= 16 long (the upper neighbour of pass 1 is always the
//    original k+1).  Each thread owns a cell and keeps its last 16 slices'
//    (ground, cost) in a shared-memory ring; per k the block ORs a 64-bit mask.
//  * triples_kernel: any() for an explicit batch of (below, k, above)
//    triples — later passes and long chains; the host batches the remainder
//    of the pass speculatively (no further removals), blocks exit early once
//    a triple is known unique.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <vector>

#include "pct_internal.h"

namespace pct {
namespace {

constexpr int kWin = 16;      // lower-neighbour window of window_kernel (power of 2)
constexpr int kBit = 32;      // bit index for "no lower neighbour"
constexpr int kWinNT = 128;

struct SimpArgs {
  const float *ground;
  const float *cost;
  int64_t cells;
  int64_t stride;  // floats between consecutive slices (== cells for a dense stack)
  int S;
  double eps_e;
  float c_barrier32;  // numpy compares float32 costs with the weak Python scalar in float32
};

// side condition of simplify.py:18-28 for a valid, traversable cell
__device__ __forceinline__ bool not_covered(float e, float cst, float enb, float cnb, double eps,
                                            bool lower) {
  if (!finite32(enb)) return true;
  const double a = (double)e, b = (double)enb;
  const bool higher = lower ? (a - b > eps) : (b - a > eps);
  return higher || (cst < cnb);
}

// side tests with a bit-equality shortcut: equal elevations differ by 0,
// which is not > eps_e unless eps_e < 0, so the float64 subtraction is only
// evaluated for elevations that differ
__device__ __forceinline__ bool higher_than(float hi, float lo, double eps) {
  return (f32_bits(hi) != f32_bits(lo) || eps < 0.0) && ((double)hi - (double)lo > eps);
}

// Persistent blocks walk cells grid-stride; a thread owns one cell at a time
// and walks its slices; warps OR their masks into a per-block table in
// shared memory (no block barrier per slice), flushed once at the end.
// Warps with no traversable, upper-uncovered cell at slice k skip the
// lower-neighbour tests and the reductions.
__device__ __forceinline__ void window_phase(const SimpArgs &A,
                                             unsigned long long *__restrict__ table) {
  __shared__ float ring_e[kWin][kWinNT];
  __shared__ float ring_c[kWin][kWinNT];
  extern __shared__ unsigned long long btab[];  // [S]
  for (int k = threadIdx.x; k < A.S; k += kWinNT) btab[k] = 0ull;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * kWinNT;
  const int64_t span = (A.cells + kWinNT - 1) / kWinNT * kWinNT;  // whole warps iterate together
  const float nanf_ = bits_f32(kNaNBits);
  constexpr int KB = 4;  // slices per register block; the next block is loaded ahead
  for (int64_t cell = (int64_t)blockIdx.x * kWinNT + threadIdx.x; cell < span; cell += stride) {
    const bool live = cell < A.cells;
    float ce[KB + 1], cc[KB + 1];  // slices k0 .. k0+KB of this cell
    // last slice whose ground dropped below the slice under it (or became
    // invalid after being valid); the older-bits shortcut needs none within
    // the window
    int last_dec = -(1 << 20);
    float e_prev = nanf_;
    // running pointers to the next slice to load (no 64-bit multiply per load)
    const float *pg = A.ground + (live ? cell : 0), *pc = A.cost + (live ? cell : 0);
    int kn = 0;  // slice pg / pc point at
    auto load = [&](float &e, float &c) {
      const bool ok = live && kn < A.S;
      e = ok ? __ldg(pg) : nanf_;
      c = ok ? __ldg(pc) : 0.f;
      pg += A.stride;
      pc += A.stride;
      ++kn;
    };
#pragma unroll
    for (int u = 0; u <= KB; ++u) load(ce[u], cc[u]);
    for (int k0 = 0; k0 < A.S; k0 += KB) {
      float ne[KB], nc[KB];  // slices k0+KB+1 .. k0+2KB, in flight while testing
#pragma unroll
      for (int u = 0; u < KB; ++u) load(ne[u], nc[u]);

#pragma unroll
      for (int u = 0; u < KB; ++u) {
        const int k = k0 + u;
        if (k >= A.S) break;  // uniform
        const float e_cur = ce[u], c_cur = cc[u], e_up = ce[u + 1], c_up = cc[u + 1];
        if (finite32(e_prev) && !(e_cur >= e_prev)) last_dec = k;  // NaN fails >= too
        e_prev = e_cur;
        const bool mono = k - last_dec > kWin;
        const bool up_ok = k + 1 >= A.S || !finite32(e_up) || higher_than(e_up, e_cur, A.eps_e) ||
                           c_cur < c_up;
        const bool cand = live && finite32(e_cur) && c_cur < A.c_barrier32 && up_ok;
        if (__any_sync(0xffffffffu, cand)) {
          unsigned long long m = 0;
          const int depth = k < kWin ? k : kWin;
          const unsigned long long want =
              (1ull << kBit) | ((depth >= 64 ? ~0ull : (1ull << depth) - 1ull));
          // bits this block has already established need no work (a stale
          // read only costs a redundant test)
          const unsigned long long known = *((volatile unsigned long long *)&btab[k]);
          if (cand && (known & want) != want) {
            m = 1ull << kBit;
            unsigned todo = (unsigned)(~known & want);
            // when this cell's ground did not decrease within the window
            // (always, for stacks built here: a prefix max over bins), once a
            // lower neighbour a is invalid or lower by more than eps_e, every
            // older one is too (double subtraction is monotone) -- the
            // remaining, older bits are set at once
            while (todo) {
              const int j = __ffs(todo) - 1;  // a = k-1-j, most recent first
              todo &= todo - 1;
              const int slot = (k - 1 - j) & (kWin - 1);
              const float ea = ring_e[slot][threadIdx.x];
              if (!finite32(ea) || higher_than(e_cur, ea, A.eps_e)) {
                m |= 1ull << j;
                if (mono) {
                  m |= (unsigned long long)todo;
                  break;
                }
              } else if (c_cur < ring_c[slot][threadIdx.x]) {
                m |= 1ull << j;
              }
            }
          }
          const unsigned lo = __reduce_or_sync(0xffffffffu, (unsigned)m);
          const unsigned hi = __reduce_or_sync(0xffffffffu, (unsigned)(m >> 32));
          if ((threadIdx.x & 31) == 0 && (lo | hi))
            atomicOr(&btab[k], ((unsigned long long)hi << 32) | lo);
        }
        ring_e[k & (kWin - 1)][threadIdx.x] = e_cur;  // own column only
        ring_c[k & (kWin - 1)][threadIdx.x] = c_cur;
      }
      ce[0] = ce[KB];
      cc[0] = cc[KB];
#pragma unroll
      for (int u = 0; u < KB; ++u) {
        ce[u + 1] = ne[u];
        cc[u + 1] = nc[u];
      }
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < A.S; k += kWinNT)
    if (btab[k]) atomicOr(table + k, btab[k]);
}

__global__ void __launch_bounds__(kWinNT) window_kernel(SimpArgs A,
                                                        unsigned long long *__restrict__ table) {
  window_phase(A, table);
}

// The same table from slice-change information, reading only where values
// change.  A cell's (ground, cost) pair is constant between the slices where
// its build mask (ground changed) or its evaluation tile's mask (some output
// of the tile may have changed) has a bit: segments.  A cell can only be a
// candidate (traversable and not covered from above) at the last slice of a
// segment -- inside a segment the slice above holds equal values, which
// cover it for eps_e >= 0 -- and a lower neighbour in its own segment covers
// it too; the lower neighbours in older segments share one test per segment.
// Warps load (coalesced) only at the union of their lanes' segment starts;
// each lane keeps its last 16 segments in shared memory.
struct SimpMasks {
  const unsigned long long *gm;   // per cell: ground slice-change mask (bit 0 set)
  const unsigned long long *tcm;  // per evaluation tile: outputs may have changed
  int cols, th, tw, tx;           // cell -> tile of tcm
};

__global__ void __launch_bounds__(kWinNT) window_skip_kernel(SimpArgs A, SimpMasks M,
                                                             unsigned long long *__restrict__ table,
                                                             unsigned long long *__restrict__ work) {
  __shared__ float seg_e[kWin][kWinNT];
  __shared__ float seg_c[kWin][kWinNT];
  __shared__ unsigned char seg_s[kWin][kWinNT];
  extern __shared__ unsigned long long btab[];  // [S]
  for (int k = threadIdx.x; k < A.S; k += kWinNT) btab[k] = 0ull;
  __syncthreads();
  const int tid = threadIdx.x;
  // Warps take groups of 32 cells (whole warps iterate together), kClaim
  // groups per claim: claimed from a global counter when `work` is given
  // (dynamic: warps in event-dense regions take fewer), else round robin.
  constexpr int kClaim = 4;
  const int lane = tid & 31;
  const int64_t groups = (A.cells + 31) / 32;
  const int64_t wid = (int64_t)blockIdx.x * (kWinNT / 32) + (tid >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * (kWinNT / 32);
  int64_t g = 0, gend = 0, nclaim = 0;
  for (;;) {
    if (g == gend) {
      long long c;
      if (work) {
        unsigned long long v = 0ull;
        if (lane == 0) v = atomicAdd(work, 1ull);
        c = (long long)__shfl_sync(0xFFFFFFFFu, v, 0);
      } else {
        c = wid + nclaim * nwarps;
        ++nclaim;
      }
      g = c * kClaim;
      if (g >= groups) break;
      gend = g + kClaim < groups ? g + kClaim : groups;
    }
    const int64_t cell = g * 32 + lane;
    ++g;
    const bool live = cell < A.cells;
    const int64_t c0 = live ? cell : 0;
    unsigned long long vm = 1ull;
    if (live) {
      // 32-bit divisions when the map has < 2^32 cells (a 64-bit division
      // by a run-time value is a ~100-instruction subroutine per warp)
      int i, j;
      if (A.cells <= 0xFFFFFFFFll) {
        const uint32_t c = (uint32_t)c0, q = c / (uint32_t)M.cols;
        i = (int)q;
        j = (int)(c - q * (uint32_t)M.cols);
      } else {
        i = (int)(c0 / M.cols);
        j = (int)(c0 - (int64_t)i * M.cols);
      }
      const uint32_t ti = (uint32_t)i / (uint32_t)M.th, tj = (uint32_t)j / (uint32_t)M.tw;
      vm |= __ldg(M.gm + c0) | __ldg(M.tcm + (int64_t)ti * M.tx + tj);
    }
    const unsigned lo = __reduce_or_sync(0xFFFFFFFFu, (unsigned)vm);
    const unsigned hi = __reduce_or_sync(0xFFFFFFFFu, (unsigned)(vm >> 32));
    unsigned long long ev = (((unsigned long long)hi << 32) | lo) & ~1ull;
    if (A.S < 64) ev &= (1ull << A.S) - 1ull;
    const float *pg = A.ground + c0, *pc = A.cost + c0;
    float cur_e = live ? __ldg(pg) : bits_f32(kNaNBits), cur_c = live ? __ldg(pc) : 0.f;
    int cur_s = 0, nseg = 0;
    // candidate test at slice k for the current segment (values e, c, start
    // s) with the slice above (eu, cu) or none
    auto candidate = [&](int k, bool has_up, float eu, float cu) {
      const float e = cur_e, c = cur_c;
      const bool up_ok = !has_up || !finite32(eu) || higher_than(eu, e, A.eps_e) || c < cu;
      if (!(live && finite32(e) && c < A.c_barrier32 && up_ok)) return;
      const int depth = k < kWin ? k : kWin;
      const unsigned long long want = (1ull << kBit) | ((1ull << depth) - 1ull);
      const unsigned long long known = *((volatile unsigned long long *)&btab[k]);
      if ((known & want) == want) return;
      unsigned long long m = 1ull << kBit;
      int end = cur_s;  // older segments, newest first: [st, end)
      for (int q = 1; q <= kWin && q <= nseg && end > k - depth; ++q) {
        const int slot = (nseg - q) & (kWin - 1);
        const int st = seg_s[slot][tid];
        const float se = seg_e[slot][tid], sc = seg_c[slot][tid];
        if (!finite32(se) || higher_than(e, se, A.eps_e) || c < sc) {
          // lower neighbours a in [max(st, k - depth), end): bits j = k-1-a
          const int a0 = st > k - depth ? st : k - depth;
          const int jlo = k - end, jhi = k - 1 - a0;  // inclusive
          m |= (((2ull << jhi) - 1ull) >> jlo) << jlo;
        }
        end = st;
      }
      if ((m & want & ~known) != 0ull) atomicOr(&btab[k], m & want);
    };
    // event slices in order; the next event's two loads are issued before
    // this one is processed (one event of latency hidden per lane)
    auto fetch = [&](int k, float &e, float &c) {
      e = live ? __ldg(pg + (int64_t)k * A.stride) : bits_f32(kNaNBits);
      c = live ? __ldg(pc + (int64_t)k * A.stride) : 0.f;
    };
    int kn = -1;
    float en = 0.f, cn = 0.f;
    if (ev) {
      kn = __ffsll((long long)ev) - 1;
      ev &= ev - 1ull;
      fetch(kn, en, cn);
    }
    while (kn >= 0) {
      const int k = kn;
      const float e = en, c = cn;
      kn = -1;
      if (ev) {
        kn = __ffsll((long long)ev) - 1;
        ev &= ev - 1ull;
        fetch(kn, en, cn);
      }
      if ((vm >> k) & 1ull) {  // this lane's segment ends at k - 1
        candidate(k - 1, true, e, c);
        const int slot = nseg & (kWin - 1);
        seg_s[slot][tid] = (unsigned char)cur_s;
        seg_e[slot][tid] = cur_e;
        seg_c[slot][tid] = cur_c;
        ++nseg;
        cur_s = k;
        cur_e = e;
        cur_c = c;
      }
    }
    candidate(A.S - 1, false, 0.f, 0.f);
  }
  __syncthreads();
  for (int k = tid; k < A.S; k += kWinNT)
    if (btab[k]) atomicOr(table + k, btab[k]);
}

struct Triple {
  int below, k, above;
};

// resident window blocks per SM (one wave; the kernel is persistent)
int window_blocks_per_sm(pct_ctx *ctx, size_t smem) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, window_kernel, kWinNT, smem) !=
          cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    per_sm = 8;
  }
  return per_sm;
}

// Is any cell of [lo, hi) a traversable cell of slice T.k not covered by
// T.below / T.above?  Block-strided, 4 cells per thread per step: the 8
// loads of the 4 cells are issued together, then the neighbour slices' loads
// of the candidates among them (early exit once any thread of the block has
// found one, or another block already has).
__device__ __forceinline__ void triple_any(const SimpArgs &A, const Triple T, int *flag,
                                           int64_t lo, int64_t hi, int64_t start, int64_t step) {
  __shared__ int skip;
  __syncthreads();  // previous triple's readers of `skip` are done
  if (threadIdx.x == 0) skip = *((volatile int *)flag);  // already known unique
  __syncthreads();
  if (skip) return;
  constexpr int U = 4;
  const float *gk = A.ground + (int64_t)T.k * A.stride, *ck = A.cost + (int64_t)T.k * A.stride;
  const float *gb = A.ground + (int64_t)T.below * A.stride, *cb = A.cost + (int64_t)T.below * A.stride;
  const float *ga = A.ground + (int64_t)T.above * A.stride, *ca = A.cost + (int64_t)T.above * A.stride;
  bool any = false;
  for (int64_t c0 = lo + start; c0 < hi && !any; c0 += U * step) {
    float e[U], c[U];
    bool cand[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t cell = c0 + u * step;
      const bool in = cell < hi;
      e[u] = in ? __ldg(gk + cell) : bits_f32(kNaNBits);
      c[u] = in ? __ldg(ck + cell) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) cand[u] = finite32(e[u]) && c[u] < A.c_barrier32;
    float eb[U], cbv[U], ea[U], cav[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t cell = c0 + u * step;
      const bool lb = cand[u] && T.below >= 0, la = cand[u] && T.above >= 0;
      eb[u] = lb ? __ldg(gb + cell) : 0.f;
      cbv[u] = lb ? __ldg(cb + cell) : 0.f;
      ea[u] = la ? __ldg(ga + cell) : 0.f;
      cav[u] = la ? __ldg(ca + cell) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!cand[u]) continue;
      bool un = true;
      if (T.below >= 0) un = not_covered(e[u], c[u], eb[u], cbv[u], A.eps_e, true);
      if (un && T.above >= 0) un = not_covered(e[u], c[u], ea[u], cav[u], A.eps_e, false);
      any = any || un;
    }
  }
  if (__syncthreads_or(any) && threadIdx.x == 0) atomicOr(flag, 1);
}

// blockIdx.y = triple (host lists), blocks stride over all cells; with a
// device count, the blocks split (triple, cell range) items instead: each
// of the n triples gets about G / n ranges, so a single triple still has the
// whole grid (G blocks)
__global__ void __launch_bounds__(256) triples_kernel(SimpArgs A, const Triple *__restrict__ tr,
                                                      int *__restrict__ flags,
                                                      const int *__restrict__ count = nullptr) {
  if (!count) {
    triple_any(A, tr[blockIdx.y], flags + blockIdx.y, 0, A.cells,
               (int64_t)blockIdx.x * blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x);
    return;
  }
  const int n = *count;
  if (n <= 0) return;
  const int G = (int)(gridDim.x * gridDim.y), b = (int)(blockIdx.y * gridDim.x + blockIdx.x);
  const int X = G / n > 1 ? G / n : 1;
  for (int w = b; w < n * X; w += G) {
    const int t = w / X, x = w - t * X;
    const int64_t lo = A.cells * x / X, hi = A.cells * (x + 1) / X;
    triple_any(A, tr[t], flags + t, lo, hi, threadIdx.x, blockDim.x);
  }
}

// The host sweep's first pass, replayed on the device from the window table
// (one thread; the keep list as a linked list), followed by the triples the
// second pass would ask assuming it removes nothing -- the speculation the
// host makes itself on a table miss.  Lets the triples kernel run without a
// host round trip in between; the host replays the whole sweep afterwards
// and only falls back to its own rounds on a miss.  count = 0: nothing to
// speculate (the first pass removed nothing, or needed a triple itself).
__device__ __forceinline__ int window_lookup(const unsigned long long *table, int S, int below,
                                             int k, int above) {  // 1 / 0, or -1 = not in table
  const bool above_ok = (above == k + 1) || (above < 0 && k == S - 1);
  if (!above_ok) return -1;
  int bit = -1;
  if (below < 0) bit = kBit;
  else if (k - 1 - below < kWin) bit = k - 1 - below;
  if (bit < 0) return -1;
  return (int)((table[k] >> bit) & 1ull);
}

constexpr int kSpecSweepMaxS = 1024;  // table + links staged in shared memory (16 KB)

__global__ void __launch_bounds__(32) spec_sweep_kernel(
    const unsigned long long *__restrict__ table, int S, Triple *__restrict__ tr,
    int *__restrict__ flags, int *__restrict__ count) {
  __shared__ unsigned long long tb[kSpecSweepMaxS];
  __shared__ int prv[kSpecSweepMaxS], nxt[kSpecSweepMaxS];
  if (S > kSpecSweepMaxS) {
    if (threadIdx.x == 0) *count = 0;
    return;
  }
  for (int k = threadIdx.x; k < S; k += 32) {  // one global read per entry
    tb[k] = table[k];
    prv[k] = k - 1;
    nxt[k] = k + 1 < S ? k + 1 : -1;
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  int head = 0, size = S, T = 0;
  bool removed = false;
  for (int k = head; k >= 0;) {  // pass 1
    const int next = nxt[k];
    if (size > 1) {
      const int u = window_lookup(tb, S, prv[k], k, next);
      if (u < 0) {  // the host's own rounds take over
        *count = 0;
        return;
      }
      if (!u) {
        if (prv[k] >= 0) nxt[prv[k]] = next;
        else head = next;
        if (next >= 0) prv[next] = prv[k];
        --size;
        removed = true;
      }
    }
    k = next;
  }
  if (removed) {
    for (int k = head; k >= 0; k = nxt[k]) {  // pass 2, assuming no removal
      if (size <= 1) break;
      if (window_lookup(tb, S, prv[k], k, nxt[k]) >= 0) continue;
      tr[T] = Triple{prv[k], k, nxt[k]};
      flags[T] = 0;
      ++T;
    }
  }
  *count = T;
}

// batched maps: blockIdx.y = map (window tables); triples carry their map
struct SimpMap {
  SimpArgs A;
  unsigned long long *table;
};
struct TripleM {
  int below, k, above, map;
};

__global__ void __launch_bounds__(kWinNT) window_batch_kernel(const SimpMap *__restrict__ maps) {
  window_phase(maps[blockIdx.y].A, maps[blockIdx.y].table);
}

__global__ void __launch_bounds__(256) triples_batch_kernel(const SimpMap *__restrict__ maps,
                                                            const TripleM *__restrict__ tr,
                                                            int *__restrict__ flags) {
  const int t = blockIdx.y;
  __shared__ int skip;
  if (threadIdx.x == 0) skip = *((volatile int *)(flags + t));
  __syncthreads();
  if (skip) return;
  const TripleM T = tr[t];
  const SimpArgs &A = maps[T.map].A;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool any = false;
  for (int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; cell < A.cells && !any;
       cell += stride) {
    const float e = __ldg(A.ground + (int64_t)T.k * A.stride + cell);
    const float c = __ldg(A.cost + (int64_t)T.k * A.stride + cell);
    if (!(finite32(e) && c < A.c_barrier32)) continue;
    bool u = true;
    if (T.below >= 0)
      u = not_covered(e, c, __ldg(A.ground + (int64_t)T.below * A.stride + cell),
                      __ldg(A.cost + (int64_t)T.below * A.stride + cell), A.eps_e, true);
    if (u && T.above >= 0)
      u = not_covered(e, c, __ldg(A.ground + (int64_t)T.above * A.stride + cell),
                      __ldg(A.cost + (int64_t)T.above * A.stride + cell), A.eps_e, false);
    any = u;
  }
  if (__syncthreads_or(any) && threadIdx.x == 0) atomicOr(flags + t, 1);
}

__global__ void __launch_bounds__(256) unique_mask_kernel(SimpArgs A, Triple T,
                                                          unsigned char *__restrict__ mask) {
  const int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (cell >= A.cells) return;
  const float e = __ldg(A.ground + (int64_t)T.k * A.stride + cell);
  const float c = __ldg(A.cost + (int64_t)T.k * A.stride + cell);
  bool u = finite32(e) && c < A.c_barrier32;
  if (u && T.below >= 0)
    u = not_covered(e, c, __ldg(A.ground + (int64_t)T.below * A.stride + cell),
                    __ldg(A.cost + (int64_t)T.below * A.stride + cell), A.eps_e, true);
  if (u && T.above >= 0)
    u = not_covered(e, c, __ldg(A.ground + (int64_t)T.above * A.stride + cell),
                    __ldg(A.cost + (int64_t)T.above * A.stride + cell), A.eps_e, false);
  mask[cell] = u ? 1 : 0;
}

}  // namespace

int launch_unique_mask(pct_ctx *ctx, const float *ground, const float *cost, int rows, int cols,
                       int k, int below, int above, double eps_e, double c_barrier,
                       uint8_t *mask) {
  SimpArgs A{ground, cost, (int64_t)rows * cols, (int64_t)rows * cols, 0, eps_e,
             (float)c_barrier};
  if (A.cells == 0) return PCT_OK;
  unique_mask_kernel<<<(unsigned)((A.cells + 255) / 256), 256, 0, ctx->stream>>>(
      A, Triple{below, k, above}, mask);
  return check_launch(ctx, "unique_mask_kernel");
}

int run_simplify(pct_ctx *ctx, const float *ground, const float *cost, int S, int rows, int cols,
                 double eps_e, double c_barrier, std::vector<int> &keep) {
  keep.clear();
  for (int k = 0; k < S; ++k) keep.push_back(k);
  if (S <= 1) return PCT_OK;
  SimpArgs A{ground, cost, (int64_t)rows * cols, (int64_t)rows * cols, S, eps_e,
             (float)c_barrier};
  // device small buffer layout: table[S] u64 | triples | flags | count
  const size_t tbytes = (size_t)S * 8;
  const size_t need = tbytes + (size_t)S * sizeof(Triple) + (size_t)S * sizeof(int) + 64;
  if (need > 65536) {
    if (int rc = ensure_scratch(ctx, need)) return rc;
  }
  char *dbase = static_cast<char *>(need > 65536 ? ctx->scratch : ctx->dsmall);
  unsigned long long *table = reinterpret_cast<unsigned long long *>(dbase);
  Triple *dtr = reinterpret_cast<Triple *>(dbase + tbytes);
  int *dflags = reinterpret_cast<int *>(dbase + tbytes + (size_t)S * sizeof(Triple));
  int *dcount = dflags + S;

  std::vector<unsigned long long> htable(S, 0);
  PCT_CUDA(ctx, cudaMemsetAsync(table, 0, tbytes, ctx->stream));
  {
    const size_t tab_smem = (size_t)S * 8;
    if (tab_smem > 160 * 1024) return fail(ctx, PCT_E_INVALID, "too many slices for simplify");
    PCT_CUDA(ctx, cudaFuncSetAttribute(window_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)tab_smem));
    const int64_t blocks_needed = (A.cells + kWinNT - 1) / kWinNT;
    const char *wb = getenv("PCT_WIN_BLOCKS");
    const int per_sm = wb ? atoi(wb) : window_blocks_per_sm(ctx, tab_smem);
    const unsigned grid = (unsigned)std::min<int64_t>(blocks_needed, (int64_t)per_sm * ctx->num_sms);
    const char *ws = getenv("PCT_WIN_SKIP");
    // the segment window pays off on large maps (cfg2 0.35 -> 0.23 ms, cfg3
    // 1.75 -> 0.63 ms); on small ones (cfg0 / cfg1, < 1M cells) the dense
    // window is faster (cfg1 92 vs 120 us)
    const bool skip_ok = ws ? ws[0] == '1' : A.cells >= (1 << 20);
    if (ctx->simp_gm && ctx->simp_tcm && S <= 64 && eps_e >= 0.0 && skip_ok) {
      SimpMasks M{ctx->simp_gm, ctx->simp_tcm, cols, ctx->simp_th, ctx->simp_tw,
                  (cols + ctx->simp_tw - 1) / ctx->simp_tw};
      PCT_CUDA(ctx, cudaFuncSetAttribute(window_skip_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tab_smem));
      // dynamic claims (PCT_WIN_DYNAMIC=0: round robin); the counter sits in
      // the small buffer's slack after `count`
      const char *wd = getenv("PCT_WIN_DYNAMIC");
      unsigned long long *wctr = nullptr;
      if (!(wd && wd[0] == '0')) {
        wctr = reinterpret_cast<unsigned long long *>(
            (reinterpret_cast<uintptr_t>(dcount + 1) + 7) & ~(uintptr_t)7);
        PCT_CUDA(ctx, cudaMemsetAsync(wctr, 0, 8, ctx->stream));
      }
      window_skip_kernel<<<grid, kWinNT, tab_smem, ctx->stream>>>(A, M, table, wctr);
    } else {
      window_kernel<<<grid, kWinNT, tab_smem, ctx->stream>>>(A, table);
    }
  }
  if (int rc = check_launch(ctx, "window_kernel")) return rc;
  // host round trips through the context's pinned buffer (pageable copies
  // are staged and cost latency)
  const size_t rbytes = tbytes + (size_t)S * (sizeof(Triple) + sizeof(int)) + sizeof(int);
  const bool pinned = rbytes + 64 <= 65536;
  char *hbase = static_cast<char *>(ctx->hsmall);
  int spec_n = 0;
  if (pinned) {
    // first pass on the device + the second pass's triples evaluated
    // speculatively, all read back with the table in one round trip
    const char *sp = getenv("PCT_SIMPLIFY_SPEC");
    const bool spec = !(sp && sp[0] == '0');
    if (spec) {
      spec_sweep_kernel<<<1, 32, 0, ctx->stream>>>(table, S, dtr, dflags, dcount);
      if (int rc = check_launch(ctx, "spec_sweep_kernel")) return rc;
      int64_t bx = (A.cells + 1023) / 1024;
      if (bx > ctx->num_sms) bx = ctx->num_sms;
      triples_kernel<<<dim3((unsigned)bx, 8u), 256, 0, ctx->stream>>>(A, dtr, dflags, dcount);
      if (int rc = check_launch(ctx, "triples_kernel")) return rc;
      PCT_CUDA(ctx, readback_async(ctx, hbase, table, rbytes));
    } else {
      PCT_CUDA(ctx, readback_async(ctx, hbase, table, tbytes));
    }
    PCT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    std::memcpy(htable.data(), hbase, tbytes);
    if (spec) std::memcpy(&spec_n, hbase + tbytes + (size_t)S * (sizeof(Triple) + sizeof(int)),
                          sizeof(int));
  } else {
    PCT_CUDA(ctx, cudaMemcpyAsync(htable.data(), table, tbytes, cudaMemcpyDeviceToHost, ctx->stream));
    PCT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  }

  std::map<std::tuple<int, int, int>, bool> cache;
  auto from_window = [&](int below, int k, int above, bool *hit) -> bool {
    *hit = false;
    const bool above_ok = (above == k + 1) || (above < 0 && k == S - 1);
    if (!above_ok) return false;
    int bit = -1;
    if (below < 0) bit = kBit;
    else if (k - 1 - below < kWin) bit = k - 1 - below;
    if (bit < 0) return false;
    *hit = true;
    return (htable[k] >> bit) & 1ull;
  };
  if (spec_n > 0) {  // the speculated triples' answers
    const Triple *ht = reinterpret_cast<const Triple *>(hbase + tbytes);
    const int *hf = reinterpret_cast<const int *>(hbase + tbytes + (size_t)S * sizeof(Triple));
    for (int i = 0; i < spec_n; ++i) cache[{ht[i].below, ht[i].k, ht[i].above}] = hf[i] != 0;
  }
  int blocks_x = ctx->num_sms * 2;
  auto batch = [&](const std::vector<Triple> &ts) -> int {
    if (ts.empty()) return PCT_OK;
    const int T = (int)ts.size();
    int *hfl = reinterpret_cast<int *>(hbase + tbytes + (size_t)S * sizeof(Triple));
    PCT_CUDA(ctx, upload_async(ctx, dtr, ts.data(), sizeof(Triple) * T));
    PCT_CUDA(ctx, cudaMemsetAsync(dflags, 0, sizeof(int) * T, ctx->stream));
    int64_t bx = (A.cells + 255) / 256;
    if (bx > blocks_x) bx = blocks_x;
    triples_kernel<<<dim3((unsigned)bx, T), 256, 0, ctx->stream>>>(A, dtr, dflags);
    if (int rc = check_launch(ctx, "triples_kernel")) return rc;
    std::vector<int> hf(T);
    if (pinned) PCT_CUDA(ctx, readback_async(ctx, hfl, dflags, sizeof(int) * T));
    else PCT_CUDA(ctx, cudaMemcpyAsync(hf.data(), dflags, sizeof(int) * T, cudaMemcpyDeviceToHost,
                                       ctx->stream));
    PCT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (pinned) std::memcpy(hf.data(), hfl, sizeof(int) * T);
    for (int i = 0; i < T; ++i) cache[{ts[i].below, ts[i].k, ts[i].above}] = hf[i] != 0;
    return PCT_OK;
  };

  // replay of simplify.py:59-70
  for (;;) {
    bool removed = false;
    size_t p = 0;
    while (p < keep.size()) {
      if (keep.size() > 1) {
        const int k = keep[p];
        const int below = p > 0 ? keep[p - 1] : -1;
        const int above = p + 1 < keep.size() ? keep[p + 1] : -1;
        bool hit;
        bool uniq = from_window(below, k, above, &hit);
        if (!hit) {
          auto it = cache.find({below, k, above});
          if (it == cache.end()) {
            // speculate: the rest of this pass with no further removals
            std::vector<Triple> ts;
            for (size_t q = p; q < keep.size() && (int)ts.size() < S; ++q) {
              Triple t{q > 0 ? keep[q - 1] : -1, keep[q], q + 1 < keep.size() ? keep[q + 1] : -1};
              bool h2;
              from_window(t.below, t.k, t.above, &h2);
              if (!h2 && !cache.count({t.below, t.k, t.above})) ts.push_back(t);
            }
            if (int rc = batch(ts)) return rc;
            it = cache.find({below, k, above});
          }
          uniq = it->second;
        }
        if (!uniq) {
          keep.erase(keep.begin() + p);
          removed = true;
          continue;
        }
      }
      ++p;
    }
    if (!removed) break;
  }
  return PCT_OK;
}

}  // namespace pct

// ---------------------------------------------------------------------------
// primitives for a sweep replayed outside (row-band sharded maps: the any()s
// of every rank are OR-reduced before the shared sweep decides)
namespace pct {

int simplify_window_table(pct_ctx *ctx, const float *ground, const float *cost, int S,
                          int64_t cells, int64_t stride, double eps_e, double c_barrier,
                          uint64_t *table_host) {
  if (S <= 0) return PCT_OK;
  SimpArgs A{ground, cost, cells, stride, S, eps_e, (float)c_barrier};
  const size_t tbytes = (size_t)S * 8;
  if (tbytes > 65536 - 128) return fail(ctx, PCT_E_INVALID, "too many slices");
  unsigned long long *table = static_cast<unsigned long long *>(ctx->dsmall);
  PCT_CUDA(ctx, cudaMemsetAsync(table, 0, tbytes, ctx->stream));
  if (cells > 0) {
    PCT_CUDA(ctx, cudaFuncSetAttribute(window_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)tbytes));
    const int64_t blocks_needed = (cells + kWinNT - 1) / kWinNT;
    const unsigned grid = (unsigned)std::min<int64_t>(
        blocks_needed, (int64_t)window_blocks_per_sm(ctx, tbytes) * ctx->num_sms);
    window_kernel<<<grid, kWinNT, tbytes, ctx->stream>>>(A, table);
    if (int rc = check_launch(ctx, "window_kernel")) return rc;
  }
  PCT_CUDA(ctx, cudaMemcpyAsync(table_host, table, tbytes, cudaMemcpyDeviceToHost, ctx->stream));
  PCT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return PCT_OK;
}

// no host synchronisation: the table / flags land in pinned host memory
int simplify_window_async(pct_ctx *ctx, const float *ground, const float *cost, int S,
                          int64_t cells, double eps_e, double c_barrier, uint64_t *table_host) {
  if (S <= 0) return PCT_OK;
  SimpArgs A{ground, cost, cells, cells, S, eps_e, (float)c_barrier};
  const size_t tbytes = (size_t)S * 8;
  if (tbytes > 65536 - 128) return fail(ctx, PCT_E_INVALID, "too many slices");
  unsigned long long *table = static_cast<unsigned long long *>(ctx->dsmall);
  PCT_CUDA(ctx, cudaMemsetAsync(table, 0, tbytes, ctx->stream));
  if (cells > 0) {
    PCT_CUDA(ctx, cudaFuncSetAttribute(window_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)tbytes));
    const int64_t blocks_needed = (cells + kWinNT - 1) / kWinNT;
    const unsigned grid = (unsigned)std::min<int64_t>(
        blocks_needed, (int64_t)window_blocks_per_sm(ctx, tbytes) * ctx->num_sms);
    window_kernel<<<grid, kWinNT, tbytes, ctx->stream>>>(A, table);
    if (int rc = check_launch(ctx, "window_kernel")) return rc;
  }
  PCT_CUDA(ctx, cudaMemcpyAsync(table_host, table, tbytes, cudaMemcpyDeviceToHost, ctx->stream));
  return PCT_OK;
}

int simplify_triples_async(pct_ctx *ctx, const float *ground, const float *cost, int S,
                           int64_t cells, double eps_e, double c_barrier, const int32_t *tri_host,
                           int n, int32_t *flags_host) {
  if (n <= 0) return PCT_OK;
  SimpArgs A{ground, cost, cells, cells, S, eps_e, (float)c_barrier};
  const size_t need = (size_t)n * (sizeof(Triple) + sizeof(int)) + 64;
  if (need > 65536 - 128) return fail(ctx, PCT_E_INVALID, "too many triples in one batch");
  char *dbase = static_cast<char *>(ctx->dsmall);
  Triple *dtr = reinterpret_cast<Triple *>(dbase);
  int *dflags = reinterpret_cast<int *>(dbase + (size_t)n * sizeof(Triple));
  static_assert(sizeof(Triple) == 3 * sizeof(int32_t), "triple layout");
  PCT_CUDA(ctx, cudaMemcpyAsync(dtr, tri_host, sizeof(Triple) * n, cudaMemcpyHostToDevice,
                                ctx->stream));
  PCT_CUDA(ctx, cudaMemsetAsync(dflags, 0, sizeof(int) * n, ctx->stream));
  if (cells > 0) {
    int64_t bx = (cells + 255) / 256;
    if (bx > 2LL * ctx->num_sms) bx = 2LL * ctx->num_sms;
    triples_kernel<<<dim3((unsigned)bx, n), 256, 0, ctx->stream>>>(A, dtr, dflags);
    if (int rc = check_launch(ctx, "triples_kernel")) return rc;
  }
  PCT_CUDA(ctx, cudaMemcpyAsync(flags_host, dflags, sizeof(int) * n, cudaMemcpyDeviceToHost,
                                ctx->stream));
  return PCT_OK;
}

// batched maps: one window launch for every map's table (tables_host: S_max
// u64 per map, pinned), one triples launch for a round of every map's
// triples (tri_host: (below, k, above, map) int32 x n, flags_host: n)
int simplify_window_batch(pct_ctx *ctx, int n_maps, const float *const *ground,
                          const float *const *cost, const int *S, const int64_t *cells,
                          int S_max, double eps_e, double c_barrier, uint64_t *tables_host) {
  const size_t tbytes = (size_t)n_maps * S_max * 8;
  const size_t dbytes = ((sizeof(SimpMap) * (size_t)n_maps + 255) / 256) * 256;
  if ((size_t)S_max * 8 > 160 * 1024) return fail(ctx, PCT_E_INVALID, "too many slices for simplify");
  if (int rc = ensure_staging(ctx, dbytes + tbytes)) return rc;
  SimpMap *dd = static_cast<SimpMap *>(ctx->staging);
  unsigned long long *dt = reinterpret_cast<unsigned long long *>(static_cast<char *>(ctx->staging) + dbytes);
  std::vector<SimpMap> h(n_maps);
  int64_t cmax = 1;
  for (int m = 0; m < n_maps; ++m) {
    h[m].A = SimpArgs{ground[m], cost[m], cells[m], cells[m], S[m], eps_e, (float)c_barrier};
    h[m].table = dt + (size_t)m * S_max;
    cmax = std::max<int64_t>(cmax, cells[m]);
  }
  PCT_CUDA(ctx, upload_async(ctx, dd, h.data(), sizeof(SimpMap) * n_maps));
  PCT_CUDA(ctx, cudaMemsetAsync(dt, 0, tbytes, ctx->stream));
  const size_t smem = (size_t)S_max * 8;
  PCT_CUDA(ctx, cudaFuncSetAttribute(window_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  // per map about as many blocks as its cells need, the whole launch <= 12
  // resident blocks per SM
  const int64_t per_map = std::max<int64_t>(
      1, std::min<int64_t>((cmax + kWinNT - 1) / kWinNT,
                           (int64_t)window_blocks_per_sm(ctx, smem) * ctx->num_sms / std::max(1, n_maps)));
  window_batch_kernel<<<dim3((unsigned)per_map, n_maps), kWinNT, smem, ctx->stream>>>(dd);
  if (int rc = check_launch(ctx, "window_batch_kernel")) return rc;
  PCT_CUDA(ctx, cudaMemcpyAsync(tables_host, dt, tbytes, cudaMemcpyDeviceToHost, ctx->stream));
  return PCT_OK;
}

int simplify_triples_batch(pct_ctx *ctx, int n_maps, int n, const int32_t *tri_host,
                           int32_t *flags_host) {
  if (n <= 0) return PCT_OK;
  // descriptors stay in the staging buffer from simplify_window_batch
  const size_t dbytes = ((sizeof(SimpMap) * (size_t)n_maps + 255) / 256) * 256;
  SimpMap *dd = static_cast<SimpMap *>(ctx->staging);
  const size_t need = (size_t)n * (sizeof(TripleM) + sizeof(int)) + 64;
  if (int rc = ensure_scratch(ctx, need)) return rc;
  TripleM *dtr = static_cast<TripleM *>(ctx->scratch);
  int *dflags = reinterpret_cast<int *>(dtr + n);
  (void)dbytes;
  PCT_CUDA(ctx, cudaMemcpyAsync(dtr, tri_host, sizeof(TripleM) * n, cudaMemcpyHostToDevice,
                                ctx->stream));
  PCT_CUDA(ctx, cudaMemsetAsync(dflags, 0, sizeof(int) * n, ctx->stream));
  triples_batch_kernel<<<dim3(8, n), 256, 0, ctx->stream>>>(dd, dtr, dflags);
  if (int rc = check_launch(ctx, "triples_batch_kernel")) return rc;
  PCT_CUDA(ctx, cudaMemcpyAsync(flags_host, dflags, sizeof(int) * n, cudaMemcpyDeviceToHost,
                                ctx->stream));
  return PCT_OK;
}

int simplify_triple_flags(pct_ctx *ctx, const float *ground, const float *cost, int S,
                          int64_t cells, int64_t stride, double eps_e, double c_barrier,
                          const int32_t *triples, int n, int32_t *flags_host) {
  if (n <= 0) return PCT_OK;
  SimpArgs A{ground, cost, cells, stride, S, eps_e, (float)c_barrier};
  const size_t need = (size_t)n * (sizeof(Triple) + sizeof(int)) + 64;
  if (need > 65536 - 128) return fail(ctx, PCT_E_INVALID, "too many triples in one batch");
  char *dbase = static_cast<char *>(ctx->dsmall);
  Triple *dtr = reinterpret_cast<Triple *>(dbase);
  int *dflags = reinterpret_cast<int *>(dbase + (size_t)n * sizeof(Triple));
  std::vector<Triple> ts(n);
  for (int i = 0; i < n; ++i) ts[i] = Triple{triples[3 * i], triples[3 * i + 1], triples[3 * i + 2]};
  PCT_CUDA(ctx, cudaMemcpyAsync(dtr, ts.data(), sizeof(Triple) * n, cudaMemcpyHostToDevice,
                                ctx->stream));
  PCT_CUDA(ctx, cudaMemsetAsync(dflags, 0, sizeof(int) * n, ctx->stream));
  if (cells > 0) {
    int64_t bx = (cells + 255) / 256;
    if (bx > 2LL * ctx->num_sms) bx = 2LL * ctx->num_sms;
    triples_kernel<<<dim3((unsigned)bx, n), 256, 0, ctx->stream>>>(A, dtr, dflags);
    if (int rc = check_launch(ctx, "triples_kernel")) return rc;
  }
  PCT_CUDA(ctx, cudaMemcpyAsync(flags_host, dflags, sizeof(int) * n, cudaMemcpyDeviceToHost,
                                ctx->stream));
  PCT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return PCT_OK;
}

}  // namespace pct
