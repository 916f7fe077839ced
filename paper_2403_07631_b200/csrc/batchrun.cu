// batchrun.cu — pct_tomo_run_batch: the whole hot path for many independent
// maps (BASELINE config 4) with one launch per stage for the whole batch.
//
// A small map (config 0/4: 250k points, 203 x 204 x 13) fills a fraction of
// the GPU per kernel and pct_tomo_run adds three host synchronisations per
// map.  Here each stage runs once over every map of a group (descriptor
// arrays in device memory; blockIdx.y or flattened work items pick the map):
//   1  bounds (one launch)                                          -> sync
//   2  frames on the host; build (scatter + scan), evaluate (walk +
//      branch-and-bound resolve/inflate), simplify window tables, one launch
//      each                                                         -> sync
//   3  simplify replays on the host (SweepState, exactly as run_simplify);
//      each round's triples of every map in one launch              -> sync
// Results equal pct_tomo_run map by map (tests/test_gpu_parity.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "pct_internal.h"

// capi.cu (defined inside its extern "C" block)
extern "C" int tomo_alloc(pct_ctx *ctx, const pct_frame &fr, pct_tomo **out);

namespace pct {
namespace {

constexpr int kWinB = 16;  // window of simplify_window_async's table (k_simplify.cu)
constexpr int kBitB = 32;  // its "no lower neighbour" bit

// resumable replay of simplify.py:59-70 over one map's table
struct SweepState {
  int S = 0;
  std::vector<int> keep;
  const uint64_t *table = nullptr;
  std::map<std::tuple<int, int, int>, bool> cache;
  size_t p = 0;
  bool removed = false;
  bool done = false;

  bool from_window(int below, int k, int above, bool *hit) const {
    *hit = false;
    const bool above_ok = (above == k + 1) || (above < 0 && k == S - 1);
    if (!above_ok) return false;
    int bit = -1;
    if (below < 0) bit = kBitB;
    else if (k - 1 - below < kWinB) bit = k - 1 - below;
    if (bit < 0) return false;
    *hit = true;
    return (table[k] >> bit) & 1ull;
  }

  // advance; returns false with `need` filled when triples must be evaluated
  bool run(std::vector<int32_t> &need) {
    need.clear();
    for (;;) {
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
              for (size_t q = p; q < keep.size() && (int)(need.size() / 3) < S; ++q) {
                const int tb = q > 0 ? keep[q - 1] : -1, tk = keep[q];
                const int ta = q + 1 < keep.size() ? keep[q + 1] : -1;
                bool h2;
                from_window(tb, tk, ta, &h2);
                if (!h2 && !cache.count({tb, tk, ta})) {
                  need.push_back(tb);
                  need.push_back(tk);
                  need.push_back(ta);
                }
              }
              return false;
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
      if (!removed) {
        done = true;
        return true;
      }
      p = 0;
      removed = false;
    }
  }

  void feed(const std::vector<int32_t> &tri, const int32_t *flags) {
    for (size_t i = 0; i < tri.size() / 3; ++i)
      cache[{tri[3 * i], tri[3 * i + 1], tri[3 * i + 2]}] = flags[i] != 0;
  }
};

int sync_all(pct_ctx **ctxs, int n_ctx) {
  for (int c = 0; c < n_ctx; ++c) PCT_CUDA(ctxs[c], cudaStreamSynchronize(ctxs[c]->stream));
  return PCT_OK;
}

int ensure_pinned(pct_ctx *ctx, size_t bytes) {
  if (ctx->pinned_batch_bytes >= bytes) return PCT_OK;
  if (ctx->pinned_batch) cudaFreeHost(ctx->pinned_batch);
  ctx->pinned_batch = nullptr;
  ctx->pinned_batch_bytes = 0;
  const size_t want = bytes + bytes / 4;
  PCT_CUDA(ctx, cudaMallocHost(&ctx->pinned_batch, want));
  ctx->pinned_batch_bytes = want;
  return PCT_OK;
}

}  // namespace
}  // namespace pct

using namespace pct;

namespace {

// one group of <= kGroup maps: every stage is one launch for the whole group
constexpr int kGroup = 512;

int run_group(pct_ctx *c0, int n_maps, const void *const *xyz, const int64_t *n_points,
              int dtype, double d_s, double r_g, int64_t max_grid_side, const pct_trav_params *p,
              const float *kernel_w, int32_t kside, double eps_e, double c_barrier,
              pct_tomo **out, int32_t *keep_host, int32_t keep_stride, int32_t *n_keep) {
  // 1. bounds (one launch, keys into pinned slots)
  if (c0->timing) cudaEventRecord(c0->ev[0], c0->stream);  // stage events as pct_tomo_run
  if (int rc = ensure_pinned(c0, (size_t)n_maps * 64 + 64)) return rc;
  unsigned long long *bk = static_cast<unsigned long long *>(c0->pinned_batch);
  if (int rc = launch_bounds_batch(c0, n_maps, xyz, n_points, dtype, bk)) return rc;
  PCT_CUDA(c0, cudaStreamSynchronize(c0->stream));
  // 2. frames; build, evaluate, simplify tables: one launch per stage
  std::vector<pct_frame> frames(n_maps);
  std::vector<std::vector<double>> heights(n_maps);
  int max_S = 1;
  for (int m = 0; m < n_maps; ++m) {
    double lo[3], hi[3];
    if (!bounds_from_keys(bk + 8 * (size_t)m, lo, hi))
      return fail(c0, PCT_E_NONFINITE, "point cloud contains non-finite coordinates");
    const int rc = pct_frame_compute(lo, hi, d_s, r_g, max_grid_side, &frames[m], nullptr, 0);
    if (rc == PCT_E_GRID)
      return fail(c0, PCT_E_GRID, "grid " + std::to_string(frames[m].rows) + "x" +
                                      std::to_string(frames[m].cols) + " exceeds the " +
                                      std::to_string(max_grid_side) + " per-side limit");
    if (rc) return fail(c0, rc, "invalid grid frame");
    heights[m].resize(frames[m].n_slices);
    pct_frame_compute(lo, hi, d_s, r_g, max_grid_side, &frames[m], heights[m].data(),
                      frames[m].n_slices);
    max_S = std::max(max_S, frames[m].n_slices);
  }
  if (max_S > keep_stride) return fail(c0, PCT_E_INVALID, "keep_stride below the slice count");
  std::vector<pct_tomo *> toms(n_maps, nullptr);
  auto free_all = [&]() {
    for (int m = 0; m < n_maps; ++m)
      if (toms[m]) pct_tomo_free(c0, toms[m]);
  };
  std::vector<float *> g(n_maps), c(n_maps), co(n_maps);
  std::vector<const double *> hp(n_maps);
  std::vector<int> Sv(n_maps);
  std::vector<int64_t> cells(n_maps);
  for (int m = 0; m < n_maps; ++m) {
    const pct_frame &fr = frames[m];
    if (int rc = tomo_alloc(c0, fr, &toms[m])) {
      free_all();
      return rc;
    }
    pct_tomo *t = toms[m];
    t->heights = heights[m];
    const size_t bytes = (size_t)fr.n_slices * fr.rows * fr.cols * sizeof(float);
    if (cudaMallocFromPoolAsync(reinterpret_cast<void **>(&t->cost), bytes, c0->mempool, c0->stream) != cudaSuccess) {
      free_all();
      return fail(c0, PCT_E_NOMEM, "cudaMallocAsync(cost)");
    }
    g[m] = t->ground;
    c[m] = t->ceiling;
    co[m] = t->cost;
    hp[m] = t->heights.data();
    Sv[m] = fr.n_slices;
    cells[m] = (int64_t)fr.rows * fr.cols;
  }
  // pinned: tables (S_max u64 per map) | triples (4 x S_max i32 per map) |
  // flags (S_max i32 per map); the bounds keys are consumed
  const size_t tab_b = (size_t)n_maps * max_S * 8, tri_b = (size_t)n_maps * max_S * 16,
               flg_b = (size_t)n_maps * max_S * 4;
  if (int rc = ensure_pinned(c0, tab_b + tri_b + flg_b + 256)) {
    free_all();
    return rc;
  }
  char *pb = static_cast<char *>(c0->pinned_batch);
  uint64_t *tables = reinterpret_cast<uint64_t *>(pb);
  int32_t *tris = reinterpret_cast<int32_t *>(pb + tab_b);
  int32_t *flags = reinterpret_cast<int32_t *>(pb + tab_b + tri_b);
  int rc = launch_build_batch(c0, n_maps, xyz, n_points, dtype, frames.data(), hp.data(), g.data(),
                              c.data());
  if (!rc && c0->timing) cudaEventRecord(c0->ev[1], c0->stream);
  if (!rc) rc = launch_evaluate_batch(c0, n_maps, g.data(), c.data(), frames.data(), *p, kernel_w,
                                      kside, co.data());
  if (!rc && c0->timing) cudaEventRecord(c0->ev[2], c0->stream);
  if (!rc) rc = simplify_window_batch(c0, n_maps, g.data(), co.data(), Sv.data(), cells.data(),
                                     max_S, eps_e, c_barrier, tables);
  if (!rc && cudaStreamSynchronize(c0->stream) != cudaSuccess) rc = fail(c0, PCT_E_CUDA, "sync");
  if (rc) {
    free_all();
    return rc;
  }
  // 3. simplify replays; each round's triples of every map in one launch
  std::vector<SweepState> sw(n_maps);
  for (int m = 0; m < n_maps; ++m) {
    sw[m].S = frames[m].n_slices;
    sw[m].table = tables + (size_t)m * max_S;
    for (int k = 0; k < sw[m].S; ++k) sw[m].keep.push_back(k);
  }
  std::vector<std::vector<int32_t>> need(n_maps);
  std::vector<int> first(n_maps);
  for (;;) {
    int total = 0;
    for (int m = 0; m < n_maps; ++m) {
      first[m] = total;
      if (sw[m].done || sw[m].run(need[m])) {
        need[m].clear();
        continue;
      }
      for (size_t i = 0; i < need[m].size() / 3; ++i) {
        int32_t *t = tris + 4 * (size_t)(total++);
        t[0] = need[m][3 * i];
        t[1] = need[m][3 * i + 1];
        t[2] = need[m][3 * i + 2];
        t[3] = m;
      }
    }
    if (total == 0) break;
    if ((rc = simplify_triples_batch(c0, n_maps, total, tris, flags)) ||
        cudaStreamSynchronize(c0->stream) != cudaSuccess) {
      free_all();
      return rc ? rc : fail(c0, PCT_E_CUDA, "sync");
    }
    for (int m = 0; m < n_maps; ++m)
      if (!need[m].empty()) sw[m].feed(need[m], flags + first[m]);
  }
  if (c0->timing) cudaEventRecord(c0->ev[3], c0->stream);
  for (int m = 0; m < n_maps; ++m) {
    n_keep[m] = (int32_t)sw[m].keep.size();
    for (size_t i = 0; i < sw[m].keep.size(); ++i)
      keep_host[(size_t)m * keep_stride + i] = sw[m].keep[i];
    if (out) out[m] = toms[m];
    else pct_tomo_free(c0, toms[m]);
    toms[m] = nullptr;
  }
  return PCT_OK;
}

}  // namespace

extern "C" int pct_tomo_run_batch(pct_ctx **ctxs, int32_t n_ctx, int32_t n_maps,
                                  const void *const *xyz, const int64_t *n_points, int dtype,
                                  double d_s, double r_g, int64_t max_grid_side,
                                  const pct_trav_params *p, const float *kernel_w, int32_t kside,
                                  double eps_e, double c_barrier, pct_tomo **out,
                                  int32_t *keep_host, int32_t keep_stride, int32_t *n_keep) {
  if (!ctxs || n_ctx <= 0 || !ctxs[0]) return PCT_E_INVALID;
  pct_ctx *c0 = ctxs[0];
  if (n_maps < 0 || !xyz || !n_points || !p || !kernel_w || !keep_host || !n_keep ||
      keep_stride <= 0 || (dtype != PCT_F32 && dtype != PCT_F64))
    return fail(c0, PCT_E_INVALID, "bad arguments to pct_tomo_run_batch");
  if (!(d_s > 0) || !(r_g > 0)) return fail(c0, PCT_E_INVALID, "d_s and r_g must be positive");
  PCT_CUDA(c0, cudaSetDevice(c0->device));
  for (int m = 0; m < n_maps; ++m)
    if (n_points[m] <= 0) return fail(c0, PCT_E_EMPTY, "zero valid points");
  for (int m0 = 0; m0 < n_maps; m0 += kGroup) {
    const int nm = std::min(kGroup, n_maps - m0);
    if (int rc = run_group(c0, nm, xyz + m0, n_points + m0, dtype, d_s, r_g, max_grid_side, p,
                           kernel_w, kside, eps_e, c_barrier, out ? out + m0 : nullptr,
                           keep_host + (size_t)m0 * keep_stride, keep_stride, n_keep + m0))
      return rc;
  }
  return PCT_OK;
}
