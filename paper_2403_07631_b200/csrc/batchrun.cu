// batchrun.cu — pct_tomo_run_batch: the whole hot path for many independent
// maps (BASELINE config 4) from one host thread.
//
// pct_tomo_run synchronises three times per map (bounds -> grid frame, the
// simplify table, triple batches).  Here the maps are spread over several
// contexts (one CUDA stream and one set of scratch buffers each; map m goes
// to context m % n_ctx) and the work is issued phase by phase, so each phase
// costs one synchronisation for the whole batch:
//   1  bounds of every map (keys into pinned per-map slots)       -> sync
//   2  frames on the host; build + evaluate + simplify window table of every
//      map (tables into pinned slots)                             -> sync
//   3  rounds of the simplify replay: every map whose sweep needs triples the
//      table cannot answer posts them; one triples launch per such map,
//      one sync per round (SweepState replays simplify.py:59-70 exactly as
//      run_simplify does)
// Within a context, stream order protects its scratch buffers between maps.
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
  for (int c = 0; c < n_ctx; ++c)
    if (!ctxs[c] || ctxs[c]->device != c0->device)
      return fail(c0, PCT_E_INVALID, "batch contexts must share one device");
  PCT_CUDA(c0, cudaSetDevice(c0->device));
  for (int m = 0; m < n_maps; ++m)
    if (n_points[m] <= 0) return fail(c0, PCT_E_EMPTY, "zero valid points");
  auto ctx_of = [&](int m) { return ctxs[m % n_ctx]; };

  // pinned slots: init keys | bounds keys (8 u64 per map) | tables | triples
  // | flags (tables / triples sized once the frames are known)
  const size_t bounds_bytes = 64 + (size_t)n_maps * 64;
  if (int rc = ensure_pinned(c0, bounds_bytes)) return rc;
  unsigned long long *init = static_cast<unsigned long long *>(c0->pinned_batch);
  const unsigned long long init_v[7] = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull, 0ull};
  std::memcpy(init, init_v, sizeof(init_v));
  // 1. bounds
  for (int m = 0; m < n_maps; ++m) {
    unsigned long long *slot = init + 8 + 8 * (size_t)m;
    if (int rc = launch_bounds_async(ctx_of(m), xyz[m], n_points[m], dtype, slot, init))
      return rc;
  }
  if (int rc = sync_all(ctxs, n_ctx)) return rc;
  // 2. frames, build, evaluate, simplify window table
  std::vector<pct_frame> frames(n_maps);
  std::vector<std::vector<double>> heights(n_maps);
  int max_S = 1;
  for (int m = 0; m < n_maps; ++m) {
    double lo[3], hi[3];
    if (!bounds_from_keys(init + 8 + 8 * (size_t)m, lo, hi))
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
  // tables (S u64 per map) | triples (3 S i32 per map) | flags (S i32 per map);
  // the bounds slots are no longer needed
  const size_t tab_b = (size_t)n_maps * max_S * 8, tri_b = (size_t)n_maps * max_S * 12,
               flg_b = (size_t)n_maps * max_S * 4;
  if (int rc = ensure_pinned(c0, tab_b + tri_b + flg_b + 256)) return rc;
  char *pb = static_cast<char *>(c0->pinned_batch);
  uint64_t *tables = reinterpret_cast<uint64_t *>(pb);
  int32_t *tris = reinterpret_cast<int32_t *>(pb + tab_b);
  int32_t *flags = reinterpret_cast<int32_t *>(pb + tab_b + tri_b);
  std::vector<pct_tomo *> toms(n_maps, nullptr);
  auto free_all = [&]() {
    for (int m = 0; m < n_maps; ++m)
      if (toms[m]) pct_tomo_free(ctx_of(m), toms[m]);
  };
  for (int m = 0; m < n_maps; ++m) {
    pct_ctx *ctx = ctx_of(m);
    const pct_frame &fr = frames[m];
    int rc = tomo_alloc(ctx, fr, &toms[m]);
    if (rc) {
      free_all();
      return rc;
    }
    pct_tomo *t = toms[m];
    t->heights = heights[m];
    const size_t bytes = (size_t)fr.n_slices * fr.rows * fr.cols * sizeof(float);
    if (cudaMallocAsync(reinterpret_cast<void **>(&t->cost), bytes, ctx->stream) != cudaSuccess) {
      free_all();
      return fail(c0, PCT_E_NOMEM, "cudaMallocAsync(cost)");
    }
    if ((rc = launch_build(ctx, xyz[m], n_points[m], dtype, fr, t->heights.data(), t->ground,
                           t->ceiling)) ||
        (rc = launch_evaluate(ctx, t->ground, t->ceiling, fr.n_slices, fr.rows, fr.cols, fr.r_g,
                              *p, kernel_w, kside, t->cost, kEvalFull)) ||
        (rc = simplify_window_async(ctx, t->ground, t->cost, fr.n_slices,
                                    (int64_t)fr.rows * fr.cols, eps_e, c_barrier,
                                    tables + (size_t)m * max_S))) {
      if (ctx != c0) c0->err = ctx->err;
      free_all();
      return rc;
    }
  }
  if (int rc = sync_all(ctxs, n_ctx)) {
    free_all();
    return rc;
  }
  // 3. simplify replays, triple batches in rounds
  std::vector<SweepState> sw(n_maps);
  for (int m = 0; m < n_maps; ++m) {
    sw[m].S = frames[m].n_slices;
    sw[m].table = tables + (size_t)m * max_S;
    for (int k = 0; k < sw[m].S; ++k) sw[m].keep.push_back(k);
  }
  std::vector<std::vector<int32_t>> need(n_maps);
  for (;;) {
    bool any = false;
    for (int m = 0; m < n_maps; ++m) {
      if (sw[m].done) continue;
      if (sw[m].run(need[m])) continue;
      const int n = (int)(need[m].size() / 3);
      if (n == 0) continue;  // cannot happen: a miss always yields its own triple
      std::memcpy(tris + (size_t)m * max_S * 3, need[m].data(), need[m].size() * 4);
      pct_ctx *ctx = ctx_of(m);
      const pct_frame &fr = frames[m];
      if (int rc = simplify_triples_async(ctx, toms[m]->ground, toms[m]->cost, fr.n_slices,
                                          (int64_t)fr.rows * fr.cols, eps_e, c_barrier,
                                          tris + (size_t)m * max_S * 3, n,
                                          flags + (size_t)m * max_S)) {
        free_all();
        return rc;
      }
      any = true;
    }
    if (!any) break;
    if (int rc = sync_all(ctxs, n_ctx)) {
      free_all();
      return rc;
    }
    for (int m = 0; m < n_maps; ++m)
      if (!sw[m].done && !need[m].empty()) sw[m].feed(need[m], flags + (size_t)m * max_S);
  }
  for (int m = 0; m < n_maps; ++m) {
    n_keep[m] = (int32_t)sw[m].keep.size();
    for (size_t i = 0; i < sw[m].keep.size(); ++i)
      keep_host[(size_t)m * keep_stride + i] = sw[m].keep[i];
    if (out) {
      out[m] = toms[m];
    } else {
      pct_tomo_free(ctx_of(m), toms[m]);
    }
    toms[m] = nullptr;
  }
  return PCT_OK;
}
