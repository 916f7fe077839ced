// pct_internal.h — context, device tomogram and kernel launchers shared by
// the translation units of libpct.so (not part of the public ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/pct.h"
#include "cellmath.cuh"

constexpr int kXferEvents = 8;  // event slots of pct_xfer_fence / pct_xfer_wait

struct pct_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  std::string err;
  int64_t launches = 0;
  // grow-only device scratch (build keys, staging of host points)
  void *scratch = nullptr;
  size_t scratch_bytes = 0;
  void *staging = nullptr;  // device copy of host xyz / PCD payload chunks
  size_t staging_bytes = 0;
  void *pinned_io = nullptr;  // pinned double buffer of the PCD file reader
  size_t pinned_io_bytes = 0;
  void *pinned_batch = nullptr;  // per-map result slots of pct_tomo_run_batch
  size_t pinned_batch_bytes = 0;
  // pinned ring for small host->device copies (constants, descriptors,
  // heights): copies from pageable memory may synchronise with the stream
  cudaMemPool_t mempool = nullptr;  // this context's stream-ordered allocations
  void *upload = nullptr;
  size_t upload_off = 0;
  // small device/pinned buffers for reductions and flags
  void *dsmall = nullptr;   // 64 KiB device
  void *hsmall = nullptr;   // 64 KiB pinned host
  // build key planes (gkey | ckey): the scan resets every key it reads, so a
  // layout that was built once needs no memset (keys_tag = S, cells)
  void *keys = nullptr;
  size_t keys_bytes = 0;
  int64_t keys_tag[2] = {-1, -1};
  // single-map layout: ground keys in the first half of the buffer, ceiling
  // keys in the second; clean = every key empty (the scan restores that)
  bool keys_clean = false;
  cudaEvent_t spec_ev = nullptr;  // bounds read back ahead of the speculative scatter
  cudaEvent_t switch_ev = nullptr;  // pct_set_stream: old stream -> new stream join
  cudaEvent_t xfer_ev[8] = {};      // pct_xfer_fence / pct_xfer_wait slots
  // per-cell slice-change masks ([2][cells] uint64: ground, ceiling; bit k =
  // the layer differs from slice k-1, bit 0 set; S <= 64): build_masks, when
  // set, is where the whole-grid build writes them; eval_masks, when set,
  // the evaluation's walk reads them instead of deriving them again
  unsigned long long *build_masks = nullptr;
  bool build_masks_written = false;
  const unsigned long long *eval_masks = nullptr;
  // per evaluation tile (th x tw cells): bit k = the tile's costs may differ
  // from slice k-1.  eval_tcm, when set, is where the bnb evaluation writes
  // them (eval_tcm_written, geometry in tcm_th / tcm_tw); simp_gm / simp_tcm,
  // when set, let the simplify window read only where values change
  unsigned long long *eval_tcm = nullptr;
  bool eval_tcm_written = false;
  int tcm_th = 0, tcm_tw = 0;
  const unsigned long long *simp_gm = nullptr, *simp_tcm = nullptr;
  int simp_th = 0, simp_tw = 0;
  // zero-padded encoded c_init stacks of the split evaluation; the padding
  // is cleared only when the layout changes (the interior is rewritten)
  void *enc = nullptr;
  size_t enc_bytes = 0;
  int64_t enc_tag[6] = {-1, -1, -1, -1, -1, -1};  // S, rows, cols, R, tile h, w of the cleared layout
  // optional stage events of pct_tomo_run (pct_set_timing)
  bool timing = false;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
};

struct pct_tomo {
  pct_frame fr{};
  std::vector<double> heights;
  float *ground = nullptr;   // (S, rows, cols)
  float *ceiling = nullptr;
  float *cost = nullptr;     // nullptr until evaluated
  // slice-change masks written by the build (S <= 64), read by the walk
  unsigned long long *masks = nullptr;
  // per evaluation tile cost-change masks written by the evaluation (S <= 64)
  unsigned long long *tcm = nullptr;
  int tcm_th = 0, tcm_tw = 0;
};

namespace pct {

int fail(pct_ctx *ctx, int code, const std::string &msg);
int cuda_fail(pct_ctx *ctx, cudaError_t e, const char *what);
int ensure_scratch(pct_ctx *ctx, size_t bytes);
int ensure_staging(pct_ctx *ctx, size_t bytes);
int check_launch(pct_ctx *ctx, const char *what);
// copy n bytes of host data into the context's pinned upload ring and return
// the pinned address (src itself if it does not fit)
const void *pin_upload(pct_ctx *ctx, const void *src, size_t n);
// small transfers moved by a kernel through mapped pinned memory instead of
// the copy engines, so they never queue behind another context's bulk copy:
// upload_async stages src in the upload ring and copies it to ddst;
// readback_async copies n bytes of device memory to pinned host memory hdst
// (visible to the host after the stream synchronises)
cudaError_t upload_async(pct_ctx *ctx, void *ddst, const void *src, size_t n);

// __constant__ symbols (parameters, inflation weights) are shared by every
// context on a device.  A ConstBank scope serialises their use: set() skips
// the upload when the symbol already holds these bytes (waiting for the
// upload that put them there), and before changing them waits for every
// other context's last launch that read constants; the destructor records
// this context's use after the launches made inside the scope.
class ConstBank {
 public:
  explicit ConstBank(pct_ctx *ctx);
  ~ConstBank();
  ConstBank(const ConstBank &) = delete;
  ConstBank &operator=(const ConstBank &) = delete;
  cudaError_t set(void *symbol_addr, const void *src, size_t n);
  template <class T>
  cudaError_t set_symbol(const T &symbol, const void *src, size_t n) {
    void *d = nullptr;
    cudaError_t e = cudaGetSymbolAddress(&d, symbol);
    return e == cudaSuccess ? set(d, src, n) : e;
  }

 private:
  pct_ctx *ctx_;
};
void const_bank_forget(pct_ctx *ctx);  // context teardown
cudaError_t readback_async(pct_ctx *ctx, void *hdst, const void *dsrc, size_t n);

#define PCT_CUDA(ctx, call)                                  \
  do {                                                       \
    cudaError_t e_ = (call);                                 \
    if (e_ != cudaSuccess) return pct::cuda_fail(ctx, e_, #call); \
  } while (0)

// stage launchers (return PCT_OK or error code)
int launch_bounds(pct_ctx *ctx, const void *xyz, int64_t n, int dtype, double lo[3],
                  double hi[3]);
// row0/nrows select a band of global rows (nrows < 0: whole grid); output
// slice k at k*out_stride floats (<= 0: dense)
int launch_build(pct_ctx *ctx, const void *xyz, int64_t n, int dtype, const pct_frame &fr,
                 const double *heights_host, float *ground, float *ceiling, int row0 = 0,
                 int nrows = -1, int64_t out_stride = 0, bool keys_scattered = false);
// bounds + (when the key buffer allows) the scatter of the frame the device
// derives from them, before the host has the bounds: *scattered tells
// whether the keys of that frame are already in place
int launch_bounds_spec(pct_ctx *ctx, const void *xyz, int64_t n, int dtype, double d_s,
                       double r_g, int64_t max_grid_side, double lo[3], double hi[3],
                       pct_frame *dev_frame, bool *scattered);
int launch_evaluate(pct_ctx *ctx, const float *ground, const float *ceiling, int S, int rows,
                    int cols, double r_g, const pct_trav_params &p, const float *kernel_w,
                    int kside, float *cost, int mode);
int launch_inflate(pct_ctx *ctx, const float *cost, int rows, int cols, const float *kernel_w,
                   int kside, float *out);
int run_simplify(pct_ctx *ctx, const float *ground, const float *cost, int S, int rows,
                 int cols, double eps_e, double c_barrier, std::vector<int> &keep);
int launch_unique_mask(pct_ctx *ctx, const float *ground, const float *cost, int rows, int cols,
                       int k, int below, int above, double eps_e, double c_barrier,
                       uint8_t *mask);

EvalConsts make_consts(const pct_trav_params &p, double r_g);

// asynchronous pieces of the whole-pipeline call (results land in pinned
// host memory; the caller synchronises the stream) used by pct_tomo_run_batch
int launch_bounds_async(pct_ctx *ctx, const void *xyz, int64_t n, int dtype,
                        unsigned long long *keys_host, const unsigned long long *init_host);
bool bounds_from_keys(const unsigned long long *keys, double lo[3], double hi[3]);
// batched maps: one launch per stage (keys_host: 8 u64 per map, pinned)
int launch_bounds_batch(pct_ctx *ctx, int n_maps, const void *const *xyz, const int64_t *n,
                        int dtype, unsigned long long *keys_host);
int simplify_window_batch(pct_ctx *ctx, int n_maps, const float *const *ground,
                          const float *const *cost, const int *S, const int64_t *cells,
                          int S_max, double eps_e, double c_barrier, uint64_t *tables_host);
int simplify_triples_batch(pct_ctx *ctx, int n_maps, int n, const int32_t *tri_host,
                           int32_t *flags_host);
int launch_evaluate_batch(pct_ctx *ctx, int n_maps, float *const *ground,
                          float *const *ceiling, const pct_frame *frames,
                          const pct_trav_params &p, const float *kernel_w, int kside,
                          float *const *cost);
int launch_build_batch(pct_ctx *ctx, int n_maps, const void *const *xyz, const int64_t *n,
                       int dtype, const pct_frame *frames, const double *const *heights,
                       float *const *ground, float *const *ceiling);
int simplify_window_async(pct_ctx *ctx, const float *ground, const float *cost, int S,
                          int64_t cells, double eps_e, double c_barrier, uint64_t *table_host);
int simplify_triples_async(pct_ctx *ctx, const float *ground, const float *cost, int S,
                           int64_t cells, double eps_e, double c_barrier, const int32_t *tri_host,
                           int n, int32_t *flags_host);

// evaluate modes for the per-op entry points
enum EvalMode { kEvalFull = 0, kEvalGroundCost = 1, kEvalInterval = 2, kEvalCinit = 3 };

}  // namespace pct
