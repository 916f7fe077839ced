// capi.cu — extern "C" entry points of libpct.so (include/pct.h).
//
// Validation happens here, before any launch, with the reference's error
// texts (tomogram.py:134-142, traversability.py:61-62,196-197,
// simplify.py:34-50).  CUDA failures become PCT_E_CUDA with the runtime's
// message; nothing throws across the ABI.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "pct_internal.h"

namespace pct {

int fail(pct_ctx *ctx, int code, const std::string &msg) {
  if (ctx) ctx->err = msg;
  return code;
}

int cuda_fail(pct_ctx *ctx, cudaError_t e, const char *what) {
  return fail(ctx, e == cudaErrorMemoryAllocation ? PCT_E_NOMEM : PCT_E_CUDA,
              std::string(what) + ": " + cudaGetErrorString(e));
}

int check_launch(pct_ctx *ctx, const char *what) {
  ctx->launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, what);
  return PCT_OK;
}

static int ensure_buffer(pct_ctx *ctx, void **buf, size_t *have, size_t bytes) {
  if (*have >= bytes) return PCT_OK;
  if (*buf) {
    cudaStreamSynchronize(ctx->stream);
    cudaFree(*buf);
    *buf = nullptr;
    *have = 0;
  }
  size_t want = bytes + bytes / 8;
  cudaError_t e = cudaMalloc(buf, want);
  if (e != cudaSuccess) {
    cudaGetLastError();
    e = cudaMalloc(buf, bytes);
    want = bytes;
  }
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc(scratch)");
  *have = want;
  return PCT_OK;
}

constexpr size_t kUploadRing = 256 * 1024;

const void *pin_upload(pct_ctx *ctx, const void *src, size_t n) {
  if (!ctx->upload || n > kUploadRing / 4) return src;
  size_t off = (ctx->upload_off + 15) & ~(size_t)15;
  if (off + n > kUploadRing) {  // wrap: the oldest copies must have run
    cudaStreamSynchronize(ctx->stream);
    off = 0;
  }
  char *dst = static_cast<char *>(ctx->upload) + off;
  std::memcpy(dst, src, n);
  ctx->upload_off = off + n;
  return dst;
}

namespace {
__global__ void small_copy_kernel(uint32_t *__restrict__ dst, const uint32_t *__restrict__ src,
                                  size_t words, unsigned char *__restrict__ dtail,
                                  const unsigned char *__restrict__ stail, int ntail) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < words;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
  if (blockIdx.x == 0 && (int)threadIdx.x < ntail) dtail[threadIdx.x] = stail[threadIdx.x];
}

cudaError_t small_copy(pct_ctx *ctx, void *dst, const void *src, size_t n) {
  if (n == 0) return cudaSuccess;
  if ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 3)
    return cudaMemcpyAsync(dst, src, n, cudaMemcpyDefault, ctx->stream);
  const size_t words = n / 4;
  const int ntail = (int)(n & 3);
  const unsigned grid = (unsigned)std::max<size_t>(1, std::min<size_t>((words + 255) / 256, 64));
  small_copy_kernel<<<grid, 256, 0, ctx->stream>>>(
      static_cast<uint32_t *>(dst), static_cast<const uint32_t *>(src), words,
      static_cast<unsigned char *>(dst) + 4 * words,
      static_cast<const unsigned char *>(src) + 4 * words, ntail);
  ctx->launches++;
  return cudaGetLastError();
}
}  // namespace

cudaError_t upload_async(pct_ctx *ctx, void *ddst, const void *src, size_t n) {
  const void *p = pin_upload(ctx, src, n);
  if (p == src) return cudaMemcpyAsync(ddst, src, n, cudaMemcpyHostToDevice, ctx->stream);
  return small_copy(ctx, ddst, p, n);  // pinned host memory is device-addressable (UVA)
}

cudaError_t readback_async(pct_ctx *ctx, void *hdst, const void *dsrc, size_t n) {
  return small_copy(ctx, hdst, dsrc, n);
}

namespace {
struct ResidentConst {
  std::vector<char> bytes;
  cudaEvent_t uploaded = nullptr;
  const pct_ctx *uploader = nullptr;
};
std::recursive_mutex g_const_mu;
std::map<void *, ResidentConst> g_const;     // symbol device address -> content
std::map<pct_ctx *, cudaEvent_t> g_const_users;  // last launch reading constants
}  // namespace

ConstBank::ConstBank(pct_ctx *ctx) : ctx_(ctx) { g_const_mu.lock(); }

ConstBank::~ConstBank() {
  cudaEvent_t &ev = g_const_users[ctx_];
  if (!ev) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (ev) cudaEventRecord(ev, ctx_->stream);
  g_const_mu.unlock();
}

cudaError_t ConstBank::set(void *addr, const void *src, size_t n) {
  ResidentConst &r = g_const[addr];
  if (r.bytes.size() == n && std::memcmp(r.bytes.data(), src, n) == 0) {
    if (r.uploaded && r.uploader != ctx_) return cudaStreamWaitEvent(ctx_->stream, r.uploaded, 0);
    return cudaSuccess;
  }
  for (auto &u : g_const_users)
    if (u.first != ctx_ && u.first->device == ctx_->device && u.second)
      if (cudaError_t e = cudaStreamWaitEvent(ctx_->stream, u.second, 0)) return e;
  if (cudaError_t e = cudaMemcpyAsync(addr, pin_upload(ctx_, src, n), n, cudaMemcpyHostToDevice,
                                      ctx_->stream))
    return e;
  if (!r.uploaded)
    if (cudaError_t e = cudaEventCreateWithFlags(&r.uploaded, cudaEventDisableTiming)) return e;
  if (cudaError_t e = cudaEventRecord(r.uploaded, ctx_->stream)) return e;
  r.uploader = ctx_;
  r.bytes.assign(static_cast<const char *>(src), static_cast<const char *>(src) + n);
  return cudaSuccess;
}

void const_bank_forget(pct_ctx *ctx) {
  std::lock_guard<std::recursive_mutex> lk(g_const_mu);
  auto it = g_const_users.find(ctx);
  if (it != g_const_users.end()) {
    if (it->second) cudaEventDestroy(it->second);
    g_const_users.erase(it);
  }
  for (auto &r : g_const)
    if (r.second.uploader == ctx) r.second.uploader = nullptr;
}

int ensure_scratch(pct_ctx *ctx, size_t bytes) {
  return ensure_buffer(ctx, &ctx->scratch, &ctx->scratch_bytes, bytes);
}
int ensure_staging(pct_ctx *ctx, size_t bytes) {
  return ensure_buffer(ctx, &ctx->staging, &ctx->staging_bytes, bytes);
}

int launch_slope(pct_ctx *, const float *, int, int, double, double *, double *, uint8_t *);
int launch_gentle_fraction(pct_ctx *, const uint8_t *, int, int, int, double *);
int launch_terrain_values(pct_ctx *, const double *, const double *, const double *, int64_t,
                          const pct_trav_params &, double *);
int launch_fuse(pct_ctx *, const float *, const float *, const uint8_t *, int64_t,
                const pct_trav_params &, float *);

static int check_params(pct_ctx *ctx, const pct_trav_params *p) {
  if (!p) return fail(ctx, PCT_E_INVALID, "params is NULL");
  if (!(0 < p->d_min && p->d_min <= p->d_ref)) return fail(ctx, PCT_E_INVALID, "need 0 < d_min <= d_ref");
  if (!(0 < p->theta_s && p->theta_s <= p->theta_b))
    return fail(ctx, PCT_E_INVALID, "need 0 < theta_s <= theta_b");
  if (!(0 <= p->theta_p && p->theta_p <= 1)) return fail(ctx, PCT_E_INVALID, "theta_p must lie in [0, 1]");
  if (p->c_barrier <= 0) return fail(ctx, PCT_E_INVALID, "c_barrier must be positive");
  if (p->patch_radius < 0) return fail(ctx, PCT_E_INVALID, "patch radius must be >= 0");
  return PCT_OK;
}

static int set_device(pct_ctx *ctx) {
  PCT_CUDA(ctx, cudaSetDevice(ctx->device));
  return PCT_OK;
}

}  // namespace pct

using namespace pct;

#define CTX_GUARD(ctx)                                           \
  do {                                                           \
    if (!(ctx)) return PCT_E_INVALID;                            \
    if (int rc_ = set_device(ctx)) return rc_;                   \
  } while (0)

extern "C" {

int pct_abi_version(void) { return PCT_ABI_VERSION; }

int pct_ctx_create(int device, pct_ctx **out) {
  if (!out) return PCT_E_INVALID;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    return PCT_E_CUDA;
  }
  if (device < 0 || device >= n) return PCT_E_INVALID;
  pct_ctx *ctx = new (std::nothrow) pct_ctx();
  if (!ctx) return PCT_E_NOMEM;
  ctx->device = device;
  int rc = PCT_OK;
  do {
    if ((rc = set_device(ctx))) break;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) { rc = PCT_E_CUDA; break; }
    if (prop.major < 10) {
      rc = fail(ctx, PCT_E_CUDA, "libpct requires an sm_100a (Blackwell) device");
      break;
    }
    ctx->num_sms = prop.multiProcessorCount;
    if (cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
      rc = PCT_E_CUDA;
      break;
    }
    ctx->stream = ctx->own_stream;
    // a memory pool per context: stacks freed on this context's stream are
    // re-used in stream order by its next map (no growth, no dependency on
    // another context's queue); freed memory stays cached in the pool
    {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = device;
      if (cudaMemPoolCreate(&ctx->mempool, &props) != cudaSuccess) { rc = PCT_E_CUDA; break; }
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(ctx->mempool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    if (cudaMalloc(&ctx->dsmall, 65536) != cudaSuccess) { rc = PCT_E_NOMEM; break; }
    if (cudaMallocHost(&ctx->hsmall, 65536) != cudaSuccess) { rc = PCT_E_NOMEM; break; }
    if (cudaMallocHost(&ctx->upload, kUploadRing) != cudaSuccess) { rc = PCT_E_NOMEM; break; }
  } while (0);
  if (rc) {
    pct_ctx_destroy(ctx);
    return rc;
  }
  *out = ctx;
  return PCT_OK;
}

int pct_ctx_destroy(pct_ctx *ctx) {
  if (!ctx) return PCT_OK;
  cudaSetDevice(ctx->device);
  if (ctx->own_stream) cudaStreamSynchronize(ctx->own_stream);
  const_bank_forget(ctx);
  if (ctx->scratch) cudaFree(ctx->scratch);
  if (ctx->staging) cudaFree(ctx->staging);
  if (ctx->dsmall) cudaFree(ctx->dsmall);
  if (ctx->enc) cudaFree(ctx->enc);
  if (ctx->keys) cudaFree(ctx->keys);
  if (ctx->spec_ev) cudaEventDestroy(ctx->spec_ev);
  if (ctx->switch_ev) cudaEventDestroy(ctx->switch_ev);
  for (auto &e : ctx->xfer_ev)
    if (e) cudaEventDestroy(e);
  for (auto e : ctx->ev)
    if (e) cudaEventDestroy(e);
  if (ctx->hsmall) cudaFreeHost(ctx->hsmall);
  if (ctx->pinned_io) cudaFreeHost(ctx->pinned_io);
  if (ctx->pinned_batch) cudaFreeHost(ctx->pinned_batch);
  if (ctx->upload) cudaFreeHost(ctx->upload);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  if (ctx->mempool) cudaMemPoolDestroy(ctx->mempool);  // deferred while blocks are live
  delete ctx;
  return PCT_OK;
}

const char *pct_last_error(const pct_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int pct_sync(pct_ctx *ctx) {
  CTX_GUARD(ctx);
  PCT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return PCT_OK;
}

int64_t pct_launch_count(const pct_ctx *ctx) { return ctx ? ctx->launches : 0; }

int pct_set_stream(pct_ctx *ctx, void *stream) {
  CTX_GUARD(ctx);
  cudaStream_t next = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  if (next == ctx->stream) return PCT_OK;
  // join: work already queued on the old stream (copies out of the pinned
  // upload ring, constant uploads, kernels writing buffers the caller reuses)
  // is ordered before everything issued on the new one
  if (!ctx->switch_ev)
    PCT_CUDA(ctx, cudaEventCreateWithFlags(&ctx->switch_ev, cudaEventDisableTiming));
  PCT_CUDA(ctx, cudaEventRecord(ctx->switch_ev, ctx->stream));
  PCT_CUDA(ctx, cudaStreamWaitEvent(next, ctx->switch_ev, 0));
  ctx->stream = next;
  return PCT_OK;
}

int pct_malloc(pct_ctx *ctx, size_t bytes, void **dptr) {
  CTX_GUARD(ctx);
  if (!dptr) return fail(ctx, PCT_E_INVALID, "dptr is NULL");
  *dptr = nullptr;
  if (bytes == 0) bytes = 1;
  PCT_CUDA(ctx, cudaMallocFromPoolAsync(dptr, bytes, ctx->mempool, ctx->stream));
  return PCT_OK;
}

int pct_free(pct_ctx *ctx, void *dptr) {
  CTX_GUARD(ctx);
  if (dptr) PCT_CUDA(ctx, cudaFreeAsync(dptr, ctx->stream));
  return PCT_OK;
}

int pct_host_alloc(pct_ctx *ctx, size_t bytes, void **hptr) {
  CTX_GUARD(ctx);
  if (!hptr) return fail(ctx, PCT_E_INVALID, "hptr is NULL");
  PCT_CUDA(ctx, cudaMallocHost(hptr, bytes ? bytes : 1));
  return PCT_OK;
}

int pct_host_free(pct_ctx *ctx, void *hptr) {
  CTX_GUARD(ctx);
  if (hptr) PCT_CUDA(ctx, cudaFreeHost(hptr));
  return PCT_OK;
}

int pct_host_register(pct_ctx *ctx, void *hptr, size_t bytes) {
  CTX_GUARD(ctx);
  if (!hptr || !bytes) return fail(ctx, PCT_E_INVALID, "bad arguments to pct_host_register");
  PCT_CUDA(ctx, cudaHostRegister(hptr, bytes, cudaHostRegisterPortable));
  return PCT_OK;
}

int pct_host_unregister(pct_ctx *ctx, void *hptr) {
  CTX_GUARD(ctx);
  if (hptr) PCT_CUDA(ctx, cudaHostUnregister(hptr));
  return PCT_OK;
}

int pct_memcpy_h2d(pct_ctx *ctx, void *dst, const void *src, size_t bytes) {
  CTX_GUARD(ctx);
  if (bytes) PCT_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return PCT_OK;
}

int pct_memcpy_d2h(pct_ctx *ctx, void *dst, const void *src, size_t bytes) {
  CTX_GUARD(ctx);
  if (bytes) PCT_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  PCT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return PCT_OK;
}

int pct_memcpy_d2h_async(pct_ctx *ctx, void *dst, const void *src, size_t bytes) {
  CTX_GUARD(ctx);
  if (bytes) PCT_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  return PCT_OK;
}

int pct_bounds(pct_ctx *ctx, const void *xyz, int64_t n, int dtype, double lo[3], double hi[3]) {
  CTX_GUARD(ctx);
  if (!xyz || !lo || !hi || (dtype != PCT_F32 && dtype != PCT_F64))
    return fail(ctx, PCT_E_INVALID, "bad arguments to pct_bounds");
  return launch_bounds(ctx, xyz, n, dtype, lo, hi);
}

int pct_frame_compute(const double lo[3], const double hi[3], double d_s, double r_g,
                      int64_t max_grid_side, pct_frame *fr, double *heights_out,
                      int32_t heights_cap) {
  if (!lo || !hi || !fr) return PCT_E_INVALID;
  if (!(d_s > 0) || !(r_g > 0)) return PCT_E_INVALID;  // "d_s and r_g must be positive"
  // tomogram.py:138-145, evaluated in IEEE double without contraction
  volatile double dy = hi[1] - lo[1], dx = hi[0] - lo[0], dz = hi[2] - lo[2];
  volatile double qy = dy / r_g, qx = dx / r_g, qz = dz / d_s;
  const double rows_d = std::floor(qy + 0.5) + 2.0;
  const double cols_d = std::floor(qx + 0.5) + 2.0;
  double s = std::ceil(qz - 1e-9);
  if (s < 1) s = 1;
  fr->origin_x = lo[0];
  fr->origin_y = lo[1];
  fr->z_min = lo[2];
  fr->d_s = d_s;
  fr->r_g = r_g;
  if (rows_d > (double)max_grid_side || cols_d > (double)max_grid_side) {
    fr->rows = rows_d > 2147483647.0 ? -1 : (int32_t)rows_d;
    fr->cols = cols_d > 2147483647.0 ? -1 : (int32_t)cols_d;
    fr->n_slices = 0;
    return PCT_E_GRID;
  }
  if (s > 1e8) return PCT_E_INVALID;
  fr->rows = (int32_t)rows_d;
  fr->cols = (int32_t)cols_d;
  fr->n_slices = (int32_t)s;
  if (heights_out) {
    if (heights_cap < fr->n_slices) return PCT_E_INVALID;
    for (int k = 0; k < fr->n_slices; ++k) {
      volatile double t = d_s * ((double)k + 1.0);
      heights_out[k] = lo[2] + t;
    }
  }
  return PCT_OK;
}

int pct_build(pct_ctx *ctx, const void *xyz, int64_t n, int dtype, const pct_frame *fr,
              const double *heights, float *ground, float *ceiling) {
  CTX_GUARD(ctx);
  if (!fr || !heights || !ground || !ceiling || (n > 0 && !xyz) ||
      (dtype != PCT_F32 && dtype != PCT_F64) || fr->rows <= 0 || fr->cols <= 0 ||
      fr->n_slices <= 0)
    return fail(ctx, PCT_E_INVALID, "bad arguments to pct_build");
  return launch_build(ctx, xyz, n, dtype, *fr, heights, ground, ceiling);
}

int pct_evaluate(pct_ctx *ctx, const float *ground, const float *ceiling, int32_t n_slices,
                 int32_t rows, int32_t cols, double r_g, const pct_trav_params *p,
                 const float *kernel_w, int32_t kside, float *cost) {
  CTX_GUARD(ctx);
  if (int rc = check_params(ctx, p)) return rc;
  if (!ground || !ceiling || !cost || !kernel_w || !(r_g > 0) || n_slices > 65535)
    return fail(ctx, PCT_E_INVALID, "bad arguments to pct_evaluate");
  return launch_evaluate(ctx, ground, ceiling, n_slices, rows, cols, r_g, *p, kernel_w, kside,
                         cost, kEvalFull);
}

int pct_evaluate_masked(pct_ctx *ctx, const float *ground, const float *ceiling, int32_t n_slices,
                        int32_t rows, int32_t cols, double r_g, const pct_trav_params *p,
                        const float *kernel_w, int32_t kside, const uint64_t *masks,
                        float *cost) {
  CTX_GUARD(ctx);
  ctx->eval_masks = n_slices <= 64 ? reinterpret_cast<const unsigned long long *>(masks) : nullptr;
  const int rc = pct_evaluate(ctx, ground, ceiling, n_slices, rows, cols, r_g, p, kernel_w, kside,
                              cost);
  ctx->eval_masks = nullptr;
  return rc;
}

int64_t pct_tile_masks_bytes(int32_t rows, int32_t cols) {
  if (rows <= 0 || cols <= 0) return 0;
  return (int64_t)((rows + 15) / 16) * ((cols + 31) / 32) * 8;  // tiles >= 16 x 32
}

int pct_evaluate_tiles(pct_ctx *ctx, const float *ground, const float *ceiling, int32_t n_slices,
                       int32_t rows, int32_t cols, double r_g, const pct_trav_params *p,
                       const float *kernel_w, int32_t kside, const uint64_t *masks, float *cost,
                       uint64_t *tile_masks, int32_t *tile_geom) {
  CTX_GUARD(ctx);
  if (tile_geom) tile_geom[0] = tile_geom[1] = 0;
  ctx->eval_masks = n_slices <= 64 ? reinterpret_cast<const unsigned long long *>(masks) : nullptr;
  ctx->eval_tcm = (ctx->eval_masks && tile_masks && tile_geom)
                      ? reinterpret_cast<unsigned long long *>(tile_masks)
                      : nullptr;
  ctx->eval_tcm_written = false;
  const int rc = pct_evaluate(ctx, ground, ceiling, n_slices, rows, cols, r_g, p, kernel_w, kside,
                              cost);
  if (rc == PCT_OK && ctx->eval_tcm && ctx->eval_tcm_written) {
    tile_geom[0] = ctx->tcm_th;
    tile_geom[1] = ctx->tcm_tw;
  }
  ctx->eval_masks = nullptr;
  ctx->eval_tcm = nullptr;
  return rc;
}

int pct_simplify_masked(pct_ctx *ctx, const float *ground, const float *cost, int32_t n_slices,
                        int32_t rows, int32_t cols, double eps_e, double c_barrier,
                        const uint64_t *masks, const uint64_t *tile_masks,
                        const int32_t *tile_geom, int32_t *keep_host, int32_t *n_keep) {
  CTX_GUARD(ctx);
  if (masks && tile_masks && tile_geom && tile_geom[0] > 0 && tile_geom[1] > 0) {
    ctx->simp_gm = reinterpret_cast<const unsigned long long *>(masks);
    ctx->simp_tcm = reinterpret_cast<const unsigned long long *>(tile_masks);
    ctx->simp_th = tile_geom[0];
    ctx->simp_tw = tile_geom[1];
  }
  const int rc = pct_simplify(ctx, ground, cost, n_slices, rows, cols, eps_e, c_barrier, keep_host,
                              n_keep);
  ctx->simp_gm = ctx->simp_tcm = nullptr;
  return rc;
}

const uint64_t *pct_tomo_masks(const pct_tomo *t) {
  return t ? reinterpret_cast<const uint64_t *>(t->masks) : nullptr;
}

int pct_interval_cost(pct_ctx *ctx, const float *ground, const float *ceiling, int32_t rows,
                      int32_t cols, const pct_trav_params *p, float *out) {
  CTX_GUARD(ctx);
  if (int rc = check_params(ctx, p)) return rc;
  pct_trav_params q = *p;
  q.patch_radius = 0;
  return launch_evaluate(ctx, ground, ceiling, 1, rows, cols, 1.0, q, nullptr, 0, out,
                         kEvalInterval);
}

int pct_ground_cost(pct_ctx *ctx, const float *ground, int32_t rows, int32_t cols, double r_g,
                    const pct_trav_params *p, float *out) {
  CTX_GUARD(ctx);
  if (int rc = check_params(ctx, p)) return rc;
  if (!(r_g > 0)) return fail(ctx, PCT_E_INVALID, "resolution must be positive");
  return launch_evaluate(ctx, ground, nullptr, 1, rows, cols, r_g, *p, nullptr, 0, out,
                         kEvalGroundCost);
}

int pct_slope_magnitudes(pct_ctx *ctx, const float *ground, int32_t rows, int32_t cols,
                         double r_g, double *m_xy, double *m_grad, uint8_t *isolated) {
  CTX_GUARD(ctx);
  return launch_slope(ctx, ground, rows, cols, r_g, m_xy, m_grad, isolated);
}

int pct_fuse_costs(pct_ctx *ctx, const float *c_interval, const float *c_ground,
                   const uint8_t *ground_valid, int32_t rows, int32_t cols,
                   const pct_trav_params *p, float *out) {
  CTX_GUARD(ctx);
  if (!p) return fail(ctx, PCT_E_INVALID, "params is NULL");
  return launch_fuse(ctx, c_interval, c_ground, ground_valid, (int64_t)rows * cols, *p, out);
}

int pct_inflate(pct_ctx *ctx, const float *cost, int32_t rows, int32_t cols,
                const float *kernel_w, int32_t kside, float *out) {
  CTX_GUARD(ctx);
  if (!cost || !out || !kernel_w) return fail(ctx, PCT_E_INVALID, "bad arguments to pct_inflate");
  return launch_inflate(ctx, cost, rows, cols, kernel_w, kside, out);
}

int pct_gentle_fraction(pct_ctx *ctx, const uint8_t *gentle, int32_t rows, int32_t cols,
                        int32_t radius, double *out) {
  CTX_GUARD(ctx);
  if (radius < 0) return fail(ctx, PCT_E_INVALID, "radius must be >= 0");
  return launch_gentle_fraction(ctx, gentle, rows, cols, radius, out);
}

int pct_terrain_cost_values(pct_ctx *ctx, const double *m_xy, const double *m_grad,
                            const double *p_s, int64_t n, const pct_trav_params *p, double *out) {
  CTX_GUARD(ctx);
  if (!p) return fail(ctx, PCT_E_INVALID, "params is NULL");
  return launch_terrain_values(ctx, m_xy, m_grad, p_s, n, *p, out);
}

int pct_simplify(pct_ctx *ctx, const float *ground, const float *cost, int32_t n_slices,
                 int32_t rows, int32_t cols, double eps_e, double c_barrier, int32_t *keep_host,
                 int32_t *n_keep) {
  CTX_GUARD(ctx);
  if (!ground || !cost || !keep_host || !n_keep || n_slices < 0)
    return fail(ctx, PCT_E_INVALID, "bad arguments to pct_simplify");
  std::vector<int> keep;
  if (int rc = run_simplify(ctx, ground, cost, n_slices, rows, cols, eps_e, c_barrier, keep))
    return rc;
  for (size_t i = 0; i < keep.size(); ++i) keep_host[i] = keep[i];
  *n_keep = (int32_t)keep.size();
  return PCT_OK;
}

int pct_unique_mask(pct_ctx *ctx, const float *ground, const float *cost, int32_t rows,
                    int32_t cols, int32_t k, int32_t below, int32_t above, double eps_e,
                    double c_barrier, uint8_t *mask) {
  CTX_GUARD(ctx);
  if (!ground || !cost || !mask) return fail(ctx, PCT_E_INVALID, "bad arguments to pct_unique_mask");
  return launch_unique_mask(ctx, ground, cost, rows, cols, k, below, above, eps_e, c_barrier,
                            mask);
}

// ------------------------------------------------------- device tomogram
int tomo_alloc(pct_ctx *ctx, const pct_frame &fr, pct_tomo **out) {
  pct_tomo *t = new (std::nothrow) pct_tomo();
  if (!t) return fail(ctx, PCT_E_NOMEM, "out of host memory");
  t->fr = fr;
  const size_t bytes = (size_t)fr.n_slices * fr.rows * fr.cols * sizeof(float);
  cudaError_t e = cudaMallocFromPoolAsync(reinterpret_cast<void **>(&t->ground), bytes, ctx->mempool, ctx->stream);
  if (e == cudaSuccess)
    e = cudaMallocFromPoolAsync(reinterpret_cast<void **>(&t->ceiling), bytes, ctx->mempool, ctx->stream);
  if (e != cudaSuccess) {
    pct_tomo_free(ctx, t);
    return cuda_fail(ctx, e, "cudaMallocAsync(tomogram)");
  }

  *out = t;
  return PCT_OK;
}

int pct_tomo_build(pct_ctx *ctx, const void *xyz, int64_t n, int dtype, int xyz_on_host,
                   double d_s, double r_g, int64_t max_grid_side, pct_tomo **out) {
  CTX_GUARD(ctx);
  if (!out) return fail(ctx, PCT_E_INVALID, "out is NULL");
  *out = nullptr;
  if (!(d_s > 0) || !(r_g > 0)) return fail(ctx, PCT_E_INVALID, "d_s and r_g must be positive");
  if (n <= 0) return fail(ctx, PCT_E_EMPTY, "zero valid points");
  if (!xyz || (dtype != PCT_F32 && dtype != PCT_F64))
    return fail(ctx, PCT_E_INVALID, "bad arguments to pct_tomo_build");
  const void *dxyz = xyz;
  if (xyz_on_host) {
    const size_t bytes = (size_t)n * 3 * (dtype == PCT_F32 ? 4 : 8);
    if (int rc = ensure_staging(ctx, bytes)) return rc;
    PCT_CUDA(ctx, cudaMemcpyAsync(ctx->staging, xyz, bytes, cudaMemcpyHostToDevice, ctx->stream));
    dxyz = ctx->staging;
  }
  double lo[3], hi[3];
  pct_frame dfr{};
  bool scattered = false;
  if (int rc = launch_bounds_spec(ctx, dxyz, n, dtype, d_s, r_g, max_grid_side, lo, hi, &dfr,
                                  &scattered))
    return rc;
  pct_frame fr;
  int rc = pct_frame_compute(lo, hi, d_s, r_g, max_grid_side, &fr, nullptr, 0);
  // the device derived the frame the same way; should it ever differ, its
  // keys are dropped (the key buffer is not clean, so the build below clears
  // it and scatters again)
  if (scattered && (rc || dfr.rows != fr.rows || dfr.cols != fr.cols ||
                    dfr.n_slices != fr.n_slices || dfr.origin_x != fr.origin_x ||
                    dfr.origin_y != fr.origin_y || dfr.z_min != fr.z_min))
    scattered = false;
  if (rc == PCT_E_GRID)
    return fail(ctx, PCT_E_GRID, "grid " + std::to_string(fr.rows) + "x" + std::to_string(fr.cols) +
                                     " exceeds the " + std::to_string(max_grid_side) +
                                     " per-side limit");
  if (rc) return fail(ctx, rc, "invalid grid frame");
  pct_tomo *t = nullptr;
  if ((rc = tomo_alloc(ctx, fr, &t))) return rc;
  t->heights.resize(fr.n_slices);
  pct_frame_compute(lo, hi, d_s, r_g, max_grid_side, &fr, t->heights.data(), fr.n_slices);
  if (fr.n_slices <= 64) {  // slice-change masks for the evaluation (16 B per cell)
    const size_t mb = 2 * (size_t)fr.rows * fr.cols * sizeof(unsigned long long);
    if (cudaMallocFromPoolAsync(reinterpret_cast<void **>(&t->masks), mb, ctx->mempool,
                                ctx->stream) != cudaSuccess) {
      cudaGetLastError();
      t->masks = nullptr;  // optional: the walk derives them
    }
  }
  ctx->build_masks = t->masks;
  ctx->build_masks_written = false;
  rc = launch_build(ctx, dxyz, n, dtype, fr, t->heights.data(), t->ground, t->ceiling, 0, -1, 0,
                    scattered);
  ctx->build_masks = nullptr;
  if (t->masks && !ctx->build_masks_written) {  // a build path that does not emit them
    cudaFreeAsync(t->masks, ctx->stream);
    t->masks = nullptr;
  }
  if (rc) {
    pct_tomo_free(ctx, t);
    return rc;
  }
  *out = t;
  return PCT_OK;
}

int pct_tomo_upload(pct_ctx *ctx, const pct_frame *fr, const double *heights,
                    const float *ground_host, const float *ceiling_host, pct_tomo **out) {
  CTX_GUARD(ctx);
  if (!fr || !heights || !ground_host || !ceiling_host || !out || fr->rows <= 0 || fr->cols <= 0 ||
      fr->n_slices <= 0)
    return fail(ctx, PCT_E_INVALID, "bad arguments to pct_tomo_upload");
  pct_tomo *t = nullptr;
  if (int rc = tomo_alloc(ctx, *fr, &t)) return rc;
  t->heights.assign(heights, heights + fr->n_slices);
  const size_t bytes = (size_t)fr->n_slices * fr->rows * fr->cols * sizeof(float);
  cudaError_t e = cudaMemcpyAsync(t->ground, ground_host, bytes, cudaMemcpyHostToDevice, ctx->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(t->ceiling, ceiling_host, bytes, cudaMemcpyHostToDevice, ctx->stream);
  if (e != cudaSuccess) {
    pct_tomo_free(ctx, t);
    return cuda_fail(ctx, e, "cudaMemcpyAsync(upload)");
  }
  *out = t;
  return PCT_OK;
}

int pct_tomo_evaluate(pct_ctx *ctx, pct_tomo *t, const pct_trav_params *p, const float *kernel_w,
                      int32_t kside) {
  CTX_GUARD(ctx);
  if (!t) return fail(ctx, PCT_E_INVALID, "tomogram is NULL");
  if (int rc = check_params(ctx, p)) return rc;
  const size_t bytes = (size_t)t->fr.n_slices * t->fr.rows * t->fr.cols * sizeof(float);
  if (!t->cost) PCT_CUDA(ctx, cudaMallocFromPoolAsync(reinterpret_cast<void **>(&t->cost), bytes, ctx->mempool, ctx->stream));
  ctx->eval_masks = t->masks;  // written by this tomogram's build (NULL: derived again)
  // per-tile cost-change masks for the simplify window (room for tiles of
  // >= 16 rows x 32 columns)
  if (t->masks && t->fr.n_slices <= 64 && !t->tcm) {
    const size_t tb = (size_t)((t->fr.rows + 15) / 16) * ((t->fr.cols + 31) / 32) * 8;
    if (cudaMallocFromPoolAsync(reinterpret_cast<void **>(&t->tcm), tb, ctx->mempool,
                                ctx->stream) != cudaSuccess) {
      cudaGetLastError();
      t->tcm = nullptr;
    }
  }
  ctx->eval_tcm = t->tcm;
  ctx->eval_tcm_written = false;
  const int rc = launch_evaluate(ctx, t->ground, t->ceiling, t->fr.n_slices, t->fr.rows,
                                 t->fr.cols, t->fr.r_g, *p, kernel_w, kside, t->cost, kEvalFull);
  ctx->eval_masks = nullptr;
  ctx->eval_tcm = nullptr;
  if (t->tcm && !ctx->eval_tcm_written) {  // an evaluation path that does not record them
    cudaFreeAsync(t->tcm, ctx->stream);
    t->tcm = nullptr;
  } else if (t->tcm) {
    t->tcm_th = ctx->tcm_th;
    t->tcm_tw = ctx->tcm_tw;
  }
  return rc;
}

int pct_tomo_simplify(pct_ctx *ctx, pct_tomo *t, double eps_e, double c_barrier,
                      int32_t *keep_host, int32_t *n_keep) {
  CTX_GUARD(ctx);
  if (!t) return fail(ctx, PCT_E_INVALID, "tomogram is NULL");
  if (!t->cost) return fail(ctx, PCT_E_NOCOST, "slice has no cost layer; evaluate the tomogram first");
  if (t->masks && t->tcm) {  // slice-change information of its build and evaluation
    ctx->simp_gm = t->masks;
    ctx->simp_tcm = t->tcm;
    ctx->simp_th = t->tcm_th;
    ctx->simp_tw = t->tcm_tw;
  }
  const int rc = pct_simplify(ctx, t->ground, t->cost, t->fr.n_slices, t->fr.rows, t->fr.cols,
                              eps_e, c_barrier, keep_host, n_keep);
  ctx->simp_gm = ctx->simp_tcm = nullptr;
  return rc;
}

int pct_tomo_run(pct_ctx *ctx, const void *xyz, int64_t n, int dtype, int xyz_on_host,
                 double d_s, double r_g, int64_t max_grid_side, const pct_trav_params *p,
                 const float *kernel_w, int32_t kside, double eps_e, double c_barrier,
                 pct_tomo **out, int32_t *keep_host, int32_t *n_keep) {
  CTX_GUARD(ctx);
  if (!out || !keep_host || !n_keep) return fail(ctx, PCT_E_INVALID, "bad arguments to pct_tomo_run");
  pct_tomo *t = nullptr;
  if (ctx->timing) cudaEventRecord(ctx->ev[0], ctx->stream);
  int rc = pct_tomo_build(ctx, xyz, n, dtype, xyz_on_host, d_s, r_g, max_grid_side, &t);
  if (rc) return rc;
  if (ctx->timing) cudaEventRecord(ctx->ev[1], ctx->stream);
  if ((rc = pct_tomo_evaluate(ctx, t, p, kernel_w, kside))) {
    pct_tomo_free(ctx, t);
    return rc;
  }
  if (ctx->timing) cudaEventRecord(ctx->ev[2], ctx->stream);
  if ((rc = pct_tomo_simplify(ctx, t, eps_e, c_barrier, keep_host, n_keep))) {
    pct_tomo_free(ctx, t);
    return rc;
  }
  if (ctx->timing) cudaEventRecord(ctx->ev[3], ctx->stream);
  *out = t;
  return PCT_OK;
}

int pct_set_timing(pct_ctx *ctx, int on) {
  CTX_GUARD(ctx);
  if (on && !ctx->ev[0])
    for (auto &e : ctx->ev) PCT_CUDA(ctx, cudaEventCreate(&e));
  ctx->timing = on != 0;
  return PCT_OK;
}

int pct_last_stage_ms(pct_ctx *ctx, float ms[3]) {
  CTX_GUARD(ctx);
  if (!ctx->timing || !ms) return fail(ctx, PCT_E_INVALID, "timing is off");
  PCT_CUDA(ctx, cudaEventSynchronize(ctx->ev[3]));
  for (int s = 0; s < 3; ++s) PCT_CUDA(ctx, cudaEventElapsedTime(ms + s, ctx->ev[s], ctx->ev[s + 1]));
  return PCT_OK;
}

int pct_tomo_frame(const pct_tomo *t, pct_frame *fr, double *heights, int32_t heights_cap) {
  if (!t || !fr) return PCT_E_INVALID;
  *fr = t->fr;
  if (heights) {
    if (heights_cap < t->fr.n_slices) return PCT_E_INVALID;
    std::memcpy(heights, t->heights.data(), sizeof(double) * t->fr.n_slices);
  }
  return PCT_OK;
}

const float *pct_tomo_layer(const pct_tomo *t, int layer) {
  if (!t) return nullptr;
  return layer == PCT_LAYER_GROUND ? t->ground
                                   : layer == PCT_LAYER_CEILING ? t->ceiling
                                                                : layer == PCT_LAYER_COST ? t->cost
                                                                                          : nullptr;
}

int pct_tomo_download(pct_ctx *ctx, const pct_tomo *t, int layer, int32_t k, float *host) {
  CTX_GUARD(ctx);
  const float *src = pct_tomo_layer(t, layer);
  if (!src || !host) return fail(ctx, PCT_E_INVALID, "layer not available");
  if (k >= t->fr.n_slices) return fail(ctx, PCT_E_RANGE, "slice index out of range");
  const size_t plane = (size_t)t->fr.rows * t->fr.cols;
  const size_t off = k < 0 ? 0 : plane * k;
  const size_t cnt = k < 0 ? plane * t->fr.n_slices : plane;
  PCT_CUDA(ctx, cudaMemcpyAsync(host, src + off, cnt * sizeof(float), cudaMemcpyDeviceToHost,
                                ctx->stream));
  PCT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return PCT_OK;
}

int pct_tomo_free(pct_ctx *ctx, pct_tomo *t) {
  if (!t) return PCT_OK;
  if (ctx) cudaSetDevice(ctx->device);
  cudaStream_t s = ctx ? ctx->stream : nullptr;
  if (t->ground) cudaFreeAsync(t->ground, s);
  if (t->ceiling) cudaFreeAsync(t->ceiling, s);
  if (t->cost) cudaFreeAsync(t->cost, s);
  if (t->masks) cudaFreeAsync(t->masks, s);
  if (t->tcm) cudaFreeAsync(t->tcm, s);
  delete t;
  return PCT_OK;
}

}  // extern "C"
