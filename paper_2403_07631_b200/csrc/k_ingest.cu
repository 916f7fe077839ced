// k_ingest.cu — binary PCD ingest (SURVEY.md §8 f rank 3; replaces the
// payload half of cloud_io.py:123-146 + _keep_finite :53-55).
//
// The reference reads the whole payload into a bytes object, views it as a
// numpy record array, stacks x/y/z and up-casts to float64, then drops rows
// with a non-finite coordinate.  Here the payload goes file -> pinned host
// chunks (parallel pread, native threads) -> HBM (async DMA, overlapping the
// next chunk's read) and two kernels per chunk gather the float32 x/y/z of
// every record and compact the finite rows, in record order, into a dense
// (N, 3) float32 point array that the build consumes in place.  float32 ->
// float64 is exact, so the points equal the reference's PointCloud.xyz.
//
//   count_kernel   one bit per record (finite x, y, z), popcount per 1024
//                  records -> tile counts
//   offsets_kernel exclusive scan of the tile counts (one CTA), based at the
//                  running device total of earlier chunks
//   write_kernel   re-derives the bits, warp ballots + tile offsets give each
//                  survivor its output row; x/y/z stored contiguously
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "pct_internal.h"

namespace pct {
namespace {

constexpr int kIngNT = 256;                  // threads per CTA
constexpr int kIngPer = 4;                   // records per thread
constexpr int kIngTile = kIngNT * kIngPer;   // records per tile (one CTA)
constexpr int kIngWarpRecs = 32 * kIngPer;   // consecutive records per warp

struct RecLayout {
  int64_t stride;      // bytes per record
  int64_t off[3];      // byte offsets of x, y, z
  bool aligned;        // stride and offsets multiples of 4
};

__device__ __forceinline__ float load_f32(const unsigned char *p, bool aligned) {
  if (aligned) return __ldg(reinterpret_cast<const float *>(p));
  // little-endian bytes (PCD binary is "<f4", the device is little-endian)
  const uint32_t u = (uint32_t)__ldg(p) | ((uint32_t)__ldg(p + 1) << 8) |
                     ((uint32_t)__ldg(p + 2) << 16) | ((uint32_t)__ldg(p + 3) << 24);
  return __uint_as_float(u);
}

__device__ __forceinline__ bool finite_f32(float v) {
  return (__float_as_uint(v) & 0x7F800000u) != 0x7F800000u;
}

// record r of the tile handled by (warp, lane, item q): warps own 128
// consecutive records, lanes interleave inside them (coalesced loads)
__device__ __forceinline__ int64_t rec_index(int64_t tile0, int warp, int q, int lane) {
  return tile0 + (int64_t)warp * kIngWarpRecs + q * 32 + lane;
}

__global__ void __launch_bounds__(kIngNT) count_kernel(const unsigned char *__restrict__ rec,
                                                       int64_t n, RecLayout L,
                                                       uint32_t *__restrict__ tile_counts) {
  __shared__ uint32_t wsum[kIngNT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t tile0 = (int64_t)blockIdx.x * kIngTile;
  uint32_t cnt = 0;
#pragma unroll
  for (int q = 0; q < kIngPer; ++q) {
    const int64_t r = rec_index(tile0, warp, q, lane);
    bool ok = false;
    if (r < n) {
      const unsigned char *p = rec + r * L.stride;
      ok = finite_f32(load_f32(p + L.off[0], L.aligned)) &&
           finite_f32(load_f32(p + L.off[1], L.aligned)) &&
           finite_f32(load_f32(p + L.off[2], L.aligned));
    }
    cnt += __popc(__ballot_sync(0xFFFFFFFFu, ok));
  }
  if (lane == 0) wsum[warp] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
#pragma unroll
    for (int w = 0; w < kIngNT / 32; ++w) t += wsum[w];
    tile_counts[blockIdx.x] = t;
  }
}

// exclusive scan of tile counts into tile offsets (int64), starting at
// *total; *total is advanced by the chunk's survivors.  One CTA of 1024.
__global__ void __launch_bounds__(1024) offsets_kernel(const uint32_t *__restrict__ tile_counts,
                                                       int64_t tiles,
                                                       int64_t *__restrict__ tile_offsets,
                                                       unsigned long long *total) {
  __shared__ unsigned long long wsum[32];
  __shared__ unsigned long long carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = *total;
  __syncthreads();
  for (int64_t base = 0; base < tiles; base += 1024) {
    const int64_t t = base + threadIdx.x;
    const unsigned long long v = t < tiles ? tile_counts[t] : 0ull;
    unsigned long long x = v;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      unsigned long long s = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, s, o);
        if (lane >= o) s += y;
      }
      wsum[lane] = s;  // inclusive over warps
    }
    __syncthreads();
    const unsigned long long before = (warp ? wsum[warp - 1] : 0ull) + x - v;
    if (t < tiles) tile_offsets[t] = (int64_t)(carry + before);
    __syncthreads();
    if (threadIdx.x == 0) carry += wsum[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(kIngNT) write_kernel(const unsigned char *__restrict__ rec,
                                                       int64_t n, RecLayout L,
                                                       const int64_t *__restrict__ tile_offsets,
                                                       float *__restrict__ out) {
  __shared__ uint32_t wsum[kIngNT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t tile0 = (int64_t)blockIdx.x * kIngTile;
  float v[kIngPer][3];
  uint32_t ball[kIngPer];
  uint32_t cnt = 0;
#pragma unroll
  for (int q = 0; q < kIngPer; ++q) {
    const int64_t r = rec_index(tile0, warp, q, lane);
    bool ok = false;
    if (r < n) {
      const unsigned char *p = rec + r * L.stride;
      v[q][0] = load_f32(p + L.off[0], L.aligned);
      v[q][1] = load_f32(p + L.off[1], L.aligned);
      v[q][2] = load_f32(p + L.off[2], L.aligned);
      ok = finite_f32(v[q][0]) && finite_f32(v[q][1]) && finite_f32(v[q][2]);
    }
    ball[q] = __ballot_sync(0xFFFFFFFFu, ok);
    cnt += __popc(ball[q]);
  }
  if (lane == 0) wsum[warp] = cnt;
  __syncthreads();
  int64_t pos = tile_offsets[blockIdx.x];
  for (int w = 0; w < warp; ++w) pos += wsum[w];
  const uint32_t below = (1u << lane) - 1u;
#pragma unroll
  for (int q = 0; q < kIngPer; ++q) {
    if (ball[q] >> lane & 1u) {
      float *o = out + 3 * (pos + __popc(ball[q] & below));
      o[0] = v[q][0];
      o[1] = v[q][1];
      o[2] = v[q][2];
    }
    pos += __popc(ball[q]);
  }
}

// count + offsets + write for one chunk of records resident on the device;
// tile scratch: counts (u32) then offsets (i64)
int launch_extract(pct_ctx *ctx, const unsigned char *rec, int64_t n, const RecLayout &L,
                   uint32_t *tile_counts, int64_t *tile_offsets, unsigned long long *total,
                   float *out) {
  if (n <= 0) return PCT_OK;
  const int64_t tiles = (n + kIngTile - 1) / kIngTile;
  count_kernel<<<(unsigned)tiles, kIngNT, 0, ctx->stream>>>(rec, n, L, tile_counts);
  offsets_kernel<<<1, 1024, 0, ctx->stream>>>(tile_counts, tiles, tile_offsets, total);
  write_kernel<<<(unsigned)tiles, kIngNT, 0, ctx->stream>>>(rec, n, L, tile_offsets, out);
  ctx->launches += 3;
  return check_launch(ctx, "pcd extract kernels");
}

int check_layout(pct_ctx *ctx, int64_t n, int64_t stride, const int64_t off[3], RecLayout &L) {
  if (n < 0 || stride <= 0) return fail(ctx, PCT_E_INVALID, "bad PCD record count / size");
  for (int c = 0; c < 3; ++c) {
    if (off[c] < 0 || off[c] + 4 > stride)
      return fail(ctx, PCT_E_INVALID, "PCD x/y/z offset outside the record");
    L.off[c] = off[c];
  }
  L.stride = stride;
  L.aligned = stride % 4 == 0 && off[0] % 4 == 0 && off[1] % 4 == 0 && off[2] % 4 == 0;
  return PCT_OK;
}

// tile scratch for up to `recs` records per chunk + the running total
int tile_scratch(pct_ctx *ctx, int64_t recs, uint32_t *&counts, int64_t *&offsets,
                 unsigned long long *&total) {
  const int64_t tiles = (recs + kIngTile - 1) / kIngTile + 1;
  const size_t bytes = 64 + (size_t)tiles * 4 + 16 + (size_t)tiles * 8;
  if (int rc = ensure_scratch(ctx, bytes)) return rc;
  unsigned char *s = static_cast<unsigned char *>(ctx->scratch);
  total = reinterpret_cast<unsigned long long *>(s);
  counts = reinterpret_cast<uint32_t *>(s + 64);
  offsets = reinterpret_cast<int64_t *>(s + 64 + ((tiles * 4 + 15) / 16) * 16 + 16);
  PCT_CUDA(ctx, cudaMemsetAsync(total, 0, 8, ctx->stream));
  return PCT_OK;
}

int read_total(pct_ctx *ctx, const unsigned long long *total, int64_t *n_valid) {
  unsigned long long *h = static_cast<unsigned long long *>(ctx->hsmall);
  PCT_CUDA(ctx, cudaMemcpyAsync(h, total, 8, cudaMemcpyDeviceToHost, ctx->stream));
  PCT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  *n_valid = (int64_t)h[0];
  return PCT_OK;
}

// pread [off, off+bytes) into dst with up to `threads` native threads
bool pread_all(int fd, unsigned char *dst, int64_t off, int64_t bytes, int threads) {
  const int64_t min_part = 8ll << 20;
  int parts = (int)std::max<int64_t>(1, std::min<int64_t>(threads, bytes / min_part));
  std::vector<char> ok(parts, 0);
  auto work = [&](int p) {
    const int64_t a = bytes * p / parts, b = bytes * (p + 1) / parts;
    int64_t done = a;
    while (done < b) {
      const ssize_t r = pread(fd, dst + done, (size_t)(b - done), (off_t)(off + done));
      if (r < 0 && errno == EINTR) continue;
      if (r <= 0) return;
      done += r;
    }
    ok[p] = 1;
  };
  if (parts == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (int p = 0; p < parts; ++p) th.emplace_back(work, p);
    for (auto &t : th) t.join();
  }
  for (char c : ok)
    if (!c) return false;
  return true;
}

}  // namespace
}  // namespace pct

using namespace pct;

extern "C" {

int pct_pcd_extract(pct_ctx *ctx, const void *records, int64_t n_records, int64_t record_bytes,
                    const int64_t xyz_offsets[3], int records_on_host, float *xyz_out,
                    int64_t *n_valid) {
  if (!ctx) return PCT_E_INVALID;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return PCT_E_CUDA;
  if (!xyz_offsets || !n_valid || (n_records > 0 && (!records || !xyz_out)))
    return fail(ctx, PCT_E_INVALID, "bad arguments to pct_pcd_extract");
  RecLayout L;
  if (int rc = check_layout(ctx, n_records, record_bytes, xyz_offsets, L)) return rc;
  *n_valid = 0;
  if (n_records == 0) return PCT_OK;
  const unsigned char *rec = static_cast<const unsigned char *>(records);
  if (records_on_host) {
    const size_t bytes = (size_t)(n_records * record_bytes);
    if (int rc = ensure_staging(ctx, bytes)) return rc;
    PCT_CUDA(ctx, cudaMemcpyAsync(ctx->staging, records, bytes, cudaMemcpyHostToDevice,
                                  ctx->stream));
    rec = static_cast<const unsigned char *>(ctx->staging);
  }
  uint32_t *counts;
  int64_t *offsets;
  unsigned long long *total;
  if (int rc = tile_scratch(ctx, n_records, counts, offsets, total)) return rc;
  if (int rc = launch_extract(ctx, rec, n_records, L, counts, offsets, total, xyz_out)) return rc;
  return read_total(ctx, total, n_valid);
}

int pct_pcd_load(pct_ctx *ctx, const char *path, int64_t data_offset, int64_t n_records,
                 int64_t record_bytes, const int64_t xyz_offsets[3], int64_t chunk_bytes,
                 float *xyz_out, int64_t *n_valid) {
  if (!ctx) return PCT_E_INVALID;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return PCT_E_CUDA;
  if (!path || !xyz_offsets || !n_valid || data_offset < 0 || (n_records > 0 && !xyz_out))
    return fail(ctx, PCT_E_INVALID, "bad arguments to pct_pcd_load");
  RecLayout L;
  if (int rc = check_layout(ctx, n_records, record_bytes, xyz_offsets, L)) return rc;
  *n_valid = 0;
  const int fd = open(path, O_RDONLY);
  if (fd < 0) return fail(ctx, PCT_E_IO, std::string(path) + ": " + std::strerror(errno));
  struct FdGuard {
    int fd;
    ~FdGuard() { close(fd); }
  } guard{fd};
  struct stat st;
  if (fstat(fd, &st) != 0) return fail(ctx, PCT_E_IO, std::string(path) + ": fstat failed");
  const int64_t need = n_records * record_bytes;
  if ((int64_t)st.st_size - data_offset < need)
    return fail(ctx, PCT_E_IO, std::string(path) + ": truncated binary payload");
  if (n_records == 0) return PCT_OK;

  // chunk = whole records, default 64 MiB; two pinned + two device buffers
  if (chunk_bytes <= 0) chunk_bytes = 64ll << 20;
  int64_t chunk_recs = std::max<int64_t>(kIngTile, chunk_bytes / record_bytes);
  chunk_recs = std::min<int64_t>(chunk_recs, n_records);
  const int64_t cbytes = chunk_recs * record_bytes;
  const size_t slot = ((size_t)cbytes + 255) / 256 * 256;
  if (int rc = ensure_staging(ctx, 2 * slot)) return rc;
  if ((int64_t)ctx->pinned_io_bytes < (int64_t)(2 * slot)) {
    if (ctx->pinned_io) cudaFreeHost(ctx->pinned_io);
    ctx->pinned_io = nullptr;
    ctx->pinned_io_bytes = 0;
    PCT_CUDA(ctx, cudaMallocHost(&ctx->pinned_io, 2 * slot));
    ctx->pinned_io_bytes = 2 * slot;
  }
  uint32_t *counts;
  int64_t *offsets;
  unsigned long long *total;
  if (int rc = tile_scratch(ctx, chunk_recs, counts, offsets, total)) return rc;
  cudaEvent_t freed[2];
  PCT_CUDA(ctx, cudaEventCreateWithFlags(&freed[0], cudaEventDisableTiming));
  PCT_CUDA(ctx, cudaEventCreateWithFlags(&freed[1], cudaEventDisableTiming));
  struct EvGuard {
    cudaEvent_t *e;
    ~EvGuard() {
      cudaEventDestroy(e[0]);
      cudaEventDestroy(e[1]);
    }
  } evg{freed};
  const unsigned hw = std::thread::hardware_concurrency();
  const int threads = (int)std::min(8u, std::max(1u, hw / 2));
  unsigned char *host = static_cast<unsigned char *>(ctx->pinned_io);
  unsigned char *dev = static_cast<unsigned char *>(ctx->staging);
  for (int64_t c = 0, r0 = 0; r0 < n_records; ++c, r0 += chunk_recs) {
    const int b = (int)(c & 1);
    const int64_t nr = std::min(chunk_recs, n_records - r0);
    if (c >= 2) PCT_CUDA(ctx, cudaEventSynchronize(freed[b]));  // DMA out of slot b done
    if (!pread_all(fd, host + b * slot, data_offset + r0 * record_bytes, nr * record_bytes,
                   threads))
      return fail(ctx, PCT_E_IO, std::string(path) + ": read failed");
    PCT_CUDA(ctx, cudaMemcpyAsync(dev + b * slot, host + b * slot, (size_t)(nr * record_bytes),
                                  cudaMemcpyHostToDevice, ctx->stream));
    PCT_CUDA(ctx, cudaEventRecord(freed[b], ctx->stream));
    // survivors of earlier chunks are appended in order (offsets based at *total)
    if (int rc = launch_extract(ctx, dev + b * slot, nr, L, counts, offsets, total, xyz_out))
      return rc;
  }
  return read_total(ctx, total, n_valid);
}

}  // extern "C"
