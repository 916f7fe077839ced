// xfer_host.cpp — host side of the compacted layer read-back (k_xfer.cu):
// pct_xfer_expand rebuilds slices from their bitmaps and packed values.
// Compiled by g++ into libpct.so.  The rebuild is bound by the host's
// memory bandwidth (every output byte is written once, with non-temporal
// stores: no read-for-ownership), so the inner loops are kept short:
//   * AVX-512 (when the CPU has it, checked at run time): 16 cells per
//     masked expand-load (vpexpandd) -- the bitmap's 16 bits select which
//     lanes take the next packed values, the others keep their base (the
//     empty NaN, or in a delta chain the previous slice's value);
//   * otherwise SSE2: one 32-cell word at a time through a staging line.
// NaN mode (delta = 0): items are (slice, chunk) pairs.  Delta chains
// (delta = 1): items are chunks; a thread keeps its chunk's current state in
// a cache-resident buffer and patches it slice after slice.
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

extern "C" int64_t pct_xfer_chunk_cells(void);

namespace {

constexpr uint32_t kNaN = 0x7FC00000u;  // numpy's NaN: the empty cell
constexpr int kInvalid = -1;            // PCT_E_INVALID

struct Job {
  const uint32_t *bitmaps;
  const float *packed;
  const int64_t *chunk_off;
  int32_t n;
  int64_t cells, W, nchunk, chunk;
  float *const *outs;
  const float *base;  // delta chains: slice 0's predecessor (NULL: the empty NaN)
};

// ---- SSE2 path ------------------------------------------------------------
inline void put_line_sse2(float *dst, const float *line, int nc) {
  if (nc == 32 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    const __m128i *s = reinterpret_cast<const __m128i *>(line);
    __m128i *d = reinterpret_cast<__m128i *>(dst);
    for (int q = 0; q < 8; ++q) _mm_stream_si128(d + q, _mm_load_si128(s + q));
    return;
  }
  std::memcpy(dst, line, sizeof(float) * (size_t)nc);
}

void nan_item_sse2(const Job &J, int64_t it) {
  alignas(64) float line[32];
  float nanv;
  std::memcpy(&nanv, &kNaN, 4);
  const int64_t m = it / J.nchunk, c = it - m * J.nchunk;
  const uint32_t *bm = J.bitmaps + m * J.W;
  const float *p = J.packed + J.chunk_off[m * J.nchunk + c];
  float *o = J.outs[m];
  const int64_t w0 = c * (J.chunk / 32), w1 = std::min(J.W, w0 + J.chunk / 32);
  for (int64_t w = w0; w < w1; ++w) {
    const uint32_t bits = bm[w];
    const int nc = (int)std::min<int64_t>(32, J.cells - w * 32);
    if (bits == 0xFFFFFFFFu && nc == 32) {
      std::memcpy(line, p, 128);
      p += 32;
    } else {
      for (int j = 0; j < 32; ++j) line[j] = (bits >> j & 1u) ? *p++ : nanv;
    }
    put_line_sse2(o + w * 32, line, nc);
  }
}

void delta_item_sse2(const Job &J, int64_t c, float *buf) {
  float nanv;
  std::memcpy(&nanv, &kNaN, 4);
  const int64_t w0 = c * (J.chunk / 32), w1 = std::min(J.W, w0 + J.chunk / 32);
  for (int32_t m = 0; m < J.n; ++m) {
    const uint32_t *bm = J.bitmaps + m * J.W;
    const float *p = J.packed + J.chunk_off[m * J.nchunk + c];
    float *o = J.outs[m];
    for (int64_t w = w0; w < w1; ++w) {
      uint32_t bits = bm[w];
      float *line = buf + (w - w0) * 32;
      const int nc = (int)std::min<int64_t>(32, J.cells - w * 32);
      if (m == 0) {
        const float *b0 = J.base ? J.base + w * 32 : nullptr;
        for (int j = 0; j < 32; ++j)
          line[j] = (bits >> j & 1u) ? *p++ : (b0 && j < nc ? b0[j] : nanv);
      } else {
        while (bits) {
          const int j = __builtin_ctz(bits);
          bits &= bits - 1u;
          line[j] = *p++;
        }
      }
      put_line_sse2(o + w * 32, line, nc);
    }
  }
}

// ---- AVX-512 path ---------------------------------------------------------
// A 32-cell word as two 16-lane masked expand-loads over `base`, streamed
// out when the destination is 64-byte aligned and whole.
__attribute__((target("avx512f"))) inline void word_avx512(float *dst, float *state,
                                                           const float *&p, uint32_t bits,
                                                           __m512 lo, __m512 hi, int nc) {
  const __mmask16 m0 = (__mmask16)(bits & 0xFFFFu), m1 = (__mmask16)(bits >> 16);
  const __m512 v0 = _mm512_mask_expandloadu_ps(lo, m0, p);
  p += __builtin_popcount(bits & 0xFFFFu);
  const __m512 v1 = _mm512_mask_expandloadu_ps(hi, m1, p);
  p += __builtin_popcount(bits >> 16);
  if (state) {
    _mm512_store_ps(state, v0);
    _mm512_store_ps(state + 16, v1);
  }
  if (nc == 32 && (reinterpret_cast<uintptr_t>(dst) & 63) == 0) {
    _mm512_stream_ps(dst, v0);
    _mm512_stream_ps(dst + 16, v1);
  } else {
    alignas(64) float line[32];
    _mm512_store_ps(line, v0);
    _mm512_store_ps(line + 16, v1);
    std::memcpy(dst, line, sizeof(float) * (size_t)nc);
  }
}

__attribute__((target("avx512f"))) void nan_item_avx512(const Job &J, int64_t it) {
  const __m512 nanv = _mm512_castsi512_ps(_mm512_set1_epi32((int)kNaN));
  const int64_t m = it / J.nchunk, c = it - m * J.nchunk;
  const uint32_t *bm = J.bitmaps + m * J.W;
  const float *p = J.packed + J.chunk_off[m * J.nchunk + c];
  float *o = J.outs[m];
  const int64_t w0 = c * (J.chunk / 32), w1 = std::min(J.W, w0 + J.chunk / 32);
  for (int64_t w = w0; w < w1; ++w) {
    const int nc = (int)std::min<int64_t>(32, J.cells - w * 32);
    word_avx512(o + w * 32, nullptr, p, bm[w], nanv, nanv, nc);
  }
}

__attribute__((target("avx512f"))) void delta_item_avx512(const Job &J, int64_t c, float *buf) {
  const __m512 nanv = _mm512_castsi512_ps(_mm512_set1_epi32((int)kNaN));
  const int64_t w0 = c * (J.chunk / 32), w1 = std::min(J.W, w0 + J.chunk / 32);
  for (int32_t m = 0; m < J.n; ++m) {
    const uint32_t *bm = J.bitmaps + m * J.W;
    const float *p = J.packed + J.chunk_off[m * J.nchunk + c];
    float *o = J.outs[m];
    for (int64_t w = w0; w < w1; ++w) {
      float *st = buf + (w - w0) * 32;
      const int nc = (int)std::min<int64_t>(32, J.cells - w * 32);
      __m512 lo = nanv, hi = nanv;
      if (m) {
        lo = _mm512_load_ps(st);
        hi = _mm512_load_ps(st + 16);
      } else if (J.base) {  // continuing a chain: the predecessor's cells (masked tail)
        const __mmask16 ml = (__mmask16)(nc >= 16 ? 0xFFFFu : (1u << nc) - 1u);
        const __mmask16 mh = (__mmask16)(nc >= 32 ? 0xFFFFu : nc > 16 ? (1u << (nc - 16)) - 1u : 0u);
        lo = _mm512_mask_loadu_ps(nanv, ml, J.base + w * 32);
        hi = _mm512_mask_loadu_ps(nanv, mh, J.base + w * 32 + 16);
      }
      word_avx512(o + w * 32, st, p, bm[w], lo, hi, nc);
    }
  }
}

bool has_avx512() {
  static const bool v = __builtin_cpu_supports("avx512f");
  return v;
}

}  // namespace

extern "C" int pct_xfer_expand_from(const uint32_t *bitmaps, const float *packed,
                                    const int64_t *chunk_off, int32_t n, int64_t cells,
                                    int32_t delta, float *const *outs, int32_t nthreads,
                                    const float *base) {
  if (n <= 0) return 0;
  if (!bitmaps || !packed || !chunk_off || !outs || cells <= 0) return kInvalid;
  if (base && !delta) return kInvalid;
  Job J{bitmaps, packed, chunk_off, n, cells, (cells + 31) / 32, 0, pct_xfer_chunk_cells(), outs,
        base};
  J.nchunk = (cells + J.chunk - 1) / J.chunk;
  const int64_t items = delta ? J.nchunk : (int64_t)n * J.nchunk;
  const bool avx = has_avx512();
  // items are claimed in small groups from a shared counter (chunks with
  // many changed cells take longer: a static split left threads idle at the
  // end of every stack)
  std::atomic<int64_t> next{0};
  constexpr int64_t kGrab = 2;
  auto work = [&]() {
    float *buf = nullptr;
    if (delta) buf = static_cast<float *>(aligned_alloc(64, (size_t)J.chunk * 4 + 64));
    for (;;) {
      const int64_t i0 = next.fetch_add(kGrab, std::memory_order_relaxed);
      if (i0 >= items) break;
      const int64_t i1 = std::min(items, i0 + kGrab);
      for (int64_t it = i0; it < i1; ++it) {
        if (delta) {
          if (avx) delta_item_avx512(J, it, buf);
          else delta_item_sse2(J, it, buf);
        } else {
          if (avx) nan_item_avx512(J, it);
          else nan_item_sse2(J, it);
        }
      }
    }
    _mm_sfence();
    free(buf);
  };
  int nt = std::max(1, std::min<int>(nthreads, (int)std::min<int64_t>(items, 256)));
  if (nt == 1) {
    work();
    return 0;
  }
  std::vector<std::thread> th;
  th.reserve((size_t)nt - 1);
  for (int t = 1; t < nt; ++t) th.emplace_back(work);
  work();  // the calling thread takes items too
  for (auto &x : th) x.join();
  return 0;
}

extern "C" int pct_xfer_expand(const uint32_t *bitmaps, const float *packed,
                               const int64_t *chunk_off, int32_t n, int64_t cells,
                               int32_t delta, float *const *outs, int32_t nthreads) {
  return pct_xfer_expand_from(bitmaps, packed, chunk_off, n, cells, delta, outs, nthreads,
                              nullptr);
}
