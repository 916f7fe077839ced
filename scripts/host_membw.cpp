// Host write-bandwidth probe (diagnostic): 16 threads filling a 2 GB buffer
// with plain stores, SSE2 non-temporal stores and AVX-512 non-temporal stores.
#include <immintrin.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
int main() {
  const size_t n = (size_t)2 << 30;
  char *buf = (char *)aligned_alloc(4096, n);
  memset(buf, 1, n);  // fault in
  int nt = std::thread::hardware_concurrency();
  auto run = [&](int mode) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
      th.emplace_back([&, t] {
        char *a = buf + n / nt * t, *b = buf + n / nt * (t + 1);
        if (mode == 0) { for (char *p = a; p < b; p += 64) { memset(p, t, 64); } }
        else if (mode == 1) { __m128i v = _mm_set1_epi32(t); for (char *p = a; p < b; p += 16) _mm_stream_si128((__m128i *)p, v); _mm_sfence(); }
        else { __m512i v = _mm512_set1_epi32(t); for (char *p = a; p < b; p += 64) _mm512_stream_si512((__m512i *)p, v); _mm_sfence(); }
      });
    for (auto &x : th) x.join();
    double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("mode %d (%s): %.1f GB/s\n", mode, mode == 0 ? "plain" : mode == 1 ? "sse2 NT" : "avx512 NT", n / s / 1e9);
  };
  for (int r = 0; r < 2; ++r) for (int m = 0; m < 3; ++m) run(m);
}
