// Host write-bandwidth probe (diagnostic): AVX-512 non-temporal stores by all
// host threads into a 2 GB buffer of 4 KB pages vs transparent huge pages
// (mmap + madvise(MADV_HUGEPAGE)).
#include <immintrin.h>
#include <sys/mman.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
int main() {
  const size_t n = (size_t)2 << 30;
  char *small = (char *)mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  madvise(small, n, MADV_NOHUGEPAGE);
  char *huge = (char *)mmap(nullptr, n + (2 << 20), PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  huge = (char *)(((uintptr_t)huge + (2 << 20) - 1) & ~(uintptr_t)((2 << 20) - 1));
  int rc = madvise(huge, n, MADV_HUGEPAGE);
  memset(small, 1, n);
  memset(huge, 1, n);
  int nt = std::thread::hardware_concurrency();
  auto run = [&](char *buf, const char *name) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
      th.emplace_back([&, t] {
        char *a = buf + n / nt * t, *b = buf + n / nt * (t + 1);
        __m512i v = _mm512_set1_epi32(t);
        for (char *p = a; p < b; p += 64) _mm512_stream_si512((__m512i *)p, v);
        _mm_sfence();
      });
    for (auto &x : th) x.join();
    double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("%s: %.1f GB/s\n", name, n / s / 1e9);
  };
  printf("madvise(MADV_HUGEPAGE) rc %d\n", rc);
  for (int r = 0; r < 3; ++r) { run(small, "4K pages NT"); run(huge, "THP NT"); }
}
