// Host DRAM read bandwidth probe (the host expert lane's roofline): T threads stream a
// buffer far larger than the LLC with 64-byte AVX-512 loads (sum-reduced so the loads
// are not elided), best of R passes. Build: gcc -O3 -mavx512f -fopenmp host_stream.c
#include <immintrin.h>
#include <omp.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>

int main(int argc, char** argv) {
  const size_t gb = argc > 1 ? (size_t)atol(argv[1]) : 16;
  const int reps = argc > 2 ? atoi(argv[2]) : 5;
  const size_t n = gb << 30;
  char* buf = mmap(NULL, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  madvise(buf, n, MADV_HUGEPAGE);
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < n; i += 4096) buf[i] = (char)i;
  double best = 0;
  for (int r = 0; r < reps; ++r) {
    double t0 = omp_get_wtime();
    __m512i acc_all = _mm512_setzero_si512();
#pragma omp parallel
    {
      __m512i acc = _mm512_setzero_si512();
#pragma omp for schedule(static)
      for (size_t i = 0; i < n; i += 256) {
        acc = _mm512_add_epi64(acc, _mm512_load_si512((const void*)(buf + i)));
        acc = _mm512_add_epi64(acc, _mm512_load_si512((const void*)(buf + i + 64)));
        acc = _mm512_add_epi64(acc, _mm512_load_si512((const void*)(buf + i + 128)));
        acc = _mm512_add_epi64(acc, _mm512_load_si512((const void*)(buf + i + 192)));
      }
#pragma omp critical
      acc_all = _mm512_add_epi64(acc_all, acc);
    }
    double dt = omp_get_wtime() - t0;
    long long s[8];
    _mm512_storeu_si512(s, acc_all);
    double gbs = n / dt / 1e9;
    if (gbs > best) best = gbs;
    fprintf(stderr, "pass %d: %.1f GB/s (checksum %lld)\n", r, gbs, s[0]);
  }
  printf("{\"probe\": \"host_dram_read\", \"threads\": %d, \"buffer_gb\": %zu, \"best_gbs\": %.1f}\n",
         omp_get_max_threads(), gb, best);
  return 0;
}
