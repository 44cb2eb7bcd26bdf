/* TEST / BASELINE INFRASTRUCTURE ONLY — never linked into the product.
 *
 * CPU port of the MoE layer for bench.py's CPU baseline (`--impl reference` and the
 * `cpu_baseline` leg). The reference has no expert FFN (it only
 * simulates the layer), so the arm's expert computation is this port of the SAME
 * arithmetic the oracle (oracle.c or_moe_layer) and the GPU path compute:
 * y_t = sum_{e in topk(t)} w_t[e] * W_down (SiLU(W_gate x_t) * (W_up x_t)), bf16 weights
 * and inputs, h rounded to bf16, combine in the full-softmax gate weights
 * (workload.cpp:190-195).
 *
 * Unlike oracle.c (one f64 GEMV per (token, expert) pair: the checker, slow on purpose)
 * this is written to be a fair CPU baseline: each routed expert's weights are streamed
 * ONCE per layer for all of its tokens, rows split over OpenMP threads, f32 accumulation
 * in AVX-512 (16 lanes, bf16 -> f32 by a 16-bit shift) when the host has it, so the port
 * runs near the host's DRAM bandwidth instead of its scalar f64 rate. */
#include <immintrin.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define TOK_GROUP 8 /* tokens per weight pass (register accumulators) */

static inline float bf16f(uint16_t v) {
  union { uint32_t u; float f; } c;
  c.u = (uint32_t)v << 16;
  return c.f;
}

static inline uint16_t f2bf16(float f) { /* round to nearest even (finite values) */
  union { uint32_t u; float f; } c;
  c.f = f;
  return (uint16_t)((c.u + 0x7FFFu + ((c.u >> 16) & 1u)) >> 16);
}

/* acc[j] = sum_d w[d] * x[j*ld + d], j < m (m <= TOK_GROUP), n % 16 == 0 */
__attribute__((target("avx512f,avx512bw"))) static void dot_avx512(const uint16_t* w, const float* x, int ld, int n,
                                                                   int m, float* acc) {
  __m512 a[TOK_GROUP];
  for (int j = 0; j < TOK_GROUP; ++j) a[j] = _mm512_setzero_ps();
  for (int d = 0; d < n; d += 16) {
    const __m512 wv = _mm512_castsi512_ps(
        _mm512_slli_epi32(_mm512_cvtepu16_epi32(_mm256_loadu_si256((const __m256i*)(w + d))), 16));
    switch (m) { /* fallthrough: accumulators j < m */
      case 8: a[7] = _mm512_fmadd_ps(wv, _mm512_loadu_ps(x + 7 * (size_t)ld + d), a[7]); /* fall through */
      case 7: a[6] = _mm512_fmadd_ps(wv, _mm512_loadu_ps(x + 6 * (size_t)ld + d), a[6]); /* fall through */
      case 6: a[5] = _mm512_fmadd_ps(wv, _mm512_loadu_ps(x + 5 * (size_t)ld + d), a[5]); /* fall through */
      case 5: a[4] = _mm512_fmadd_ps(wv, _mm512_loadu_ps(x + 4 * (size_t)ld + d), a[4]); /* fall through */
      case 4: a[3] = _mm512_fmadd_ps(wv, _mm512_loadu_ps(x + 3 * (size_t)ld + d), a[3]); /* fall through */
      case 3: a[2] = _mm512_fmadd_ps(wv, _mm512_loadu_ps(x + 2 * (size_t)ld + d), a[2]); /* fall through */
      case 2: a[1] = _mm512_fmadd_ps(wv, _mm512_loadu_ps(x + 1 * (size_t)ld + d), a[1]); /* fall through */
      default: a[0] = _mm512_fmadd_ps(wv, _mm512_loadu_ps(x + d), a[0]);
    }
  }
  for (int j = 0; j < m; ++j) acc[j] = _mm512_reduce_add_ps(a[j]);
}

static void dot_scalar(const uint16_t* w, const float* x, int ld, int n, int m, float* acc) {
  for (int j = 0; j < m; ++j) {
    float s = 0.f;
    for (int d = 0; d < n; ++d) s += bf16f(w[d]) * x[(size_t)j * ld + d];
    acc[j] = s;
  }
}

static int use_avx512(int n) {
  static int have = -1;
  if (have < 0) have = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw");
  return have && n % 16 == 0;
}

/* One expert over its m tokens (rows of xf [m, H] f32) -> ye [m, H] f32. hf: [m, F] scratch. */
static void expert_ffn(const uint16_t* slab, int H, int F, int m, const float* xf, float* hf, float* ye,
                       int threads) {
  const uint16_t* wg = slab;
  const uint16_t* wu = slab + (size_t)F * H;
  const uint16_t* wd = slab + (size_t)2 * F * H;
  const int vec_h = use_avx512(H), vec_f = use_avx512(F);
  for (int j0 = 0; j0 < m; j0 += TOK_GROUP) {
    const int mg = m - j0 < TOK_GROUP ? m - j0 : TOK_GROUP;
#pragma omp parallel for schedule(static) num_threads(threads)
    for (int f = 0; f < F; ++f) {
      float g[TOK_GROUP], u[TOK_GROUP];
      (vec_h ? dot_avx512 : dot_scalar)(wg + (size_t)f * H, xf + (size_t)j0 * H, H, H, mg, g);
      (vec_h ? dot_avx512 : dot_scalar)(wu + (size_t)f * H, xf + (size_t)j0 * H, H, H, mg, u);
      for (int j = 0; j < mg; ++j) {
        const float s = g[j] / (1.f + expf(-g[j]));
        hf[(size_t)(j0 + j) * F + f] = bf16f(f2bf16(s * u[j]));
      }
    }
#pragma omp parallel for schedule(static) num_threads(threads)
    for (int r = 0; r < H; ++r) {
      float acc[TOK_GROUP];
      (vec_f ? dot_avx512 : dot_scalar)(wd + (size_t)r * F, hf + (size_t)j0 * F, F, F, mg, acc);
      for (int j = 0; j < mg; ++j) ye[(size_t)(j0 + j) * H + r] = acc[j];
    }
  }
}

/* slab[E] (null for unrouted experts), x [B,H] bf16, ids [B,k], gate [B,E] -> y [B,H]. */
void bl_moe_layer(const uint16_t* const* slab, int H, int F, int B, int k, int E, const uint16_t* x,
                  const int32_t* ids, const float* gate, float* y, int threads) {
  if (threads < 1) threads = 1;
  int* cnt = (int*)calloc((size_t)E, sizeof(int));
  for (int i = 0; i < B * k; ++i) cnt[ids[i]]++;
  int mmax = 0;
  for (int e = 0; e < E; ++e) mmax = cnt[e] > mmax ? cnt[e] : mmax;
  float* xf = (float*)malloc(sizeof(float) * (size_t)mmax * H);
  float* hf = (float*)malloc(sizeof(float) * (size_t)mmax * F);
  float* ye = (float*)malloc(sizeof(float) * (size_t)mmax * H);
  int* tok = (int*)malloc(sizeof(int) * (size_t)mmax);
  float* out = (float*)calloc((size_t)B * H, sizeof(float));
  for (int e = 0; e < E; ++e) {
    if (!cnt[e]) continue;
    int m = 0;
    for (int t = 0; t < B; ++t)
      for (int j = 0; j < k; ++j)
        if (ids[t * k + j] == e) tok[m++] = t;
    for (int i = 0; i < m; ++i)
      for (int d = 0; d < H; ++d) xf[(size_t)i * H + d] = bf16f(x[(size_t)tok[i] * H + d]);
    expert_ffn(slab[e], H, F, m, xf, hf, ye, threads);
    for (int i = 0; i < m; ++i) {
      const float w = gate[(size_t)tok[i] * E + e];
      float* o = out + (size_t)tok[i] * H;
      for (int d = 0; d < H; ++d) o[d] += w * ye[(size_t)i * H + d];
    }
  }
  memcpy(y, out, sizeof(float) * (size_t)B * H);
  free(cnt);
  free(xf);
  free(hf);
  free(ye);
  free(tok);
  free(out);
}

/* Parallel synthetic-weight materialisation for the baseline (one expert per thread):
 * the same values as oracle.c or_init_slab. */
void or_init_slab(uint16_t* slab, int H, int F, uint64_t seed, int layer, int expert);
void bl_init_slabs(uint16_t* const* out, const int32_t* layer, const int32_t* expert, int n, int H, int F,
                   uint64_t seed, int threads) {
#pragma omp parallel for schedule(dynamic) num_threads(threads > 0 ? threads : 1)
  for (int i = 0; i < n; ++i) or_init_slab(out[i], H, F, seed, layer[i], expert[i]);
}
