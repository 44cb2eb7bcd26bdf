// Per-CTA device timeline of the persistent decode FFN kernel (globaltimer at item
// begin / dependency satisfied / stages consumed / epilogue done, producer item begin).
// Includes the kernel TU with PS_FFN_TRACE so the product build carries no hooks.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I../../include
//        -I../../paper_2509_23638_b200/csrc -o ffn_trace ffn_trace.cu
//   ./ffn_trace <experts> <tokens>  -> JSON lines per CTA item
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
__device__ unsigned long long g_trace[148][96][5];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PS_FFN_TRACE 1
#define PS_STAGE_CHECK(it, k0, hf, kl, mt, a0, a8)
#define PS_TRACE(ord, k) \
  do { if ((ord) < 96 && blockIdx.x < 148) g_trace[blockIdx.x][(ord)][(k)] = gtime(); } while (0)
#include "k3_ffn_decode.cu"

int main(int argc, char** argv) {
  const int E = argc > 1 ? atoi(argv[1]) : 1, M = argc > 2 ? atoi(argv[2]) : 4;
  const int H = 4096, F = 14336, k = 1;
  std::vector<uint16_t*> slabs(E);
  for (auto& s : slabs) cudaMalloc(&s, 3ull * H * F * 2);
  for (int e = 0; e < E; ++e) ps_init_expert_slab(slabs[e], H, F, 1, 0, e, nullptr);
  const int rows = E * M;
  std::vector<int32_t> off(E + 1), src(rows), counts(E, M);
  for (int e = 0; e <= E; ++e) off[e] = e * M;
  for (int r = 0; r < rows; ++r) src[r] = r;
  int32_t *doff, *dsrc; uint16_t *x, *h; float* y;
  cudaMalloc(&doff, sizeof(int32_t) * (E + 1)); cudaMalloc(&dsrc, sizeof(int32_t) * rows);
  cudaMemcpy(doff, off.data(), sizeof(int32_t) * (E + 1), cudaMemcpyHostToDevice);
  cudaMemcpy(dsrc, src.data(), sizeof(int32_t) * rows, cudaMemcpyHostToDevice);
  cudaMalloc(&x, 2ull * rows * H); cudaMemset(x, 0, 2ull * rows * H);
  cudaMalloc(&h, 2ull * rows * F);
  const int ns = ps_ffn_down_splits(H, F);
  cudaMalloc(&y, 4ull * ns * rows * H);
  ps_expert_group g{};
  g.n = E;
  for (int e = 0; e < E; ++e) { g.experts[e] = e; g.slabs[e] = slabs[e]; }
  for (int it = 0; it < 3; ++it) ps_expert_ffn(&g, counts.data(), doff, dsrc, k, x, H, F, h, y, ns, rows, nullptr);
  cudaDeviceSynchronize();
  static unsigned long long zero[148][96][5];
  cudaMemcpyToSymbol(g_trace, zero, sizeof(zero));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  int st = ps_expert_ffn(&g, counts.data(), doff, dsrc, k, x, H, F, h, y, ns, rows, nullptr);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  static unsigned long long tr[148][96][5];
  cudaMemcpyFromSymbol(tr, g_trace, sizeof(tr));
  unsigned long long t0 = ~0ull;
  for (int c = 0; c < 148; ++c) if (tr[c][0][4]) t0 = std::min(t0, tr[c][0][4]);
  printf("{\"status\": %d, \"experts\": %d, \"tokens\": %d, \"event_us\": %.2f}\n", st, E, M, ms * 1e3);
  for (int c = 0; c < 148; ++c)
    for (int o = 0; o < 96; ++o) {
      if (!tr[c][o][0]) continue;
      printf("{\"cta\": %d, \"ord\": %d, \"prod\": %.2f, \"begin\": %.2f, \"dep\": %.2f, \"stages\": %.2f, \"end\": %.2f}\n", c, o,
             (tr[c][o][4] - t0) / 1e3, (tr[c][o][0] - t0) / 1e3, (tr[c][o][1] - t0) / 1e3, (tr[c][o][2] - t0) / 1e3,
             (tr[c][o][3] - t0) / 1e3);
    }
  return 0;
}
