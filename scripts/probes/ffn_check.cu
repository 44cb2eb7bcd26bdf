// Debug harness: verifies every A fragment the decode FFN consumers read from the shared-
// memory ring against the weights in global memory, and run-to-run determinism.
//   ./ffn_check <experts> <tokens B> <H> <F> <reps> <top-k>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
__device__ const uint16_t* g_slab[256];
__device__ unsigned int g_bad;
__device__ int g_first[8];
#define PS_FFN_TRACE 1
#define PS_TRACE(ord, k)
#ifdef NOCHECK
#define PS_STAGE_CHECK(it, k0, hf, kl, mt, a0, a8)
#else
#define PS_STAGE_CHECK(it, k0, hf, kl, mt, a0, a8)                                                      \
  do {                                                                                                    \
    const uint16_t* sl = g_slab[p.expert[it.i]];                                                          \
    const int col = k0 + hf * 256 + kl;                                                                   \
    if (col < it.kend) {                                                                                  \
      for (int h_ = 0; h_ < 2; ++h_) {                                                                    \
        const int rr = 16 * mt + gid + 8 * h_; /* row inside the item */                                 \
        const uint16_t* row;                                                                              \
        bool ok;                                                                                          \
        if (!it.down) {                                                                                   \
          const int half = 8 * MT; /* gate rows [0, half), up rows [half, 2 half) */                     \
          const int f = it.r0 + (rr % half);                                                              \
          ok = f < p.F;                                                                                   \
          row = sl + (size_t)((rr < half ? 0 : p.F) + f) * p.H;                                           \
        } else {                                                                                          \
          ok = it.r0 + rr < p.H;                                                                          \
          row = sl + 2ull * p.F * p.H + (size_t)(it.r0 + rr) * p.F;                                       \
        }                                                                                                 \
        if (!ok) continue;                                                                                \
        const uint4 want = *reinterpret_cast<const uint4*>(row + col);                                    \
        const uint4 got = h_ ? a8 : a0;                                                                   \
        if (want.x != got.x || want.y != got.y || want.z != got.z || want.w != got.w) {                   \
          if (atomicAdd(&g_bad, 1u) == 0) {                                                               \
            g_first[0] = blockIdx.x; g_first[1] = it.i; g_first[2] = it.down; g_first[3] = it.r0;         \
            g_first[4] = col; g_first[5] = rr; g_first[6] = (int)n; g_first[7] = warp;                    \
          }                                                                                               \
        }                                                                                                 \
      }                                                                                                   \
    }                                                                                                     \
  } while (0)
#endif
#include "k3_ffn_decode.cu"

int main(int argc, char** argv) {
  const int E = argc > 1 ? atoi(argv[1]) : 10, M = argc > 2 ? atoi(argv[2]) : 1;
  const int H = argc > 3 ? atoi(argv[3]) : 2048, F = argc > 4 ? atoi(argv[4]) : 768;
  const int reps = argc > 5 ? atoi(argv[5]) : 5;
  std::vector<uint16_t*> slabs(E);
  for (auto& s : slabs) cudaMalloc(&s, 3ull * H * F * 2);
  for (int e = 0; e < E; ++e) ps_init_expert_slab(slabs[e], H, F, 1, 0, e, nullptr);
  cudaMemcpyToSymbol(g_slab, slabs.data(), sizeof(void*) * E);
  // Routing like the Python stress: B tokens, top-K distinct experts each (LCG), permuted by K2.
  const int B = M, K = argc > 6 ? atoi(argv[6]) : 2;
  const int k = K;
  std::vector<int32_t> ids((size_t)B * K);
  uint64_t st_ = 12345;
  auto rnd = [&]() { st_ = st_ * 6364136223846793005ull + 1442695040888963407ull; return (int)(st_ >> 33); };
  for (int t = 0; t < B; ++t)
    for (int j = 0; j < K; ++j) {
      int e;
      bool dup;
      do { e = rnd() % E; dup = false; for (int q = 0; q < j; ++q) dup |= ids[t * K + q] == e; } while (dup);
      ids[t * K + j] = e;
    }
  const int rows = B * K;
  std::vector<int32_t> counts(E, 0);
  for (int v : ids) counts[v]++;
  int32_t *dids, *doff, *dsrc, *dinv;
  cudaMalloc(&dids, 4 * rows); cudaMalloc(&doff, 4 * (E + 1)); cudaMalloc(&dsrc, 4 * rows); cudaMalloc(&dinv, 4 * rows);
  cudaMemcpy(dids, ids.data(), 4 * rows, cudaMemcpyHostToDevice);
  ps_permute(dids, B, K, E, doff, dsrc, dinv, nullptr, H, nullptr, nullptr);
  uint16_t *x, *h; float* y;
  std::vector<uint16_t> xh((size_t)rows * H);
  for (size_t i = 0; i < xh.size(); ++i) xh[i] = 0x3c00 + (uint16_t)(i * 2654435761u >> 24) % 64;  // small bf16s
  cudaMalloc(&x, 2ull * rows * H); cudaMemcpy(x, xh.data(), 2ull * B * H, cudaMemcpyHostToDevice);
  cudaMalloc(&h, 2ull * rows * F);
  const int ns = ps_ffn_down_splits(H, F);
  cudaMalloc(&y, 4ull * ns * rows * H);
  ps_expert_group g{};
  g.n = E;
  for (int e = 0; e < E; ++e) { g.experts[e] = e; g.slabs[e] = slabs[e]; }
  std::vector<float> y0((size_t)ns * rows * H), y1(y0.size());
  std::vector<uint16_t> h0((size_t)rows * F), h1(h0.size());
  const bool fresh = getenv("FRESH") != nullptr;
  for (int r = 0; r < reps; ++r) {
    if (fresh) {  // new output buffers each rep (like torch.full per rep); old ones leak
      cudaMalloc(&h, 2ull * rows * F);
      cudaMalloc(&y, 4ull * ns * rows * H);
    }
    cudaMemset(h, 0xff, 2ull * rows * F);
    cudaMemset(y, 0xff, 4ull * ns * rows * H);
    unsigned zero = 0;
    cudaMemcpyToSymbol(g_bad, &zero, 4);
    int st = ps_expert_ffn(&g, counts.data(), doff, dsrc, k, x, H, F, h, y, ns, rows, nullptr);
    cudaError_t ce = cudaDeviceSynchronize();
    unsigned bad; int first[8];
    cudaMemcpyFromSymbol(&bad, g_bad, 4); cudaMemcpyFromSymbol(first, g_first, sizeof(first));
    cudaMemcpy(r == 0 ? y0.data() : y1.data(), y, 4 * y0.size(), cudaMemcpyDeviceToHost);
    cudaMemcpy(r == 0 ? h0.data() : h1.data(), h, 2 * h0.size(), cudaMemcpyDeviceToHost);
    int ydiff = 0, hdiff = 0;
    if (r > 0) {
      for (size_t i = 0; i < y0.size(); ++i) ydiff += memcmp(&y0[i], &y1[i], 4) != 0;
      for (size_t i = 0; i < h0.size(); ++i) hdiff += h0[i] != h1[i];
    }
    printf("rep %d status %d cuda %s: bad fragments %u (cta %d entry %d down %d r0 %d col %d q %d n %d warp %d); h diffs %d y diffs %d\n",
           r, st, cudaGetErrorString(ce), bad, first[0], first[1], first[2], first[3], first[4], first[5], first[6], first[7],
           hdiff, ydiff);
  }
  return 0;
}
