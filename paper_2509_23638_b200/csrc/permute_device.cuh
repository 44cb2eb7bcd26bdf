// Stable counting-sort permute of one block of top-k ids (K2 index pass), shared by the
// standalone K2 kernel (1024 threads) and the fused route+permute decode kernel (the
// last route CTA, 256 threads). Rows are ordered (expert asc, flat index asc): per
// kThreads-element chunk each warp ranks equal experts with __match_any_sync and the
// per-warp counts go through a [warps][E] shared table, so positions are deterministic
// without global atomics. kCoherent: ids were written by other CTAs of the same launch
// (read them from L2, never a stale L1 line).
#pragma once
#include "device_common.cuh"

namespace ps {

constexpr int kPermMaxE = 256;

template <int kThreads, bool kCoherent>
__device__ __forceinline__ void permute_block(const int32_t* __restrict__ ids, int n, int E,
                                              int32_t* __restrict__ offsets, int32_t* __restrict__ perm_src,
                                              int32_t* __restrict__ inv, int* s_base,
                                              int (*s_warp_cnt)[kPermMaxE]) {
  constexpr int kWarps = kThreads / 32;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  auto load_id = [&](int i) { return kCoherent ? __ldcg(ids + i) : ids[i]; };

  // Histogram -> exclusive scan -> offsets.
  for (int e = tid; e <= E; e += kThreads) s_base[e] = 0;
  __syncthreads();
  for (int i = tid; i < n; i += kThreads) atomicAdd(&s_base[load_id(i) + 1], 1);
  __syncthreads();
  if (warp == 0) {  // warp-level inclusive scan over E+1 entries, 32 at a time
    int carry = 0;
    for (int e0 = 0; e0 <= E; e0 += 32) {
      int v = e0 + lane <= E ? s_base[e0 + lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
      }
      v += carry;
      if (e0 + lane <= E) s_base[e0 + lane] = v;
      carry = __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  for (int e = tid; e <= E; e += kThreads) offsets[e] = s_base[e];
  // s_base[e] now holds the running insertion base of expert e.

  const unsigned lt_mask = (1u << lane) - 1u;
  for (int c0 = 0; c0 < n; c0 += kThreads) {
    for (int i = tid; i < kWarps * E; i += kThreads) s_warp_cnt[i / E][i % E] = 0;
    __syncthreads();
    const int i = c0 + tid;
    const bool valid = i < n;
    const int e = valid ? load_id(i) : -1 - lane;  // invalid lanes never match anyone
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const int rank = __popc(peers & lt_mask);
    if (valid && rank == 0) s_warp_cnt[warp][e] = __popc(peers);
    __syncthreads();
    if (valid) {
      int before = 0;
      for (int w = 0; w < warp; ++w) before += s_warp_cnt[w][e];
      const int pos = s_base[e] + before + rank;
      perm_src[pos] = i;
      inv[i] = pos;
    }
    __syncthreads();
    for (int ee = tid; ee < E; ee += kThreads) {
      int tot = 0;
      for (int w = 0; w < kWarps; ++w) tot += s_warp_cnt[w][ee];
      s_base[ee] += tot;
    }
    __syncthreads();
  }
}

}  // namespace ps
