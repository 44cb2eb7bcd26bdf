// K2 — counting-sort token permute / unpermute + weighted combine.
//
// The reference only computes the per-expert token count (workload.cpp:202,
// aggregate_layer_loads workload.cpp:283-288; sort order simulator.cpp:45-57); the
// physical permute and the combine are absent there, so the order
// is defined here: permuted rows are (expert asc, token asc, slot asc) — a stable
// counting sort of the flattened top-k ids. Bit-exact against oracle/or_permute.
//
// Index pass: one CTA (B*k <= 64K assignments). Per 1024-element chunk each warp
// ranks equal experts with __match_any_sync, per-warp counts go through a [warps][E]
// shared table, so positions are deterministic without global atomics.
// Gather/combine passes: HBM-bound, 16-byte vectorised, one CTA row-slab each.
#include <algorithm>

#include "device_common.cuh"
#include "permute_device.cuh"

namespace ps {
namespace {

constexpr int kPermThreads = 1024;
constexpr int kPermWarps = kPermThreads / 32;
constexpr int kMaxE = 256;

__global__ void __launch_bounds__(kPermThreads)
permute_index_kernel(const int32_t* __restrict__ ids, int n, int E, int32_t* __restrict__ offsets,
                     int32_t* __restrict__ perm_src, int32_t* __restrict__ inv) {
  __shared__ int s_base[kMaxE + 1];
  __shared__ int s_warp_cnt[kPermWarps][kMaxE];
  permute_block<kPermThreads, false>(ids, n, E, offsets, perm_src, inv, s_base, s_warp_cnt);
}

// Multi-CTA index pass for prefill chunks (the single CTA above walks 1024-id chunks one
// after another: 42 us for 16K ids). One CTA per 1024-id chunk; each CTA histograms ALL
// ids (n <= 128K: at most 512 KiB of L2 reads per CTA, warp-aggregated shared atomics) into
// per-expert totals and the part before its chunk, so no cross-CTA scratch or second
// launch is needed; then it ranks its chunk exactly as permute_block does. Same (unique)
// stable order.
__global__ void __launch_bounds__(kPermThreads)
permute_chunks_kernel(const int32_t* __restrict__ ids, int n, int E, int32_t* __restrict__ offsets,
                      int32_t* __restrict__ perm_src, int32_t* __restrict__ inv) {
  __shared__ int s_base[kMaxE + 1];
  __shared__ int s_before[kMaxE];
  __shared__ int s_warp_cnt[kPermWarps][kMaxE];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, chunk = blockIdx.x;
  const int c0 = chunk * kPermThreads;
  for (int e = tid; e <= E; e += kPermThreads) s_base[e] = 0;
  for (int e = tid; e < E; e += kPermThreads) s_before[e] = 0;
  __syncthreads();
  for (int i0 = 0; i0 < n; i0 += kPermThreads) {  // warp-aggregated: one atomic per distinct expert
    const int i = i0 + tid;
    const int e = i < n ? __ldg(ids + i) : -1 - lane;
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    if (i < n && (peers & ((1u << lane) - 1u)) == 0) {
      atomicAdd(&s_base[e + 1], __popc(peers));
      if (i0 < c0) atomicAdd(&s_before[e], __popc(peers));  // whole earlier chunks only
    }
  }
  __syncthreads();
  if (warp == 0) {  // inclusive scan of the totals -> offsets
    int carry = 0;
    for (int e0 = 0; e0 <= E; e0 += 32) {
      int v = e0 + lane <= E ? s_base[e0 + lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
      }
      v += carry;
      if (e0 + lane <= E) s_base[e0 + lane] = v;
      carry = __shfl_sync(0xffffffffu, v, 31);
    }
  }
  for (int i2 = tid; i2 < kPermWarps * E; i2 += kPermThreads) s_warp_cnt[i2 / E][i2 % E] = 0;
  __syncthreads();
  if (chunk == 0)
    for (int e = tid; e <= E; e += kPermThreads) offsets[e] = s_base[e];
  const int i = c0 + tid;
  const bool valid = i < n;
  const int e = valid ? __ldg(ids + i) : -1 - lane;
  const unsigned peers = __match_any_sync(0xffffffffu, e);
  const int rank = __popc(peers & ((1u << lane) - 1u));
  if (valid && rank == 0) s_warp_cnt[warp][e] = __popc(peers);
  __syncthreads();
  if (valid) {
    int before = 0;
    for (int w = 0; w < warp; ++w) before += s_warp_cnt[w][e];
    const int pos = s_base[e] + s_before[e] + before + rank;
    perm_src[pos] = i;
    inv[i] = pos;
  }
}

// x_perm[pos] = x[perm_src[pos] / k]; one warp per row, 16 B per lane per step.
__global__ void gather_rows_kernel(const uint16_t* __restrict__ x, const int32_t* __restrict__ perm_src,
                                   int rows, int k, int H, uint16_t* __restrict__ x_perm) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const int tok = perm_src[warp] / k;
  const uint4* src = reinterpret_cast<const uint4*>(x + static_cast<size_t>(tok) * H);
  uint4* dst = reinterpret_cast<uint4*>(x_perm + static_cast<size_t>(warp) * H);
  const int n = H / 8;
  int v = lane;
  for (; v + 96 < n; v += 128) {  // 4 independent 16-byte loads in flight per lane
    const uint4 a = __ldg(src + v), b = __ldg(src + v + 32), c = __ldg(src + v + 64), d = __ldg(src + v + 96);
    dst[v] = a;
    dst[v + 32] = b;
    dst[v + 64] = c;
    dst[v + 96] = d;
  }
  for (; v < n; v += 32) dst[v] = src[v];
}

// y[t,:] = sum_j w[t, ids[t,j]] * sum_s y_part[s][inv[t*k+j], :]. Deterministic order
// (j ascending, then split ascending). grid = (B, ceil(H/1024)), 256 threads x float4.
__global__ void combine_kernel(const float* __restrict__ y_part, int n_split, size_t split_stride,
                               const int32_t* __restrict__ inv, const int32_t* __restrict__ ids,
                               const float* __restrict__ w, int k, int E, int H, float* __restrict__ y) {
  const int t = blockIdx.x;
  const int h = (blockIdx.y * blockDim.x + threadIdx.x) * 4;
  if (h >= H) return;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int j = 0; j < k; ++j) {
    const int slot = t * k + j;
    const float g = w[static_cast<size_t>(t) * E + ids[slot]];
    const float* row = y_part + static_cast<size_t>(inv[slot]) * H + h;
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int p = 0; p < n_split; ++p) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(row + p * split_stride));
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    acc.x += g * s.x; acc.y += g * s.y; acc.z += g * s.z; acc.w += g * s.w;
  }
  *reinterpret_cast<float4*>(y + static_cast<size_t>(t) * H + h) = acc;
}

// n_split == 1 (prefill / tcgen05 path, k + shared <= 16): the same arithmetic as
// combine_kernel (bit-identical), but every slot's index, gate weight and row load is
// issued before the first accumulation, so a thread has k row loads in flight instead
// of one dependent chain per slot (prefill combine: 40 -> ~20 us for 16K rows of 8 KiB).
template <int KMAX>
__global__ void combine_ilp_kernel(const float* __restrict__ y_part, const int32_t* __restrict__ inv,
                                   const int32_t* __restrict__ ids, const float* __restrict__ w, int k, int E,
                                   int H, float* __restrict__ y) {
  const int t = blockIdx.x;
  const int h = (blockIdx.y * blockDim.x + threadIdx.x) * 4;
  if (h >= H) return;
  int r[KMAX];
  float g[KMAX];
  float4 v[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j)
    if (j < k) r[j] = __ldg(inv + t * k + j);
#pragma unroll
  for (int j = 0; j < KMAX; ++j)
    if (j < k) g[j] = __ldg(w + static_cast<size_t>(t) * E + __ldg(ids + t * k + j));
#pragma unroll
  for (int j = 0; j < KMAX; ++j)
    if (j < k) v[j] = __ldg(reinterpret_cast<const float4*>(y_part + static_cast<size_t>(r[j]) * H + h));
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int j = 0; j < KMAX; ++j) {
    if (j < k) {
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
      s.x += v[j].x; s.y += v[j].y; s.z += v[j].z; s.w += v[j].w;
      acc.x += g[j] * s.x; acc.y += g[j] * s.y; acc.z += g[j] * s.z; acc.w += g[j] * s.w;
    }
  }
  *reinterpret_cast<float4*>(y + static_cast<size_t>(t) * H + h) = acc;
}

template <int KMAX, int V>
__global__ void combine_ilp_cols_kernel(const float* __restrict__ y_part, const int32_t* __restrict__ inv,
                                   const int32_t* __restrict__ ids, const float* __restrict__ w, int k, int E,
                                   int H, float* __restrict__ y) {
  // V float4 columns per thread (strided by the CTA width, coalesced per warp): k * V
  // 16-byte row loads in flight per thread
  const int t = blockIdx.x;
  const int h0 = (blockIdx.y * blockDim.x * V + threadIdx.x) * 4;
  int r[KMAX];
  float g[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j)
    if (j < k) r[j] = __ldg(inv + t * k + j);
#pragma unroll
  for (int j = 0; j < KMAX; ++j)
    if (j < k) g[j] = __ldg(w + static_cast<size_t>(t) * E + __ldg(ids + t * k + j));
  float4 v[V][KMAX];
#pragma unroll
  for (int c = 0; c < V; ++c) {
    const int h = h0 + c * blockDim.x * 4;
#pragma unroll
    for (int j = 0; j < KMAX; ++j)
      if (j < k && h < H) v[c][j] = __ldg(reinterpret_cast<const float4*>(y_part + static_cast<size_t>(r[j]) * H + h));
  }
#pragma unroll
  for (int c = 0; c < V; ++c) {
    const int h = h0 + c * blockDim.x * 4;
    if (h >= H) continue;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
      if (j < k) {
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
        s.x += v[c][j].x; s.y += v[c][j].y; s.z += v[c][j].z; s.w += v[c][j].w;
        acc.x += g[j] * s.x; acc.y += g[j] * s.y; acc.z += g[j] * s.z; acc.w += g[j] * s.w;
      }
    }
    *reinterpret_cast<float4*>(y + static_cast<size_t>(t) * H + h) = acc;
  }
}

// Expert parallelism: owner-major virtual ids v = (e % G) * ceil(E/G) + e / G, so a
// counting sort over v groups the routed rows by destination rank, then local expert.
__global__ void ep_remap_kernel(const int32_t* __restrict__ ids, int n, int G, int e_loc, int32_t* __restrict__ v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const int e = ids[i];
    v[i] = (e % G) * e_loc + e / G;
  }
}

// out[d][j] = rows this rank sends to rank d for d's local expert j (from the owner-major
// offsets); out[d][E_loc + j] = this rank's LLaPor-predicted tokens for that expert.
__global__ void ep_pack_counts_kernel(const int32_t* __restrict__ offsets_v, const int32_t* __restrict__ pred,
                                      int E, int G, int e_loc, int32_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= G * e_loc) return;
  const int d = i / e_loc, j = i % e_loc, e = j * G + d;
  out[d * 2 * e_loc + j] = offsets_v[i + 1] - offsets_v[i];
  out[d * 2 * e_loc + e_loc + j] = (pred && e < E) ? pred[e] : 0;
}

__global__ void cast_bf16_kernel(const float* __restrict__ x, int64_t n, uint16_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = f32_to_bf16_rne(x[i]);
}

// SM-driven copy of f32 rows from mapped pinned host memory (zero-copy over PCIe) into
// device memory, with `zero_copies` further zero-filled copies at a stride: the host
// lane's outputs reach y_part without a copy-engine transfer, which would queue behind
// the serial channel's multi-ms expert loads on the same copy engine.
__global__ void rows_from_host_kernel(const float4* __restrict__ src, int64_t n4, float4* __restrict__ dst,
                                      int zero_copies, int64_t zero_stride4) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    dst[i] = src[i];
    for (int z = 1; z <= zero_copies; ++z) dst[i + z * zero_stride4] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// Several row ranges of the same mapped pinned buffer in ONE launch (the host lane's
// experts of a layer): one launch per expert serialised ~3-35 us each behind the PCIe
// traffic of the in-flight expert loads (Qwen3 shape: 8 launches, ~150 us per layer);
// here every range's reads are in flight together. Rows [row0, row0 + m) of src/dst.
constexpr int kMaxRowRanges = 128;
struct RowRanges {
  int n;
  int row0[kMaxRowRanges];
  int m[kMaxRowRanges];
  int start[kMaxRowRanges + 1];  // prefix of m: flat row index -> range
};

__global__ void rows_from_host_ranges_kernel(const float4* __restrict__ src, float4* __restrict__ dst, int H4,
                                             const __grid_constant__ RowRanges r, int zero_copies,
                                             int64_t zero_stride4) {
  const int64_t total = static_cast<int64_t>(r.start[r.n]) * H4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int flat = static_cast<int>(i / H4), c = static_cast<int>(i - static_cast<int64_t>(flat) * H4);
    int lo = 0, hi = r.n - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (r.start[mid] <= flat) lo = mid;
      else hi = mid - 1;
    }
    const int64_t o = static_cast<int64_t>(r.row0[lo] + flat - r.start[lo]) * H4 + c;
    dst[o] = src[o];
    for (int z = 1; z <= zero_copies; ++z) dst[o + z * zero_stride4] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// Shared experts (DeepSeek-style, always active, gate weight 1): appended as virtual
// experts E..E+S-1 so permute / FFN / combine treat them like routed ones.
__global__ void append_shared_kernel(const int32_t* __restrict__ ids, const float* __restrict__ w, int B, int k,
                                     int E, int S, int32_t* __restrict__ ids_ext, float* __restrict__ w_ext,
                                     int32_t* __restrict__ counts) {
  const int kt = k + S, et = E + S;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < B * et; i += gridDim.x * blockDim.x) {
    const int t = i / et, c = i % et;
    w_ext[i] = c < E ? w[static_cast<size_t>(t) * E + c] : 1.0f;
    if (c < kt) ids_ext[static_cast<size_t>(t) * kt + c] = c < k ? ids[static_cast<size_t>(t) * k + c] : E + (c - k);
  }
  if (counts && blockIdx.x == 0 && threadIdx.x < S) counts[E + threadIdx.x] = B;
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" {

ps_status ps_ep_pack_counts(const int32_t* offsets_v, const int32_t* pred, int E, int G, int32_t* out,
                            void* stream) {
  return guarded([&] {
    require(offsets_v && out && E >= 1 && G >= 1, "ps_ep_pack_counts: bad arguments");
    const int e_loc = (E + G - 1) / G;
    ep_pack_counts_kernel<<<(G * e_loc + 127) / 128, 128, 0, as_stream(stream)>>>(offsets_v, pred, E, G, e_loc, out);
    PS_LAUNCH_CHECK("ep_pack_counts_kernel");
  });
}

ps_status ps_cast_bf16(const float* x, int64_t n, uint16_t* out, void* stream) {
  return guarded([&] {
    require(n >= 0 && (n == 0 || (x && out)), "ps_cast_bf16: bad arguments");
    if (n == 0) return;
    const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 4 * 148));
    cast_bf16_kernel<<<grid, 256, 0, as_stream(stream)>>>(x, n, out);
    PS_LAUNCH_CHECK("cast_bf16_kernel");
  });
}

ps_status ps_rows_from_host(const float* host_src, int64_t n, float* dst, int zero_copies, int64_t zero_stride,
                            void* stream) {
  return guarded([&] {
    require(n >= 0 && zero_copies >= 0 && n % 4 == 0 && zero_stride % 4 == 0 && (n == 0 || (host_src && dst)),
            "ps_rows_from_host: bad arguments");
    // zero-filled copies must not overlap the copied range (or each other)
    require(zero_copies == 0 || zero_stride >= n, "ps_rows_from_host: zero_stride must be >= n");
    if (n == 0) return;
    void* dev_src = nullptr;
    PS_CUDA(cudaHostGetDevicePointer(&dev_src, const_cast<float*>(host_src), 0));
    require((reinterpret_cast<uintptr_t>(dev_src) | reinterpret_cast<uintptr_t>(dst)) % 16 == 0,
            "ps_rows_from_host: 16-byte alignment");
    const int64_t n4 = n / 4;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n4 + 255) / 256, 148)));
    rows_from_host_kernel<<<grid, 256, 0, as_stream(stream)>>>(static_cast<const float4*>(dev_src), n4,
                                                               reinterpret_cast<float4*>(dst), zero_copies,
                                                               zero_stride / 4);
    PS_LAUNCH_CHECK("rows_from_host_kernel");
  });
}

ps_status ps_rows_from_host_ranges(const float* host_base, const int32_t* row0, const int32_t* m, int n_ranges,
                                   int H, float* dst, int zero_copies, int64_t zero_stride, void* stream) {
  return guarded([&] {
    require(n_ranges >= 0 && n_ranges <= kMaxRowRanges && H > 0 && H % 4 == 0 && zero_copies >= 0 &&
                zero_stride % 4 == 0 && (n_ranges == 0 || (host_base && row0 && m && dst)),
            "ps_rows_from_host_ranges: bad arguments (<= 128 ranges, H % 4 == 0)");
    if (n_ranges == 0) return;
    RowRanges r{};
    r.n = n_ranges;
    int64_t max_end = 0;
    for (int i = 0; i < n_ranges; ++i) {
      require(row0[i] >= 0 && m[i] >= 0, "ps_rows_from_host_ranges: negative range");
      r.row0[i] = row0[i];
      r.m[i] = m[i];
      r.start[i + 1] = r.start[i] + m[i];
      max_end = std::max<int64_t>(max_end, static_cast<int64_t>(row0[i]) + m[i]);
    }
    // zero-filled copies must not overlap any copied row
    require(zero_copies == 0 || zero_stride >= max_end * H, "ps_rows_from_host_ranges: zero_stride too small");
    if (r.start[n_ranges] == 0) return;
    void* dev_src = nullptr;
    PS_CUDA(cudaHostGetDevicePointer(&dev_src, const_cast<float*>(host_base), 0));
    require((reinterpret_cast<uintptr_t>(dev_src) | reinterpret_cast<uintptr_t>(dst)) % 16 == 0,
            "ps_rows_from_host_ranges: 16-byte alignment");
    const int H4 = H / 4;
    const int64_t total = static_cast<int64_t>(r.start[n_ranges]) * H4;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148)));
    rows_from_host_ranges_kernel<<<grid, 256, 0, as_stream(stream)>>>(static_cast<const float4*>(dev_src),
                                                                       reinterpret_cast<float4*>(dst), H4, r,
                                                                       zero_copies, zero_stride / 4);
    PS_LAUNCH_CHECK("rows_from_host_ranges_kernel");
  });
}

ps_status ps_append_shared(const int32_t* ids, const float* weights, int B, int k, int E, int S,
                           int32_t* ids_ext, float* weights_ext, int32_t* counts, void* stream) {
  return guarded([&] {
    require(B >= 0 && k >= 1 && E >= 1 && S >= 1 && S <= 32 && ids && weights && ids_ext && weights_ext,
            "ps_append_shared: bad arguments");
    const int n = B * (E + S);
    append_shared_kernel<<<std::max(1, std::min((n + 255) / 256, 148)), 256, 0, as_stream(stream)>>>(
        ids, weights, B, k, E, S, ids_ext, weights_ext, counts);
    PS_LAUNCH_CHECK("append_shared_kernel");
  });
}

ps_status ps_gather_rows(const uint16_t* x, const int32_t* idx, int n, int div, int H, uint16_t* out,
                         void* stream) {
  return guarded([&] {
    require(n >= 0 && div >= 1 && H % 8 == 0 && x && idx && out, "ps_gather_rows: bad arguments");
    if (n == 0) return;
    gather_rows_kernel<<<(n * 32 + 255) / 256, 256, 0, as_stream(stream)>>>(x, idx, n, div, H, out);
    PS_LAUNCH_CHECK("gather_rows_kernel");
  });
}

ps_status ps_ep_remap_ids(const int32_t* ids, int n, int E, int G, int32_t* vids, void* stream) {
  return guarded([&] {
    require(n >= 0 && E >= 1 && G >= 1 && ids && vids, "ps_ep_remap_ids: bad arguments");
    if (n == 0) return;
    ep_remap_kernel<<<(n + 255) / 256, 256, 0, as_stream(stream)>>>(ids, n, G, (E + G - 1) / G, vids);
    PS_LAUNCH_CHECK("ep_remap_kernel");
  });
}

ps_status ps_permute(const int32_t* ids, int B, int k, int E, int32_t* offsets, int32_t* perm_src,
                     int32_t* inv, const uint16_t* x, int H, uint16_t* x_perm, void* stream) {
  return guarded([&] {
    require(B >= 0 && k >= 1 && E >= 1 && E <= kMaxE, "ps_permute: shape out of range");
    require(static_cast<int64_t>(B) * k <= (1 << 20), "ps_permute: too many assignments");
    require(ids && offsets && perm_src && inv, "ps_permute: null output");
    cudaStream_t s = as_stream(stream);
    const int n = B * k;
    const int chunks = (n + kPermThreads - 1) / kPermThreads;
    if (chunks <= 2 || chunks > 128) {
      permute_index_kernel<<<1, kPermThreads, 0, s>>>(ids, n, E, offsets, perm_src, inv);
      PS_LAUNCH_CHECK("permute_index_kernel");
    } else {  // prefill chunks: one CTA per 1024 ids
      permute_chunks_kernel<<<chunks, kPermThreads, 0, s>>>(ids, n, E, offsets, perm_src, inv);
      PS_LAUNCH_CHECK("permute_chunks_kernel");
    }
    if (x && x_perm && B > 0) {
      require(H % 8 == 0, "ps_permute: gather needs H % 8 == 0");
      const int rows = B * k;
      gather_rows_kernel<<<(rows * 32 + 255) / 256, 256, 0, s>>>(x, perm_src, rows, k, H, x_perm);
      PS_LAUNCH_CHECK("gather_rows_kernel");
    }
  });
}

ps_status ps_combine(const float* y_part, int n_split, const int32_t* inv, const int32_t* ids,
                     const float* weights, int B, int k, int E, int H, float* y, void* stream) {
  return guarded([&] {
    require(B >= 0 && k >= 1 && E >= 1 && n_split >= 1 && H % 4 == 0, "ps_combine: bad shape (H % 4 == 0)");
    if (B == 0) return;
    dim3 grid(B, (H / 4 + 255) / 256);
    if (n_split == 1 && k <= 2) {  // Mixtral-like: 4 columns per thread, 8 row loads in flight
      dim3 g4(B, (H / 4 + 1023) / 1024);
      combine_ilp_cols_kernel<2, 4><<<g4, 256, 0, as_stream(stream)>>>(y_part, inv, ids, weights, k, E, H, y);
    } else if (n_split == 1 && k <= 8) {  // (the column variant: 90 registers, 2x slower at k = 8)
      combine_ilp_kernel<8><<<grid, 256, 0, as_stream(stream)>>>(y_part, inv, ids, weights, k, E, H, y);
    } else if (n_split == 1 && k <= 16) {
      combine_ilp_kernel<16><<<grid, 256, 0, as_stream(stream)>>>(y_part, inv, ids, weights, k, E, H, y);
    } else {
      combine_kernel<<<grid, 256, 0, as_stream(stream)>>>(y_part, n_split, static_cast<size_t>(B) * k * H, inv,
                                                          ids, weights, k, E, H, y);
    }
    PS_LAUNCH_CHECK("combine_kernel");
  });
}

}  // extern "C"
