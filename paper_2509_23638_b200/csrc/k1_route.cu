// K1 — fused router: gate GEMV (fp32 accumulate) + zipf bias + kappa-follow override +
// softmax + top-k + per-expert histogram (+ fused bf16 cast of x for the expert FFN).
//
// Replaces the per-(token, layer) router loop of the reference trace generator
// (workload.cpp:176-202) and aggregate_layer_loads (workload.cpp:283-288).
// One warp per token; the gate matrix [E,H] (<= 1 MiB) is re-read from L1/L2 by every
// warp, x [H] once from HBM: HBM-bound at B*H*4 + E*H*4 bytes per launch.
//
// Top-k ranks the fp32 softmax WEIGHTS with the reference's tie-break (value desc,
// lower index first), exactly what topk_indices does on the same numbers, so the
// returned ids are bit-exact against topk_indices(weights) (tests/test_gpu_ops.py::test_route_topk_parity).
#include "device_common.cuh"
#include "permute_device.cuh"

namespace ps {
namespace {

constexpr int kWarps = 8;  // warps per token, splitting H
constexpr int kMaxE = 256;
constexpr int kMaxK = 16;
constexpr int kETile = 8;  // experts per register tile (decode); prefill chunks use 4 x 8 tokens

// Per-token tail of the router (one warp): kappa override, softmax, top-k, histogram.
__device__ __forceinline__ void finish_token_impl(int warp, int b0, float* lg, const uint8_t* __restrict__ follow,
                                                  const int32_t* __restrict__ prev_ids, int prev_k, int E, int k,
                                                  float* __restrict__ logits_out, float* __restrict__ weights_out,
                                                  int32_t* __restrict__ ids_out, int32_t* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int b = b0 + warp;

  // kappa-follow override: logits[(prev_top1+1) % E] = max + 1 (workload.cpp:183-188).
  if (follow && prev_ids && follow[b]) {
    float m = -INFINITY;
    for (int e = lane; e < E; e += 32) m = fmaxf(m, lg[e]);
    m = warp_max(m);
    const int target = (prev_ids[static_cast<size_t>(b) * prev_k] + 1) % E;
    __syncwarp();
    if (lane == 0) lg[target] = m + 1.0f;
    __syncwarp();
  }

  // Softmax (workload.cpp:190-195).
  float m = -INFINITY;
  for (int e = lane; e < E; e += 32) m = fmaxf(m, lg[e]);
  m = warp_max(m);
  float z = 0.f;
  for (int e = lane; e < E; e += 32) z += expf(lg[e] - m);
  z = warp_sum(z);
  const float inv_z = 1.0f / z;
  float w_local[kMaxE / 32];
#pragma unroll
  for (int i = 0; i < kMaxE / 32; ++i) {
    const int e = lane + 32 * i;
    w_local[i] = e < E ? expf(lg[e] - m) * inv_z : -INFINITY;
    if (e < E) {
      if (logits_out) logits_out[static_cast<size_t>(b) * E + e] = lg[e];
      if (weights_out) weights_out[static_cast<size_t>(b) * E + e] = w_local[i];
    }
  }

  // Top-k over the weights: k rounds of warp arg-max (ties -> lower index).
  for (int r = 0; r < k; ++r) {
    float bv = -INFINITY;
    int bi = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < kMaxE / 32; ++i) {
      const int e = lane + 32 * i;
      if (e < E && (w_local[i] > bv || (w_local[i] == bv && e < bi))) {
        bv = w_local[i];
        bi = e;
      }
    }
    warp_argmax(bv, bi);
    if (lane == 0) {
      ids_out[static_cast<size_t>(b) * k + r] = bi;
      if (counts) atomicAdd(counts + bi, 1);
    }
#pragma unroll
    for (int i = 0; i < kMaxE / 32; ++i)
      if (lane + 32 * i == bi) w_local[i] = -INFINITY;  // remove from later rounds
  }
}

// One CTA per TB tokens: the 8 warps split H (latency: a Mixtral token needs 4 float4
// steps per lane instead of 32) and every gate float4 loaded is applied to all TB
// tokens (TB = 1 for decode batches, 8 for prefill chunks: 8x less L2 gate traffic).
// Per-warp partial logits are summed in shared memory in fixed warp order
// (deterministic and independent of TB); warp t then finishes token t: kappa override,
// softmax, top-k, histogram. kFused: the last CTA also runs the K2 index pass.
struct FusedPermute {  // K2 index pass run by the last CTA of a decode route launch
  int32_t* offsets;
  int32_t* perm_src;
  int32_t* inv;
  int* done;  // launch ticket counter (zero between launches; the last CTA resets it)
};

template <int TB, bool kFused>
__global__ void __launch_bounds__(kWarps * 32, TB >= 8 ? 2 : 1)
route_kernel(const float* __restrict__ x, const float* __restrict__ gate, const float* __restrict__ bias,
             const uint8_t* __restrict__ follow, const int32_t* __restrict__ prev_ids, int prev_k,
             int B, int H, int E, int k, float sqrt_h, float* __restrict__ logits_out,
             float* __restrict__ weights_out, int32_t* __restrict__ ids_out,
             int32_t* __restrict__ counts, uint16_t* __restrict__ x_bf16, FusedPermute fp) {
  // per-warp partial logits [kWarps][TB][E] (dynamic: E * TB * 32 B) + logits [TB][kMaxE]
  extern __shared__ float s_dyn[];
  __shared__ float s_logit[TB][kMaxE];
  auto s_part = [&](int w, int t, int e) -> float& { return s_dyn[(w * TB + t) * E + e]; };
  // TB = 8 (prefill chunks): 4 experts x 8 tokens per register tile and one float4 step
  // in flight (~100 registers, 2 CTAs per SM, all 8 warps busy in the per-token tail);
  // the per-lane accumulation order is the same as TB = 1 / 4 (increasing h).
  constexpr int ET = TB >= 8 ? 4 : kETile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b0 = blockIdx.x * TB;
  const int nt = min(TB, B - b0);
  const bool vec = (H & 3) == 0;

  // Gate GEMV partials: warp w owns H slice [w*hs, (w+1)*hs), kETile experts at a time.
  // Vector path: kU float4 steps per lane in flight together (latency-bound at decode),
  // and the x values loaded for the first expert tile are also written out as bf16
  // (fused cast for K3).
  constexpr int kU = TB >= 8 ? 1 : 2;
  const int hs = vec ? ((H / 4 + kWarps - 1) / kWarps) * 4 : (H + kWarps - 1) / kWarps;
  const int h_lo = min(H, warp * hs), h_hi = min(H, h_lo + hs);
  // Prefill fast path (whole token tile, whole expert tiles, every warp slice a multiple of
  // 128 floats): no per-element bounds selects, row pointers hoisted. Same per-lane
  // accumulation order and dot-product expression as the general loop below (bit-identical).
  const bool fast = TB >= 8 && vec && nt == TB && E % ET == 0 && (h_hi - h_lo) % 128 == 0;
  if (fast) {
    const float* xrow = x + static_cast<size_t>(b0) * H;
    for (int e0 = 0; e0 < E; e0 += ET) {
      float acc[TB][ET];
#pragma unroll
      for (int t = 0; t < TB; ++t)
#pragma unroll
        for (int j = 0; j < ET; ++j) acc[t][j] = 0.f;
      const float* grow = gate + static_cast<size_t>(e0) * H;
      for (int h = h_lo + lane * 4; h < h_hi; h += 128) {
        float4 xv[TB], g[ET];
#pragma unroll
        for (int t = 0; t < TB; ++t) xv[t] = *reinterpret_cast<const float4*>(xrow + static_cast<size_t>(t) * H + h);
#pragma unroll
        for (int j = 0; j < ET; ++j) g[j] = __ldg(reinterpret_cast<const float4*>(grow + static_cast<size_t>(j) * H + h));
#pragma unroll
        for (int j = 0; j < ET; ++j)
#pragma unroll
          for (int t = 0; t < TB; ++t)
            acc[t][j] += g[j].x * xv[t].x + g[j].y * xv[t].y + g[j].z * xv[t].z + g[j].w * xv[t].w;
        if (x_bf16 && e0 == 0) {
#pragma unroll
          for (int t = 0; t < TB; ++t) {
            uint2 o;
            o.x = (uint32_t)f32_to_bf16_rne(xv[t].x) | ((uint32_t)f32_to_bf16_rne(xv[t].y) << 16);
            o.y = (uint32_t)f32_to_bf16_rne(xv[t].z) | ((uint32_t)f32_to_bf16_rne(xv[t].w) << 16);
            *reinterpret_cast<uint2*>(x_bf16 + static_cast<size_t>(b0 + t) * H + h) = o;
          }
        }
      }
      if constexpr (TB * ET == 32) {
        float v[32];
#pragma unroll
        for (int t = 0; t < TB; ++t)
#pragma unroll
          for (int j = 0; j < ET; ++j) v[t * ET + j] = acc[t][j];
        const float sum = warp_transpose_sum<32>(v);
        s_part(warp, lane / ET, e0 + lane % ET) = sum;
      }
    }
  }
  for (int e0 = 0; e0 < (fast ? 0 : E); e0 += ET) {
    float acc[TB][ET];
#pragma unroll
    for (int t = 0; t < TB; ++t)
#pragma unroll
      for (int j = 0; j < ET; ++j) acc[t][j] = 0.f;
    if (vec) {
      for (int hb = h_lo + lane * 4; hb < h_hi; hb += 128 * kU) {
        float4 xv[kU][TB], g[kU][ET];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int h = hb + 128 * u;
          const bool hin = h < h_hi;
#pragma unroll
          for (int t = 0; t < TB; ++t)
            xv[u][t] = hin && t < nt ? *reinterpret_cast<const float4*>(x + static_cast<size_t>(b0 + t) * H + h)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int j = 0; j < ET; ++j)
            g[u][j] = hin && e0 + j < E ? __ldg(reinterpret_cast<const float4*>(gate + static_cast<size_t>(e0 + j) * H + h))
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
#pragma unroll
          for (int j = 0; j < ET; ++j)
#pragma unroll
            for (int t = 0; t < TB; ++t)
              acc[t][j] += g[u][j].x * xv[u][t].x + g[u][j].y * xv[u][t].y + g[u][j].z * xv[u][t].z +
                           g[u][j].w * xv[u][t].w;
          const int h = hb + 128 * u;
          if (x_bf16 && e0 == 0 && h < h_hi) {
#pragma unroll
            for (int t = 0; t < TB; ++t)
              if (t < nt) {
                uint2 o;
                o.x = (uint32_t)f32_to_bf16_rne(xv[u][t].x) | ((uint32_t)f32_to_bf16_rne(xv[u][t].y) << 16);
                o.y = (uint32_t)f32_to_bf16_rne(xv[u][t].z) | ((uint32_t)f32_to_bf16_rne(xv[u][t].w) << 16);
                *reinterpret_cast<uint2*>(x_bf16 + static_cast<size_t>(b0 + t) * H + h) = o;
              }
          }
        }
      }
    } else {
      if (x_bf16 && e0 == 0)
        for (int t = 0; t < nt; ++t)
          for (int h = h_lo + lane; h < h_hi; h += 32)
            x_bf16[static_cast<size_t>(b0 + t) * H + h] = f32_to_bf16_rne(x[static_cast<size_t>(b0 + t) * H + h]);
      for (int h = h_lo + lane; h < h_hi; h += 32) {
#pragma unroll
        for (int j = 0; j < ET; ++j) {
          if (e0 + j >= E) continue;
          const float g = __ldg(gate + static_cast<size_t>(e0 + j) * H + h);
#pragma unroll
          for (int t = 0; t < TB; ++t)
            if (t < nt) acc[t][j] += g * x[static_cast<size_t>(b0 + t) * H + h];
        }
      }
    }
    if constexpr (TB * ET == 32) {
      // All 32 warp sums at once (31 shuffles instead of 160): warp_transpose_sum<32> pairs
      // lanes at distance 16, 8, 4, 2, 1 like warp_sum, so every sum is bit-identical to
      // the decode instantiation's; lane i ends up with value i = (token i / ET, expert i % ET).
      float v[32];
#pragma unroll
      for (int t = 0; t < TB; ++t)
#pragma unroll
        for (int j = 0; j < ET; ++j) v[t * ET + j] = acc[t][j];
      const float sum = warp_transpose_sum<32>(v);
      const int t = lane / ET, j = lane % ET;
      if (t < TB && e0 + j < E) s_part(warp, t, e0 + j) = sum;
    } else {
#pragma unroll
      for (int t = 0; t < TB; ++t)
#pragma unroll
        for (int j = 0; j < ET; ++j) {
          float sum = warp_sum(acc[t][j]);
          if (lane == 0 && e0 + j < E) s_part(warp, t, e0 + j) = sum;
        }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nt * E; i += kWarps * 32) {
    const int t = i / E, e = i % E;
    float sum = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) sum += s_part(w, t, e);
    s_logit[t][e] = sum * sqrt_h + (bias ? bias[e] : 0.f);
  }
  __syncthreads();
  if (warp < nt) finish_token_impl(warp, b0, s_logit[warp], follow, prev_ids, prev_k, E, k, logits_out, weights_out,
                                   ids_out, counts);
  if constexpr (kFused) {
    // Last CTA to finish runs the K2 index pass over all B*k ids (one launch instead of
    // two on the decode critical path). Release: ids stores -> fence -> ticket.
    __shared__ int s_last;
    __shared__ int s_base[kPermMaxE + 1];
    __shared__ int s_warp_cnt[kWarps][kPermMaxE];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(fp.done, 1) == static_cast<int>(gridDim.x) - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();  // acquire side: every CTA's ids are visible (read through L2)
    permute_block<kWarps * 32, true>(ids_out, B * k, E, fp.offsets, fp.perm_src, fp.inv, s_base, s_warp_cnt);
    if (threadIdx.x == 0) *fp.done = 0;
  }
}

// Decode route + permute with many experts (E >= 64): the token's experts are split over
// E/32 CTAs (B * E/32 CTAs instead of B), each computing 32 logits exactly as
// route_kernel<1> does (same per-warp H slice, same per-lane order, warp_sum, warp sums
// in fixed order: bitwise the same logits); the last CTA of a token (per-token ticket)
// gathers its logits and finishes it (kappa override, softmax, top-k); the last CTA of
// the launch permutes. The logits go through `weights` (overwritten by the softmax
// weights). Qwen3 shape (E = 128, B = 32): 32 CTAs each streaming the whole 1 MiB gate
// matrix took ~27 us.
constexpr int kSplitE = 32;

__global__ void __launch_bounds__(kWarps * 32)
route_split_kernel(const float* __restrict__ x, const float* __restrict__ gate, const float* __restrict__ bias,
                   const uint8_t* __restrict__ follow, const int32_t* __restrict__ prev_ids, int prev_k, int B, int H,
                   int E, int k, float sqrt_h, float* __restrict__ weights_out, int32_t* __restrict__ ids_out,
                   uint16_t* __restrict__ x_bf16, FusedPermute fp, int* __restrict__ tok_cnt) {
  __shared__ float s_part[kWarps][kSplitE];
  __shared__ float s_logit[kMaxE];
  __shared__ int s_flag;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int groups = (E + kSplitE - 1) / kSplitE;
  const int b = blockIdx.x / groups, grp = blockIdx.x - b * groups;
  const int e_lo = grp * kSplitE, e_hi = min(E, e_lo + kSplitE);
  constexpr int kU = 2;
  const int hs = ((H / 4 + kWarps - 1) / kWarps) * 4;
  const int h_lo = min(H, warp * hs), h_hi = min(H, h_lo + hs);
  for (int e0 = e_lo; e0 < e_hi; e0 += kETile) {
    float acc[kETile];
#pragma unroll
    for (int j = 0; j < kETile; ++j) acc[j] = 0.f;
    for (int hb = h_lo + lane * 4; hb < h_hi; hb += 128 * kU) {
      float4 xv[kU], g[kU][kETile];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int h = hb + 128 * u;
        const bool hin = h < h_hi;
        xv[u] = hin ? *reinterpret_cast<const float4*>(x + static_cast<size_t>(b) * H + h) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int j = 0; j < kETile; ++j)
          g[u][j] = hin && e0 + j < E ? __ldg(reinterpret_cast<const float4*>(gate + static_cast<size_t>(e0 + j) * H + h))
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
#pragma unroll
        for (int j = 0; j < kETile; ++j)
          acc[j] += g[u][j].x * xv[u].x + g[u][j].y * xv[u].y + g[u][j].z * xv[u].z + g[u][j].w * xv[u].w;
        const int h = hb + 128 * u;
        if (x_bf16 && e0 == 0 && h < h_hi) {
          uint2 o;
          o.x = (uint32_t)f32_to_bf16_rne(xv[u].x) | ((uint32_t)f32_to_bf16_rne(xv[u].y) << 16);
          o.y = (uint32_t)f32_to_bf16_rne(xv[u].z) | ((uint32_t)f32_to_bf16_rne(xv[u].w) << 16);
          *reinterpret_cast<uint2*>(x_bf16 + static_cast<size_t>(b) * H + h) = o;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < kETile; ++j) {
      const float sum = warp_sum(acc[j]);
      if (lane == 0 && e0 + j < e_hi) s_part[warp][e0 + j - e_lo] = sum;
    }
  }
  __syncthreads();
  if (threadIdx.x < e_hi - e_lo) {
    float sum = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) sum += s_part[w][threadIdx.x];
    const int e = e_lo + threadIdx.x;
    weights_out[static_cast<size_t>(b) * E + e] = sum * sqrt_h + (bias ? bias[e] : 0.f);
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    s_flag = atomicAdd(tok_cnt + b, 1) == groups - 1;
    if (s_flag) tok_cnt[b] = 0;  // every group of this token has arrived
  }
  __syncthreads();
  if (s_flag) {  // this token's last CTA: all of its logits are in `weights` (L2)
    __threadfence();
    for (int e = threadIdx.x; e < E; e += kWarps * 32) s_logit[e] = __ldcg(weights_out + static_cast<size_t>(b) * E + e);
    __syncthreads();
    if (warp == 0)
      finish_token_impl(0, b, s_logit, follow, prev_ids, prev_k, E, k, nullptr, weights_out, ids_out, nullptr);
  }
  // the launch's last CTA permutes all B*k ids (as route_kernel<1, true>)
  __shared__ int s_last;
  __shared__ int s_base[kPermMaxE + 1];
  __shared__ int s_warp_cnt[kWarps][kPermMaxE];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(fp.done, 1) == static_cast<int>(gridDim.x) - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  permute_block<kWarps * 32, true>(ids_out, B * k, E, fp.offsets, fp.perm_src, fp.inv, s_base, s_warp_cnt);
  if (threadIdx.x == 0) *fp.done = 0;
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" ps_status ps_route_topk(const float* x, const float* gate, const float* bias,
                                   const uint8_t* follow, const int32_t* prev_ids, int prev_k, int B,
                                   int H, int E, int k, float* logits, float* weights, int32_t* ids,
                                   int32_t* counts, uint16_t* x_bf16, void* stream) {
  return guarded([&] {
    require(B >= 0 && H >= 1 && E >= 1 && E <= kMaxE && k >= 1 && k <= E && k <= kMaxK,
            "ps_route_topk: shape out of range (E <= 256, 1 <= k <= min(E,16))");
    require(x && gate && ids, "ps_route_topk: null input");
    require(!(follow && prev_ids) || prev_k >= 1, "ps_route_topk: prev_k must be >= 1");
    require((reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(gate) & 15) == 0,
            "ps_route_topk: x and gate must be 16-byte aligned");
    cudaStream_t s = as_stream(stream);
    if (counts) PS_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * E, s));
    if (B == 0) return;
    const float sqrt_h = static_cast<float>(std::sqrt(static_cast<double>(H)));
    if (B <= 64) {
      route_kernel<1, false><<<B, kWarps * 32, kWarps * 1 * E * 4, s>>>(
          x, gate, bias, follow, prev_ids, prev_k, B, H, E, k, sqrt_h, logits, weights, ids, counts, x_bf16,
          FusedPermute{});
    } else {
      static bool attr = false;
      if (!attr) {  // E = 256: 64 KiB of partials
        PS_CUDA(cudaFuncSetAttribute(route_kernel<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kWarps * 8 * kMaxE * 4));
        attr = true;
      }
      route_kernel<8, false><<<(B + 7) / 8, kWarps * 32, kWarps * 8 * E * 4, s>>>(
          x, gate, bias, follow, prev_ids, prev_k, B, H, E, k, sqrt_h, logits, weights, ids, counts, x_bf16,
          FusedPermute{});
    }
    PS_LAUNCH_CHECK("route_kernel");
  });
}

extern "C" ps_status ps_route_permute(const float* x, const float* gate, const float* bias, const uint8_t* follow,
                                      const int32_t* prev_ids, int prev_k, int B, int H, int E, int k,
                                      float* weights, int32_t* ids, uint16_t* x_bf16, int32_t* offsets,
                                      int32_t* perm_src, int32_t* inv, int32_t* workspace, void* stream) {
  return guarded([&] {
    require(B >= 1 && B <= 64 && H >= 1 && E >= 1 && E <= kMaxE && k >= 1 && k <= E && k <= kMaxK,
            "ps_route_permute: decode shapes only (1 <= B <= 64, E <= 256, 1 <= k <= min(E,16))");
    require(x && gate && ids && offsets && perm_src && inv && workspace, "ps_route_permute: null argument");
    require(!(follow && prev_ids) || prev_k >= 1, "ps_route_permute: prev_k must be >= 1");
    require((reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(gate) & 15) == 0,
            "ps_route_permute: x and gate must be 16-byte aligned");
    const float sqrt_h = static_cast<float>(std::sqrt(static_cast<double>(H)));
    if (E >= 2 * kSplitE && (H & 3) == 0) {
      const int groups = (E + kSplitE - 1) / kSplitE;
      route_split_kernel<<<B * groups, kWarps * 32, 0, as_stream(stream)>>>(
          x, gate, bias, follow, prev_ids, prev_k, B, H, E, k, sqrt_h, weights, ids, x_bf16,
          FusedPermute{offsets, perm_src, inv, workspace}, workspace + 1);
      PS_LAUNCH_CHECK("route_split_kernel");
      return;
    }
    route_kernel<1, true><<<B, kWarps * 32, kWarps * 1 * E * 4, as_stream(stream)>>>(
        x, gate, bias, follow, prev_ids, prev_k, B, H, E, k, sqrt_h, nullptr, weights, ids, nullptr, x_bf16,
        FusedPermute{offsets, perm_src, inv, workspace});
    PS_LAUNCH_CHECK("route_kernel<fused permute>");
  });
}
