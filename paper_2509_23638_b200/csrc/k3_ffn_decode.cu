// K3 (decode path) — grouped SwiGLU expert FFN as an HBM-streaming GEMV.
//
// No reference code exists for the expert FFN; the op is
// y = W_down(SiLU(W_gate x) * (W_up x)) over the experts a
// decode step activates, with per-expert token counts m_e <= 64.
//
// Design (HBM-bound: algorithmic bytes = sum_e 3*H*F*2): each warp owns a 16-row
// tile of one expert's weight matrix and streams it once with 128-bit
// L1::no_allocate loads; the m_e token vectors are the 8-wide N side of
// mma.sync.m16n8k16 (bf16 in, fp32 accumulate). Because a dot product is invariant
// under a common permutation of K, each lane feeds the A fragment straight from its
// own coalesced 16-byte load (rows g and g+8, elements 8t..8t+7 of a 32-wide K block)
// and loads the matching 16 bytes of x for the B fragment — no shared-memory staging,
// no swizzle, ~16 loads in flight per lane.
//   gate_up: tile = 16 F-rows of W_gate and the same rows of W_up; epilogue
//            h = SiLU(g)*u -> bf16 [perm_row, F].
//   down:    tile = 16 H-rows of W_down x one K split of F; fp32 partials
//            y_part[split][perm_row][H], summed in fixed order by K2's combine.
// Deterministic (no atomics). Tail: rows >= rows_total and K beyond K are zero-filled.
#include <algorithm>
#include <vector>

#include "device_common.cuh"

namespace ps {
namespace {

constexpr int kMaxGroup = 120;
constexpr int kWarpsPerCta = 4;
constexpr int kUnroll = 4;

struct FfnLaunch {
  int n;
  int token_chunk;                 // tokens per work item (8 * NT)
  int tile_start[kMaxGroup + 1];   // prefix of warp work items per entry
  int expert[kMaxGroup];
  int tok_chunks[kMaxGroup];       // ceil(m_e / token_chunk)
  const uint16_t* slab[kMaxGroup];
};

__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                               uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// A 16x32 K-block of two rows per lane (g, g+8) times an 8-token group.
__device__ __forceinline__ void mma_block(float (&c)[4], const uint4& r0, const uint4& r8, const uint4& xv) {
  mma_bf16_16816(c, r0.x, r8.x, r0.y, r8.y, xv.x, xv.y);
  mma_bf16_16816(c, r0.z, r8.z, r0.w, r8.w, xv.z, xv.w);
}

__device__ __forceinline__ int find_entry(const FfnLaunch& g, int w) {
  int lo = 0, hi = g.n - 1;
  while (lo < hi) {  // largest i with tile_start[i] <= w
    int mid = (lo + hi + 1) >> 1;
    if (g.tile_start[mid] <= w) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ uint4 zero4() { return make_uint4(0u, 0u, 0u, 0u); }

template <int NT>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
ffn_gateup_kernel(const __grid_constant__ FfnLaunch g, const int32_t* __restrict__ offsets,
                  const int32_t* __restrict__ perm_src, int k, const uint16_t* __restrict__ x, int H, int F,
                  uint16_t* __restrict__ h_out) {
  const int w = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
  if (w >= g.tile_start[g.n]) return;
  const int lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
  const int i = find_entry(g, w);
  const int local = w - g.tile_start[i];
  const int chunk = local % g.tok_chunks[i];
  const int f0 = (local / g.tok_chunks[i]) * 16;
  const int e = g.expert[i];
  const int row0 = offsets[e];
  const int m = offsets[e + 1] - row0;
  const int tb = chunk * g.token_chunk;
  if (tb >= m) return;  // expert not routed this step (or chunk beyond its rows)

  const uint16_t* wg = g.slab[i];
  const uint16_t* wu = wg + static_cast<size_t>(F) * H;
  const bool ok0 = f0 + gid < F, ok8 = f0 + gid + 8 < F;
  const uint16_t* g0 = wg + static_cast<size_t>(ok0 ? f0 + gid : 0) * H;
  const uint16_t* g8 = wg + static_cast<size_t>(ok8 ? f0 + gid + 8 : 0) * H;
  const uint16_t* u0 = wu + static_cast<size_t>(ok0 ? f0 + gid : 0) * H;
  const uint16_t* u8 = wu + static_cast<size_t>(ok8 ? f0 + gid + 8 : 0) * H;

  const uint16_t* xr[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const int t = tb + 8 * j + gid;
    xr[j] = t < m ? x + static_cast<size_t>(perm_src[row0 + t] / k) * H : nullptr;
  }

  float cg[NT][4], cu[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) cg[j][q] = cu[j][q] = 0.f;

  for (int kb = 0; kb < H; kb += 32 * kUnroll) {
    uint4 rg0[kUnroll], rg8[kUnroll], ru0[kUnroll], ru8[kUnroll], xv[kUnroll][NT];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int off = kb + 32 * u + 8 * tig;
      const bool kin = off < H;
      rg0[u] = kin && ok0 ? ldg_stream(g0 + off) : zero4();
      rg8[u] = kin && ok8 ? ldg_stream(g8 + off) : zero4();
      ru0[u] = kin && ok0 ? ldg_stream(u0 + off) : zero4();
      ru8[u] = kin && ok8 ? ldg_stream(u8 + off) : zero4();
#pragma unroll
      for (int j = 0; j < NT; ++j) xv[u][j] = kin && xr[j] ? ldg_keep(xr[j] + off) : zero4();
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        mma_block(cg[j], rg0[u], rg8[u], xv[u][j]);
        mma_block(cu[j], ru0[u], ru8[u], xv[u][j]);
      }
  }

  // c0,c1: row gid, tokens 2*tig, 2*tig+1; c2,c3: row gid+8, same tokens.
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int t = tb + 8 * j + 2 * tig + (q & 1);
      const int f = f0 + gid + (q >> 1) * 8;
      if (t < m && f < F) {
        const float gv = cg[j][q], uv = cu[j][q];
        const float hv = gv / (1.0f + expf(-gv)) * uv;
        h_out[static_cast<size_t>(row0 + t) * F + f] = f32_to_bf16_rne(hv);
      }
    }
}

template <int NT>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
ffn_down_kernel(const __grid_constant__ FfnLaunch g, const int32_t* __restrict__ offsets, int n_split,
                int kchunk, int H, int F, const uint16_t* __restrict__ hin, float* __restrict__ y_part,
                size_t split_stride) {
  const int w = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
  if (w >= g.tile_start[g.n]) return;
  const int lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
  const int i = find_entry(g, w);
  int local = w - g.tile_start[i];
  const int chunk = local % g.tok_chunks[i];
  local /= g.tok_chunks[i];
  const int split = local % n_split;
  const int d0 = (local / n_split) * 16;
  const int e = g.expert[i];
  const int row0 = offsets[e];
  const int m = offsets[e + 1] - row0;
  const int tb = chunk * g.token_chunk;
  const int kbeg = split * kchunk, kend = min(F, kbeg + kchunk);
  if (tb >= m) return;

  const uint16_t* wd = g.slab[i] + static_cast<size_t>(2) * F * H;
  const bool ok0 = d0 + gid < H, ok8 = d0 + gid + 8 < H;
  const uint16_t* r0 = wd + static_cast<size_t>(ok0 ? d0 + gid : 0) * F;
  const uint16_t* r8 = wd + static_cast<size_t>(ok8 ? d0 + gid + 8 : 0) * F;
  const uint16_t* xr[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const int t = tb + 8 * j + gid;
    xr[j] = t < m ? hin + static_cast<size_t>(row0 + t) * F : nullptr;
  }
  float c[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) c[j][q] = 0.f;

  for (int kb = kbeg; kb < kend; kb += 32 * kUnroll) {
    uint4 a0[kUnroll], a8[kUnroll], xv[kUnroll][NT];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int off = kb + 32 * u + 8 * tig;
      const bool kin = off < kend;
      a0[u] = kin && ok0 ? ldg_stream(r0 + off) : zero4();
      a8[u] = kin && ok8 ? ldg_stream(r8 + off) : zero4();
#pragma unroll
      for (int j = 0; j < NT; ++j) xv[u][j] = kin && xr[j] ? ldg_keep(xr[j] + off) : zero4();
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
#pragma unroll
      for (int j = 0; j < NT; ++j) mma_block(c[j], a0[u], a8[u], xv[u][j]);
  }
  float* out = y_part + split * split_stride;
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int t = tb + 8 * j + 2 * tig + (q & 1);
      const int d = d0 + gid + (q >> 1) * 8;
      if (t < m && d < H) out[static_cast<size_t>(row0 + t) * H + d] = c[j][q];
    }
}

template <int NT>
void launch_pair(const FfnLaunch& gu, const FfnLaunch& dn, const int32_t* offsets, const int32_t* perm_src,
                 int k, const uint16_t* x, int H, int F, uint16_t* h, float* y_part, int n_split, int kchunk,
                 size_t split_stride, cudaStream_t s) {
  const int gu_warps = gu.tile_start[gu.n], dn_warps = dn.tile_start[dn.n];
  if (gu_warps > 0) {
    ffn_gateup_kernel<NT><<<(gu_warps + kWarpsPerCta - 1) / kWarpsPerCta, kWarpsPerCta * 32, 0, s>>>(
        gu, offsets, perm_src, k, x, H, F, h);
    PS_LAUNCH_CHECK("ffn_gateup_kernel");
  }
  if (dn_warps > 0) {
    ffn_down_kernel<NT><<<(dn_warps + kWarpsPerCta - 1) / kWarpsPerCta, kWarpsPerCta * 32, 0, s>>>(
        dn, offsets, n_split, kchunk, H, F, h, y_part, split_stride);
    PS_LAUNCH_CHECK("ffn_down_kernel");
  }
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" {

int ps_ffn_down_splits(int H, int F) {
  (void)H;
  // Keep >= ~3.5K of K per warp (long enough streams) while giving single-expert
  // launches >= 4 warps per SM: Mixtral F=14336 -> 4, DeepSeek/Qwen3 -> 1.
  return std::max(1, std::min(8, F / 3584));
}

ps_status ps_expert_ffn(const ps_expert_group* group, const int32_t* counts_host, const int32_t* offsets,
                        const int32_t* perm_src, int k, const uint16_t* x, int H, int F, uint16_t* h,
                        float* y_part, int n_split, int total_rows, void* stream) {
  return guarded([&] {
    require(group && counts_host && offsets && perm_src && x && h && y_part, "ps_expert_ffn: null argument");
    require(H >= 8 && F >= 8 && H % 8 == 0 && F % 8 == 0, "ps_expert_ffn: H and F must be multiples of 8");
    require(n_split >= 1 && group->n >= 0 && group->n <= PS_MAX_GROUP, "ps_expert_ffn: bad group/split");
    cudaStream_t s = as_stream(stream);
    int max_m = 0;
    for (int i = 0; i < group->n; ++i) {
      require(group->slabs[i] != nullptr, "ps_expert_ffn: null slab");
      max_m = std::max(max_m, counts_host[group->experts[i]]);
    }
    if (max_m == 0) return;
    const int NT = max_m <= 8 ? 1 : max_m <= 16 ? 2 : max_m <= 32 ? 4 : 8;
    const int token_chunk = 8 * NT;
    int kchunk = (F + n_split - 1) / n_split;
    kchunk = (kchunk + 31) / 32 * 32;
    const int row_tiles_f = (F + 15) / 16, row_tiles_h = (H + 15) / 16;
    require(total_rows >= max_m, "ps_expert_ffn: total_rows smaller than an expert's rows");
    const size_t split_stride = static_cast<size_t>(total_rows) * H;

    for (int base = 0; base < group->n; base += kMaxGroup) {
      FfnLaunch gu{}, dn{};
      gu.token_chunk = dn.token_chunk = token_chunk;
      for (int i = base; i < std::min(group->n, base + kMaxGroup); ++i) {
        const int e = group->experts[i];
        const int m = counts_host[e];
        if (m == 0) continue;
        const int tc = (m + token_chunk - 1) / token_chunk;
        gu.expert[gu.n] = dn.expert[dn.n] = e;
        gu.slab[gu.n] = dn.slab[dn.n] = group->slabs[i];
        gu.tok_chunks[gu.n] = dn.tok_chunks[dn.n] = tc;
        gu.tile_start[gu.n + 1] = gu.tile_start[gu.n] + row_tiles_f * tc;
        dn.tile_start[dn.n + 1] = dn.tile_start[dn.n] + row_tiles_h * n_split * tc;
        ++gu.n;
        ++dn.n;
      }
      if (gu.n == 0) continue;
      switch (NT) {
        case 1: launch_pair<1>(gu, dn, offsets, perm_src, k, x, H, F, h, y_part, n_split, kchunk, split_stride, s); break;
        case 2: launch_pair<2>(gu, dn, offsets, perm_src, k, x, H, F, h, y_part, n_split, kchunk, split_stride, s); break;
        case 4: launch_pair<4>(gu, dn, offsets, perm_src, k, x, H, F, h, y_part, n_split, kchunk, split_stride, s); break;
        default: launch_pair<8>(gu, dn, offsets, perm_src, k, x, H, F, h, y_part, n_split, kchunk, split_stride, s); break;
      }
    }
  });
}

}  // extern "C"
