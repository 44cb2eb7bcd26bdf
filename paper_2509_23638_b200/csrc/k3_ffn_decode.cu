// K3 (decode path) — grouped SwiGLU expert FFN as an HBM-streaming GEMV.
//
// No reference code exists for the expert FFN; the op is
// y = W_down(SiLU(W_gate x) * (W_up x)) over the experts a
// decode step activates, with per-expert token counts m_e <= 64 per pass.
//
// Design (HBM-bound: algorithmic bytes = sum_e 3*H*F*2):
//  * CTA = one 16-row tile of one expert's weight matrix; its W warps split the K
//    range of the tile and stream their slice once with 128-bit
//    ld.global.nc.L1::no_allocate loads (16 loads per lane in flight); the W partial
//    16xN accumulators are reduced through shared memory at the end. A single expert
//    therefore spreads over (rows/16) x W warps (7168 warps for Mixtral gate_up) —
//    enough memory-level parallelism for HBM even when one on-demand expert is
//    launched alone.
//  * m_e token vectors are the 8-wide N side of mma.sync.m16n8k16 (bf16 in, fp32
//    accumulate). A dot product is invariant under a common permutation of K, so each
//    lane feeds its A fragment straight from its own coalesced 16-byte load (rows g and
//    g+8, elements 8t..8t+7 of a 32-wide K block) and loads the matching 16 bytes of x
//    for its B fragment: no shared-memory staging, no swizzle, no descriptors.
//  * gate_up: gate and up rows of the same F range in one CTA; epilogue
//    h = SiLU(g) * u -> bf16 [perm_row, F].
//    down:    16 H-rows of W_down; optional global split-K over F (n_split) into fp32
//    partials y_part[split][perm_row][H], summed in fixed order by K2's combine.
//  * Deterministic (no atomics). Rows beyond the matrix and K tails are zero-filled.
#include <algorithm>
#include <vector>

#include "device_common.cuh"

namespace ps {
namespace {

constexpr int kMaxGroup = 120;
// K blocks in flight per lane: 4 (16 x 16 B loads for gate_up) unless many token
// groups make the x fragments the register bottleneck.
template <int NT> constexpr int unroll_for() { return NT >= 4 ? 2 : 4; }

struct FfnLaunch {
  int n;
  int token_chunk;                 // tokens per work item (8 * NT)
  int tile_start[kMaxGroup + 1];   // prefix of CTA work items per entry
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

// Streams rows (g, g+8) of NM matrices over this warp's K range [kbeg, kend),
// accumulating NM x NT 16x8 tiles.
template <int NT, int NM>
__device__ __forceinline__ void stream_tile(const uint16_t* const (&row0)[NM], const uint16_t* const (&row8)[NM],
                                            bool ok0, bool ok8, const uint16_t* const (&xr)[NT], int kbeg, int kend,
                                            int tig, float (&acc)[NM][NT][4]) {
  constexpr int kUnroll = unroll_for<NT>();
  for (int kb = kbeg; kb < kend; kb += 32 * kUnroll) {
    uint4 a0[kUnroll][NM], a8[kUnroll][NM], xv[kUnroll][NT];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int off = kb + 32 * u + 8 * tig;
      const bool kin = off < kend;
#pragma unroll
      for (int mt = 0; mt < NM; ++mt) {
        a0[u][mt] = kin && ok0 ? ldg_stream(row0[mt] + off) : zero4();
        a8[u][mt] = kin && ok8 ? ldg_stream(row8[mt] + off) : zero4();
      }
#pragma unroll
      for (int j = 0; j < NT; ++j) xv[u][j] = kin && xr[j] ? ldg_keep(xr[j] + off) : zero4();
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
#pragma unroll
      for (int mt = 0; mt < NM; ++mt)
#pragma unroll
        for (int j = 0; j < NT; ++j) mma_block(acc[mt][j], a0[u][mt], a8[u][mt], xv[u][j]);
  }
}

// Shared-memory reduction of the W warps' partial tiles, layout red[w][mt][j][q][lane].
template <int NT, int NM>
__device__ __forceinline__ void publish(float* red, const float (&acc)[NM][NT][4], int warp, int lane) {
#pragma unroll
  for (int mt = 0; mt < NM; ++mt)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) red[(((warp * NM + mt) * NT + j) * 4 + q) * 32 + lane] = acc[mt][j][q];
}

template <int NT, int NM, int W>
__device__ __forceinline__ float reduced(const float* red, int mt, int j, int q, int lane) {
  float s = 0.f;
#pragma unroll
  for (int w = 0; w < W; ++w) s += red[(((w * NM + mt) * NT + j) * 4 + q) * 32 + lane];
  return s;
}

template <int NT, int W>
__global__ void __launch_bounds__(W * 32)
ffn_gateup_kernel(const __grid_constant__ FfnLaunch g, const int32_t* __restrict__ offsets,
                  const int32_t* __restrict__ perm_src, int k, const uint16_t* __restrict__ x, int H, int F,
                  uint16_t* __restrict__ h_out) {
  extern __shared__ float red[];
  const int cta = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
  const int i = find_entry(g, cta);
  const int local = cta - g.tile_start[i];
  const int chunk = local % g.tok_chunks[i];
  const int f0 = (local / g.tok_chunks[i]) * 16;
  const int e = g.expert[i];
  const int row0 = offsets[e];
  const int m = offsets[e + 1] - row0;
  const int tb = chunk * g.token_chunk;
  if (tb >= m) return;  // expert not routed this step (uniform across the CTA)

  const uint16_t* wg = g.slab[i];
  const bool ok0 = f0 + gid < F, ok8 = f0 + gid + 8 < F;
  const size_t ra = ok0 ? f0 + gid : 0, rb = ok8 ? f0 + gid + 8 : 0;
  const uint16_t* const r0[2] = {wg + ra * H, wg + (static_cast<size_t>(F) + ra) * H};
  const uint16_t* const r8[2] = {wg + rb * H, wg + (static_cast<size_t>(F) + rb) * H};
  const uint16_t* xr[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const int t = tb + 8 * j + gid;
    xr[j] = t < m ? x + static_cast<size_t>(perm_src[row0 + t] / k) * H : nullptr;
  }
  const int nblk = (H + 31) / 32, per = (nblk + W - 1) / W;
  const int kbeg = min(H, warp * per * 32), kend = min(H, (warp + 1) * per * 32);

  float acc[2][NT][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[mt][j][q] = 0.f;
  stream_tile<NT, 2>(r0, r8, ok0, ok8, xr, kbeg, kend, tig, acc);
  publish<NT, 2>(red, acc, warp, lane);
  __syncthreads();

  // Value v = (j, q, lane): c0,c1 -> row gid, tokens 2*tig+{0,1}; c2,c3 -> row gid+8.
  for (int v = threadIdx.x; v < NT * 4 * 32; v += W * 32) {
    const int ln = v & 31, q = (v >> 5) & 3, j = v >> 7;
    const int t = tb + 8 * j + 2 * (ln & 3) + (q & 1);
    const int f = f0 + (ln >> 2) + (q >> 1) * 8;
    if (t < m && f < F) {
      const float gv = reduced<NT, 2, W>(red, 0, j, q, ln), uv = reduced<NT, 2, W>(red, 1, j, q, ln);
      const float hv = gv / (1.0f + expf(-gv)) * uv;
      h_out[static_cast<size_t>(row0 + t) * F + f] = f32_to_bf16_rne(hv);
    }
  }
}

template <int NT, int W>
__global__ void __launch_bounds__(W * 32)
ffn_down_kernel(const __grid_constant__ FfnLaunch g, const int32_t* __restrict__ offsets, int n_split,
                int kchunk, int H, int F, const uint16_t* __restrict__ hin, float* __restrict__ y_part,
                size_t split_stride) {
  extern __shared__ float red[];
  const int cta = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
  const int i = find_entry(g, cta);
  int local = cta - g.tile_start[i];
  const int chunk = local % g.tok_chunks[i];
  local /= g.tok_chunks[i];
  const int split = local % n_split;
  const int d0 = (local / n_split) * 16;
  const int e = g.expert[i];
  const int row0 = offsets[e];
  const int m = offsets[e + 1] - row0;
  const int tb = chunk * g.token_chunk;
  if (tb >= m) return;
  const int sbeg = split * kchunk, send = min(F, sbeg + kchunk);

  const uint16_t* wd = g.slab[i] + static_cast<size_t>(2) * F * H;
  const bool ok0 = d0 + gid < H, ok8 = d0 + gid + 8 < H;
  const uint16_t* const r0[1] = {wd + static_cast<size_t>(ok0 ? d0 + gid : 0) * F};
  const uint16_t* const r8[1] = {wd + static_cast<size_t>(ok8 ? d0 + gid + 8 : 0) * F};
  const uint16_t* xr[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const int t = tb + 8 * j + gid;
    xr[j] = t < m ? hin + static_cast<size_t>(row0 + t) * F : nullptr;
  }
  const int nblk = (send - sbeg + 31) / 32, per = (nblk + W - 1) / W;
  const int kbeg = min(send, sbeg + warp * per * 32), kend = min(send, sbeg + (warp + 1) * per * 32);

  float acc[1][NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[0][j][q] = 0.f;
  stream_tile<NT, 1>(r0, r8, ok0, ok8, xr, kbeg, kend, tig, acc);
  publish<NT, 1>(red, acc, warp, lane);
  __syncthreads();

  float* out = y_part + split * split_stride;
  for (int v = threadIdx.x; v < NT * 4 * 32; v += W * 32) {
    const int ln = v & 31, q = (v >> 5) & 3, j = v >> 7;
    const int t = tb + 8 * j + 2 * (ln & 3) + (q & 1);
    const int d = d0 + (ln >> 2) + (q >> 1) * 8;
    if (t < m && d < H) out[static_cast<size_t>(row0 + t) * H + d] = reduced<NT, 1, W>(red, 0, j, q, ln);
  }
}

template <int NT, int W>
void launch_pair(const FfnLaunch& gu, const FfnLaunch& dn, const int32_t* offsets, const int32_t* perm_src,
                 int k, const uint16_t* x, int H, int F, uint16_t* h, float* y_part, int n_split, int kchunk,
                 size_t split_stride, cudaStream_t s) {
  const int gu_ctas = gu.tile_start[gu.n], dn_ctas = dn.tile_start[dn.n];
  const size_t smem_gu = sizeof(float) * W * 2 * NT * 4 * 32, smem_dn = sizeof(float) * W * NT * 4 * 32;
  static bool attr_set = false;  // per template instance
  if (!attr_set) {
    PS_CUDA(cudaFuncSetAttribute(ffn_gateup_kernel<NT, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem_gu)));
    PS_CUDA(cudaFuncSetAttribute(ffn_down_kernel<NT, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem_dn)));
    attr_set = true;
  }
  if (gu_ctas > 0) {
    ffn_gateup_kernel<NT, W><<<gu_ctas, W * 32, smem_gu, s>>>(gu, offsets, perm_src, k, x, H, F, h);
    PS_LAUNCH_CHECK("ffn_gateup_kernel");
  }
  if (dn_ctas > 0) {
    ffn_down_kernel<NT, W><<<dn_ctas, W * 32, smem_dn, s>>>(dn, offsets, n_split, kchunk, H, F, h, y_part,
                                                           split_stride);
    PS_LAUNCH_CHECK("ffn_down_kernel");
  }
}

template <int W>
void launch_nt(int NT, const FfnLaunch& gu, const FfnLaunch& dn, const int32_t* offsets, const int32_t* perm_src,
               int k, const uint16_t* x, int H, int F, uint16_t* h, float* y_part, int n_split, int kchunk,
               size_t split_stride, cudaStream_t s) {
  switch (NT) {
    case 1: launch_pair<1, W>(gu, dn, offsets, perm_src, k, x, H, F, h, y_part, n_split, kchunk, split_stride, s); break;
    case 2: launch_pair<2, W>(gu, dn, offsets, perm_src, k, x, H, F, h, y_part, n_split, kchunk, split_stride, s); break;
    case 4: launch_pair<4, W>(gu, dn, offsets, perm_src, k, x, H, F, h, y_part, n_split, kchunk, split_stride, s); break;
    default: launch_pair<8, W>(gu, dn, offsets, perm_src, k, x, H, F, h, y_part, n_split, kchunk, split_stride, s); break;
  }
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" {

int ps_ffn_down_splits(int H, int F) {
  // K is split across the warps of each CTA; a long down projection (Mixtral F=14336)
  // is additionally split in two across CTAs so a single on-demand expert still puts
  // ~26 warps on every SM (the register-limited occupancy) instead of ~14.
  (void)H;
  return F >= 8192 ? 2 : 1;
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
    require(total_rows >= max_m, "ps_expert_ffn: total_rows smaller than an expert's rows");
    const size_t split_stride = static_cast<size_t>(total_rows) * H;
    const int NT = max_m <= 8 ? 1 : max_m <= 16 ? 2 : max_m <= 32 ? 4 : 8;
    const int token_chunk = 8 * NT;
    int kchunk = (F + n_split - 1) / n_split;
    kchunk = (kchunk + 31) / 32 * 32;
    const int row_tiles_f = (F + 15) / 16, row_tiles_h = (H + 15) / 16;

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
      // Warps per CTA: 8 while the launch is small (one or a few experts) so a single
      // expert still fills every SM; 4 once there are >= 16 CTAs per SM anyway.
      const int W = gu.tile_start[gu.n] >= 16 * kNumSMs ? 4 : 8;
      if (W == 8)
        launch_nt<8>(NT, gu, dn, offsets, perm_src, k, x, H, F, h, y_part, n_split, kchunk, split_stride, s);
      else
        launch_nt<4>(NT, gu, dn, offsets, perm_src, k, x, H, F, h, y_part, n_split, kchunk, split_stride, s);
    }
  });
}

}  // extern "C"
