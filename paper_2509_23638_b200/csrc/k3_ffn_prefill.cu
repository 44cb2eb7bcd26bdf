// K3 (prefill path) — grouped SwiGLU expert FFN on the 5th-generation tensor cores:
// TMA -> shared memory (128B swizzle, 4-stage mbarrier ring) -> tcgen05.mma (bf16 in,
// fp32 accumulate in TMEM, M=128 x N=256 per instruction group) -> tcgen05.ld epilogue.
//
// Problem (no reference code): for every routed
// expert e with m_e permuted rows (K2 order, x_perm contiguous):
//   gate_up:  D[m_e, 2x128 tile] = X_e . [W_gate tile ; W_up tile]^T   (K = H)
//             epilogue h = SiLU(g) * u  -> bf16 h_perm[row, F]
//   down:     D[m_e, 256 tile]   = H_e . W_down tile^T                (K = F)
//             epilogue fp32 y_perm[row, H]   (summed by K2's combine)
// Both operands are K-major (row-major with K contiguous): the natural TN layout for
// kind::f16 with a_major = b_major = K.
//
// Kernel structure (one persistent CTA per SM, 192 threads, 1 CTA/SM):
//   warp 0        TMA producer (one elected lane): A box 64x128, B boxes 64x128 (x2) or
//                 64x256, arrive.expect_tx on the stage's full barrier.
//   warp 1        MMA issuer (one lane): 4 x tcgen05.mma (K=16) per 64-wide K block,
//                 tcgen05.commit -> empty barrier (frees the smem stage) and, after the
//                 last K block, -> tmem_full barrier of the accumulator stage.
//   warps 2..5    epilogue: tcgen05.ld 32x32b.x32 of its TMEM lane quarter, activation,
//                 stores; then arrive on tmem_empty (two accumulator stages of 256 fp32
//                 columns = all 512 TMEM columns, so epilogue of tile i overlaps MMA of
//                 tile i+1).
// Tiles are ordered m-fastest within (expert, n-tile) so CTAs working on the same weight
// tile run concurrently and the B tile is fetched from HBM once, then served by L2.
//
// Three kernels (ps_set_prefill_kernel): the single-CTA M=128 kernel (0), the CTA-pair
// M=256 kernel (1), and the default token-N CTA-pair kernel (2 = auto, 3): weights on
// the M side, an expert's tokens on the N side (no padding of ragged experts beyond 16
// rows), gate_up and down in one launch with per-expert release/acquire counters.
#include <cuda.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "device_common.cuh"

namespace ps {
namespace {

constexpr int kBM = 128;            // tokens per tile (UMMA M)
constexpr int kBN = 256;            // accumulator columns per tile (UMMA N)
constexpr int kBK = 64;             // K elements per stage (128 B rows -> 128B swizzle)
constexpr int kStages = 4;
constexpr int kThreads = 192;
constexpr int kABytes = kBM * kBK * 2;         // 16 KiB
constexpr int kBBytes = kBN * kBK * 2;         // 32 KiB
constexpr int kStageBytes = kABytes + kBBytes; // 48 KiB
constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
constexpr int kMaxExperts = 128;

enum Mode { kSwiGLU = 0, kStoreF32 = 1 };

struct PrefillParams {
  int n_experts;
  int mode;
  int K;                     // reduction length (H for gate_up, F for down)
  int F, H;                  // model dims
  int n_tiles_n;             // N tiles per expert (F/128 for gate_up, H/256 for down)
  int tile_start[kMaxExperts + 1];  // prefix of tiles per entry
  int m_tiles[kMaxExperts];
  int row0[kMaxExperts];     // first permuted row of the entry
  int rows[kMaxExperts];     // m_e
  const CUtensorMap* a_map;  // device: activation map (x_perm or h_perm)
  const CUtensorMap* b_maps; // device array [n_experts] of weight tensor maps
  void* out;                 // h (bf16, [rows_total, F]) or y (f32, [rows_total, H])
  int out_ld;                // leading dimension (elements) of out
};

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// UMMA shared-memory descriptor, K-major, SWIZZLE_128B: start>>4 [0,14), LBO>>4
// [16,30) (unused for swizzled K-major, 1 as in CUTLASS), SBO>>4 [32,46) = 1024 B
// between 8-row atoms, version 1 [46,48), layout 2 = SWIZZLE_128B [61,64).
__device__ __forceinline__ uint64_t make_desc(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3fff);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// Instruction descriptor kind::f16: D=f32 [4,6), A=B=bf16 [7,10)/[10,13), K-major,
// N>>3 [17,23), M>>4 [24,29).
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(kBN >> 3) << 17) |
                            (static_cast<uint32_t>(kBM >> 4) << 24);

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%"
      "19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

struct TileCoord {
  int entry, m_tile, n_tile;
};

__device__ __forceinline__ TileCoord tile_coord(const PrefillParams& p, int t) {
  int lo = 0, hi = p.n_experts - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (p.tile_start[mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  const int local = t - p.tile_start[lo];
  return {lo, local % p.m_tiles[lo], local / p.m_tiles[lo]};  // m fastest
}

__global__ void __launch_bounds__(kThreads, 1)
ffn_prefill_kernel(const __grid_constant__ PrefillParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles = p.tile_start[p.n_experts];
  const int k_blocks = (p.K + kBK - 1) / kBK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // whole warp: TMEM allocation (512 columns = 2 accumulator stages)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // Maps live in a reused ring slot written by a host copy: order them before
    // tensormap-proxy use (drops any descriptor cached for the slot's previous contents).
    for (int i = lane; i <= p.n_experts; i += 32) {
      const CUtensorMap* m = i == 0 ? p.a_map : p.b_maps + (i - 1);
      asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(m) : "memory");
    }
    __syncwarp();
    if (lane == 0) {  // ---------------------------------------------- TMA producer
      const CUtensorMap* a_map = p.a_map;
      prefetch_map(a_map);
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const TileCoord tc = tile_coord(p, t);
        const CUtensorMap* bmap = p.b_maps + tc.entry;
        const int arow = p.row0[tc.entry] + tc.m_tile * kBM;
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * kStageBytes;
          uint8_t* sb = sa + kABytes;
          mbar_expect_tx(&full_bar[stage], kStageBytes);
          tma_load_2d(sa, a_map, &full_bar[stage], kb * kBK, arow);
          if (p.mode == kSwiGLU) {
            const int n0 = tc.n_tile * (kBN / 2);
            tma_load_2d(sb, bmap, &full_bar[stage], kb * kBK, n0);                      // gate rows
            tma_load_2d(sb + kBBytes / 2, bmap, &full_bar[stage], kb * kBK, p.F + n0);  // up rows
          } else {
            const int n0 = tc.n_tile * kBN;
            tma_load_2d(sb, bmap, &full_bar[stage], kb * kBK, n0);
            tma_load_2d(sb + kBBytes / 2, bmap, &full_bar[stage], kb * kBK, n0 + kBN / 2);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------------------------------------- MMA issuer
      int stage = 0;
      uint32_t phase = 0;
      int as = 0;
      uint32_t aphase = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        mbar_wait(&tempty_bar[as], aphase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + static_cast<uint32_t>(as * kBN);
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * kStageBytes);
          const uint32_t sb = sa + kABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {  // K=16 per instruction: +32 B in the swizzled row
            umma_f16(d, make_desc(sa + kk * 32), make_desc(sb + kk * 32), (kb | kk) != 0 ? 1u : 0u);
          }
          umma_commit(&empty_bar[stage]);  // smem stage free once these MMAs retire
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull_bar[as]);  // accumulator ready for the epilogue
        as ^= 1;
        if (as == 0) aphase ^= 1;
      }
    }
  } else {  // ------------------------------------------------------- epilogue (4 warps)
    const int quarter = warp & 3;  // TMEM lanes [32*quarter, +32) for this warp
    const int r = quarter * 32 + lane;
    int as = 0;
    uint32_t aphase = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const TileCoord tc = tile_coord(p, t);
      mbar_wait(&tfull_bar[as], aphase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + static_cast<uint32_t>(as * kBN) + (static_cast<uint32_t>(quarter * 32) << 16);
      const int row_in_expert = tc.m_tile * kBM + r;
      const bool valid = row_in_expert < p.rows[tc.entry];
      const size_t out_row = static_cast<size_t>(p.row0[tc.entry] + row_in_expert);
      if (p.mode == kSwiGLU) {
        const int n0 = tc.n_tile * (kBN / 2);
        uint16_t* out = static_cast<uint16_t*>(p.out) + out_row * p.out_ld + n0;
#pragma unroll 1
        for (int c = 0; c < kBN / 2; c += 32) {
          uint32_t g[32], u[32];
          tmem_ld32(tbase + c, g);
          tmem_ld32(tbase + kBN / 2 + c, u);
          tmem_ld_wait();
          if (valid) {
            uint32_t packed[16];
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              const float g0 = __uint_as_float(g[j]), g1 = __uint_as_float(g[j + 1]);
              const float h0 = g0 / (1.0f + expf(-g0)) * __uint_as_float(u[j]);
              const float h1 = g1 / (1.0f + expf(-g1)) * __uint_as_float(u[j + 1]);
              packed[j / 2] = static_cast<uint32_t>(f32_to_bf16_rne(h0)) |
                              (static_cast<uint32_t>(f32_to_bf16_rne(h1)) << 16);
            }
            if (n0 + c + 32 <= p.F) {
              uint4* dst = reinterpret_cast<uint4*>(out + c);
#pragma unroll
              for (int q = 0; q < 4; ++q)
                dst[q] = make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
            } else {
              for (int j = 0; j < 32 && n0 + c + j < p.F; ++j)
                out[c + j] = static_cast<uint16_t>(packed[j / 2] >> (16 * (j & 1)));
            }
          }
        }
      } else {
        const int n0 = tc.n_tile * kBN;
        float* out = static_cast<float*>(p.out) + out_row * p.out_ld + n0;
#pragma unroll 1
        for (int c = 0; c < kBN; c += 32) {
          uint32_t v[32];
          tmem_ld32(tbase + c, v);
          tmem_ld_wait();
          if (valid) {
            if (n0 + c + 32 <= p.H) {
              float4* dst = reinterpret_cast<float4*>(out + c);
#pragma unroll
              for (int q = 0; q < 8; ++q)
                dst[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                     __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
            } else {
              for (int j = 0; j < 32 && n0 + c + j < p.H; ++j) out[c + j] = __uint_as_float(v[j]);
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[as]);
      as ^= 1;
      if (as == 0) aphase ^= 1;
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
  }
}

// ------------------------------------------------------------------ CTA-pair variant
// tcgen05.mma.cta_group::2: a cluster of 2 CTAs on the two SMs of a TPC computes one
// 256 x 256 tile (M = 256 = 128 rows per CTA, N = 256). Each CTA stages only its half
// of the operands — A: its 128 token rows; B: 128 of the 256 weight rows (SwiGLU: CTA 0
// the gate rows, CTA 1 the up rows; down: consecutive halves) — so a 64-wide K stage is
// 32 KiB per CTA instead of 48 KiB: 1.5x less L2->SM traffic per flop and 6 stages in
// flight instead of 4. The leader (rank 0) issues the MMAs for the pair; both CTAs' TMA
// loads complete on the leader's full barrier; tcgen05.commit multicasts the stage-free
// and accumulator-ready signals to both CTAs; both CTAs' epilogues arrive on the
// leader's accumulator-empty barrier. Each CTA's TMEM holds its 128 rows x 256 columns.
constexpr int kPairStages = 6;
constexpr int kPairStageBytes = kABytes + kBBytes / 2;  // 32 KiB
constexpr int kPairSmemBytes = kPairStages * kPairStageBytes + 1024 + 256;
constexpr uint32_t kIdescPair = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(kBN >> 3) << 17) |
                                (static_cast<uint32_t>((2 * kBM) >> 4) << 24);

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same shared variable in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair_s(uint32_t dst, const CUtensorMap* map, uint32_t leader_bar, int c0,
                                                   int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void umma_f16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdescPair), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {  // arrive on `bar` in both CTAs
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// Pair tiles: (entry, 256-row block, n tile), m fastest; m_tiles[] count 256-row blocks.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
ffn_prefill_pair_kernel(const __grid_constant__ PrefillParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kPairStages * kPairStageBytes);
  uint64_t* empty_bar = full_bar + kPairStages;
  uint64_t* tfull_bar = empty_bar + kPairStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int n_tiles = p.tile_start[p.n_experts];
  const int k_blocks = (p.K + kBK - 1) / kBK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kPairStages; ++s) {
      mbar_init(&full_bar[s], 1);   // leader: its producer's arrive.expect_tx (both CTAs' bytes)
      mbar_init(&empty_bar[s], 1);  // one multicast commit per stage use
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 2 * 128);  // leader: the epilogue threads of both CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // TMEM: 2 accumulator stages x 256 columns, allocated for the pair
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // peer barriers initialised before any remote arrive / complete_tx
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    for (int i = lane; i <= p.n_experts; i += 32) {
      const CUtensorMap* m = i == 0 ? p.a_map : p.b_maps + (i - 1);
      asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(m) : "memory");
    }
    __syncwarp();
    if (lane == 0) {  // ---------------------------------------------- TMA producer (both CTAs)
      const CUtensorMap* a_map = p.a_map;
      prefetch_map(a_map);
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < n_tiles; t += n_pairs) {
        const TileCoord tc = tile_coord(p, t);
        const CUtensorMap* bmap = p.b_maps + tc.entry;
        const int arow = p.row0[tc.entry] + tc.m_tile * (2 * kBM) + static_cast<int>(rank) * kBM;
        int brow;
        if (p.mode == kSwiGLU) brow = (rank ? p.F : 0) + tc.n_tile * (kBN / 2);  // gate | up rows
        else brow = tc.n_tile * kBN + static_cast<int>(rank) * (kBN / 2);
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * kPairStageBytes;
          uint8_t* sb = sa + kABytes;
          const uint32_t lbar = mapa_shared(smem_u32(&full_bar[stage]), 0);
          if (leader) mbar_expect_tx(&full_bar[stage], 2 * kPairStageBytes);
          tma_load_2d_pair(sa, a_map, lbar, kb * kBK, arow);
          tma_load_2d_pair(sb, bmap, lbar, kb * kBK, brow);
          if (++stage == kPairStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {  // ------------------------------------ MMA issuer (leader only)
      int stage = 0;
      uint32_t phase = 0;
      int as = 0;
      uint32_t aphase = 0;
      for (int t = pair; t < n_tiles; t += n_pairs) {
        mbar_wait(&tempty_bar[as], aphase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + static_cast<uint32_t>(as * kBN);
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * kPairStageBytes);
          const uint32_t sb = sa + kABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk)
            umma_f16_pair(d, make_desc(sa + kk * 32), make_desc(sb + kk * 32), (kb | kk) != 0 ? 1u : 0u);
          umma_commit_pair(&empty_bar[stage]);
          if (++stage == kPairStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pair(&tfull_bar[as]);
        as ^= 1;
        if (as == 0) aphase ^= 1;
      }
    }
  } else {  // ------------------------------------------------------- epilogue (4 warps, both CTAs)
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t tempty_leader[2] = {mapa_shared(smem_u32(&tempty_bar[0]), 0), mapa_shared(smem_u32(&tempty_bar[1]), 0)};
    int as = 0;
    uint32_t aphase = 0;
    for (int t = pair; t < n_tiles; t += n_pairs) {
      const TileCoord tc = tile_coord(p, t);
      mbar_wait(&tfull_bar[as], aphase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + static_cast<uint32_t>(as * kBN) + (static_cast<uint32_t>(quarter * 32) << 16);
      const int row_in_expert = tc.m_tile * (2 * kBM) + static_cast<int>(rank) * kBM + r;
      const bool valid = row_in_expert < p.rows[tc.entry];
      const size_t out_row = static_cast<size_t>(p.row0[tc.entry] + row_in_expert);
      if (p.mode == kSwiGLU) {
        const int n0 = tc.n_tile * (kBN / 2);
        uint16_t* out = static_cast<uint16_t*>(p.out) + out_row * p.out_ld + n0;
#pragma unroll 1
        for (int c = 0; c < kBN / 2; c += 32) {
          uint32_t g[32], u[32];
          tmem_ld32(tbase + c, g);
          tmem_ld32(tbase + kBN / 2 + c, u);
          tmem_ld_wait();
          if (valid) {
            uint32_t packed[16];
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              const float g0 = __uint_as_float(g[j]), g1 = __uint_as_float(g[j + 1]);
              const float h0 = g0 / (1.0f + expf(-g0)) * __uint_as_float(u[j]);
              const float h1 = g1 / (1.0f + expf(-g1)) * __uint_as_float(u[j + 1]);
              packed[j / 2] = static_cast<uint32_t>(f32_to_bf16_rne(h0)) |
                              (static_cast<uint32_t>(f32_to_bf16_rne(h1)) << 16);
            }
            if (n0 + c + 32 <= p.F) {
              uint4* dst = reinterpret_cast<uint4*>(out + c);
#pragma unroll
              for (int q = 0; q < 4; ++q)
                dst[q] = make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
            } else {
              for (int j = 0; j < 32 && n0 + c + j < p.F; ++j)
                out[c + j] = static_cast<uint16_t>(packed[j / 2] >> (16 * (j & 1)));
            }
          }
        }
      } else {
        const int n0 = tc.n_tile * kBN;
        float* out = static_cast<float*>(p.out) + out_row * p.out_ld + n0;
#pragma unroll 1
        for (int c = 0; c < kBN; c += 32) {
          uint32_t v[32];
          tmem_ld32(tbase + c, v);
          tmem_ld_wait();
          if (valid) {
            if (n0 + c + 32 <= p.H) {
              float4* dst = reinterpret_cast<float4*>(out + c);
#pragma unroll
              for (int q = 0; q < 8; ++q)
                dst[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                     __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
            } else {
              for (int j = 0; j < 32 && n0 + c + j < p.H; ++j) out[c + j] = __uint_as_float(v[j]);
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive_cluster(tempty_leader[as]);
      as ^= 1;
      if (as == 0) aphase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer is done with every TMEM / barrier access of the pair
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
  }
}

// ------------------------------------------------------------------ token-N CTA-pair variant
// The weights are the M side and the tokens the N side of the MMA (D^T = W . X^T): a
// pair tile is 256 weight rows x N tokens with N = the expert's remaining rows rounded
// up to 16 (<= 256). The M-side kernels above pad every expert's last tile to 128 or
// 256 token rows; at DeepSeek-V2-Lite prefill (m_e ~ 192) that is 25 % of the tensor
// time, while here an expert of 192 rows is one N = 192 tile with no padding.
//   gate_up: CTA r's 128 A rows = gate rows [f0 + 64r, +64) then the same up rows (two
//            {64 x 64} TMA boxes), so TMEM lanes 0-63 hold gate and 64-127 up for the
//            same 64 features; a gate warp and the up warp of the same features swap
//            half of every 32-token chunk through shared memory (tcgen05.ld reaches only
//            a warp's own 32-lane quarter) and each writes h = SiLU(g) * u for 16 tokens
//            (64 B of one token row per store).
//   down:    CTA r's 128 A rows = W_down rows [h0 + 128r, +128) (one {64 x 128} box);
//            y_perm[token][h] fp32, 128 B of one token row per warp store.
//   B:       CTA r stages tokens [N/2 r, +N/2) of the tile (cta_group::2 splits N), from
//            a tensor map whose box is N/2 rows (the shared 128-row map or the entry's
//            own map for its last, shorter tile).
// ONE launch runs both phases: tiles [0, T0) are gate_up, [T0, T0 + T1) down, and every
// CTA pair walks its tiles in index order, so the gate_up tail overlaps the first down
// tiles and there is no second launch. A down tile of entry e needs all of e's h rows:
// every epilogue warp of a gate_up tile of e adds 1 to done[e] (release) after its h
// stores; the producer acquires done[e] >= target[e] before it TMA-loads h (the counters
// only grow: targets are host-side running sums per map-ring slot, nothing is reset). A
// pair waits only on gate_up tiles, which never wait, and all pairs are co-resident (grid
// <= the device's max active 2-CTA clusters), so the wait cannot deadlock.
constexpr int kTnABytes = 128 * kBK * 2;                 // 16 KiB of weight rows
constexpr int kTnXchgBytes = 2 * 2 * 2 * 16 * 32 * 4;    // gate <-> up hand-off: 2 bufs x 2 pairs x 2 senders x 16 x 32
constexpr int kTnStageOutBytes = 4 * 32 * 32 * 4;         // y staging: 4 epilogue warps x 32 tokens x 32 features f32
constexpr int kTnMaxN = 256;                              // largest token tile (MMA N)
// Ring geometry per maximum token tile MAXN (256: 6 stages of 16 + 16 KiB; 128: 8 stages
// of 16 + 8 KiB, i.e. a third more weight bytes in flight per SM, and an expert of more
// than 128 rows is split into equal token tiles that share the weight rows through L2).
template <int MAXN> struct TnGeo {
  static constexpr int kBMaxBytes = (MAXN / 2) * kBK * 2;
  static constexpr int kStageBytes = kTnABytes + kBMaxBytes;
  static constexpr int kStages = MAXN == 256 ? 6 : 8;
  static constexpr int kSmem = kStages * kStageBytes + kTnXchgBytes + kTnStageOutBytes + 1024 + 256;
  static_assert(kSmem <= 227 * 1024, "token-N smem");
};
constexpr uint32_t kTnSignalsPerTile = 2 * 4;            // epilogue warps of both CTAs

// Tensor maps live in a persistent device table (MapTable below: every map is a pure
// function of its address, shape and box, written once, never modified), so a launch
// passes table indices instead of uploading ~5 maps per expert.
struct TnPhase {
  int K;                            // H (gate_up) or F (down)
  int n_tiles_n;                    // weight-row tiles per expert (F/128 gate_up, H/256 down)
  int tile_start[kMaxExperts + 1];  // prefix of this phase's tiles per entry
  int w_idx[kMaxExperts];           // weights of entry i: [Wg; Wu] box {64, 64} or Wd box {64, 128}
  int tok_idx[17];                  // token operand (x_perm or h_perm) with a {64, 8j}-row box, j = 1..16
  void* out;                        // h_perm (bf16) or y_perm (f32)
  int out_ld;
  int out_idx;                      // down: y_perm as [total_rows, H] f32, box {32 features, 32 tokens}
};

// The tile schedule: built on the host from host counts (in the launch parameters), or on
// the device from K2's offsets by tn_schedule_kernel (ps_expert_ffn_prefill_dev: the
// engine launches the resident group before the host has the counts).
struct TnSched {
  int n_experts;                    // active entries (m_e > 0)
  int gidx[kMaxExperts];            // group index of active entry i (its w_idx)
  int t_tiles[kMaxExperts];         // token tiles per entry (ceil(m_e / MAXN), equal widths)
  int row0[kMaxExperts];
  int rows[kMaxExperts];
  unsigned target[kMaxExperts];     // done[e] value once all of e's gate_up tiles are stored
  // Tile order: segments of (phase, entry) — gu(0..D-1), then gu(e), dn(e - D) for e >= D,
  // then the last D down segments (D >= n: every gate_up tile first, the default). A down
  // segment trailing its gate_up by a few experts finds its h rows still in L2, but its
  // acquire may wait (profiles/r02_prefill_tn.md). seg_code = entry | phase << 16.
  int maxn, even;                   // largest token tile; equal-width token tiles (default)
  int n_seg;
  int seg_start[2 * kMaxExperts + 1];
  int seg_code[2 * kMaxExperts];
};

struct TnParams {
  const CUtensorMap* maps;          // the device map table
  int n_group;                      // valid w_idx entries
  int F, H;
  TnPhase ph[2];                    // 0 = gate_up, 1 = down
  unsigned* done;                   // gate_up signals per active entry (this map-ring slot's counters)
  const TnSched* sched_dev;         // device-built schedule, or null: `sched` below
  TnSched sched;
};

struct TnTile {
  int phase, entry, n_tile, tok0, n;  // n = MMA N (tokens, multiple of 16)
  bool last;
};

// Token tiles of an expert with m rows split into tt tiles: ceil(m / tt) rounded up to 32
// (the epilogue's chunk width; <= MAXN since MAXN is a multiple of 32), the last tile
// takes the rest.
// even == 0 (PS_TN_EVEN=0, A/B knob): MAXN-wide tiles, the last takes the rest.
__host__ __device__ __forceinline__ int tn_tile_width(int m, int tt, int even, int maxn) {
  if (!even && tt > 1) return maxn;
  return tt == 1 ? (m + 15) & ~15 : ((m + tt - 1) / tt + 31) & ~31;
}

__device__ __forceinline__ TnTile tn_tile(const TnSched& p, int t) {
  TnTile c;
  int lo = 0, hi = p.n_seg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (p.seg_start[mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  const int local = t - p.seg_start[lo];
  c.phase = p.seg_code[lo] >> 16;
  lo = p.seg_code[lo] & 0xffff;
  const int tt = p.t_tiles[lo];
  const int t_tile = local % tt;  // token tiles fastest: concurrent tiles share the weight rows
  c.entry = lo;
  c.n_tile = local / tt;
  const int ts = tn_tile_width(p.rows[lo], tt, p.even, p.maxn);  // equal widths (multiples of 32)
  c.tok0 = t_tile * ts;
  const int rem = p.rows[lo] - c.tok0;
  c.n = rem >= ts ? ts : (rem + 15) & ~15;
  c.last = t_tile == tt - 1;
  return c;
}

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}


template <int MAXN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
ffn_prefill_tn_kernel(const __grid_constant__ TnParams p) {
  using G = TnGeo<MAXN>;
  constexpr int kTnStages = G::kStages;
  constexpr int kTnStageBytes = G::kStageBytes;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* xchg = reinterpret_cast<float*>(smem + kTnStages * kTnStageBytes);  // [2][2][2][16][32]
  float* ystage = reinterpret_cast<float*>(smem + kTnStages * kTnStageBytes + kTnXchgBytes);  // [4][32][32]
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kTnStages * kTnStageBytes + kTnXchgBytes + kTnStageOutBytes);
  uint64_t* empty_bar = full_bar + kTnStages;
  uint64_t* tfull_bar = empty_bar + kTnStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const TnSched& S = p.sched_dev ? *p.sched_dev : p.sched;
  const int n_tiles = S.seg_start[S.n_seg];

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kTnStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 2 * 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    for (int ph = 0; ph < 2; ++ph)
      for (int i = lane; i < p.n_group + 16; i += 32) {
        const int idx = i < p.n_group ? p.ph[ph].w_idx[i] : p.ph[ph].tok_idx[i - p.n_group + 1];
        if (idx >= 0)
          asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(p.maps + idx) : "memory");
      }
    __syncwarp();
    if (lane == 0) {  // ---------------------------------------------- TMA producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < n_tiles; t += n_pairs) {
        const TnTile tc = tn_tile(S, t);
        const TnPhase& ph = p.ph[tc.phase];
        const CUtensorMap* wmap = p.maps + ph.w_idx[S.gidx[tc.entry]];
        const int half = tc.n >> 1;
        const CUtensorMap* tmap = p.maps + ph.tok_idx[half >> 3];
        const int trow = S.row0[tc.entry] + tc.tok0 + static_cast<int>(rank) * half;
        const uint32_t bytes = 2u * (kTnABytes + static_cast<uint32_t>(half) * kBK * 2);
        const int k_blocks = (ph.K + kBK - 1) / kBK;
        if (tc.phase == 1) {  // h of this entry complete (acquire), then visible to the async proxy
          const unsigned* d = p.done + tc.entry;
          const unsigned want = S.target[tc.entry];
          unsigned v;
          for (uint32_t spin = 0;; ++spin) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(d) : "memory");
            if (static_cast<int>(v - want) >= 0) break;
            if (spin == (1u << 26)) __trap();  // ~seconds: a lost signal fails the launch instead of hanging
            __nanosleep(64);
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          const uint32_t sa = smem_u32(smem + stage * kTnStageBytes);
          const uint32_t lbar = mapa_shared(smem_u32(&full_bar[stage]), 0);
          if (leader) mbar_expect_tx(&full_bar[stage], bytes);
          if (tc.phase == 0) {
            const int f = tc.n_tile * 128 + static_cast<int>(rank) * 64;
            tma_load_2d_pair_s(sa, wmap, lbar, kb * kBK, f);                          // gate rows
            tma_load_2d_pair_s(sa + kTnABytes / 2, wmap, lbar, kb * kBK, p.F + f);    // up rows
          } else {
            tma_load_2d_pair_s(sa, wmap, lbar, kb * kBK, tc.n_tile * 256 + static_cast<int>(rank) * 128);
          }
          tma_load_2d_pair_s(sa + kTnABytes, tmap, lbar, kb * kBK, trow);
          if (++stage == kTnStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {  // ------------------------------------ MMA issuer (leader only)
      int stage = 0;
      uint32_t phase = 0;
      int as = 0;
      uint32_t aphase = 0;
      for (int t = pair; t < n_tiles; t += n_pairs) {
        const TnTile tc = tn_tile(S, t);
        const int k_blocks = (p.ph[tc.phase].K + kBK - 1) / kBK;
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(tc.n >> 3) << 17) |
                               (static_cast<uint32_t>(256 >> 4) << 24);
        mbar_wait(&tempty_bar[as], aphase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + static_cast<uint32_t>(as * MAXN);
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * kTnStageBytes);
          const uint32_t sb = sa + kTnABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint32_t acc = (kb | kk) != 0 ? 1u : 0u;
            asm volatile(
                "{\n"
                ".reg .pred p;\n"
                "setp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
                "}\n" ::"r"(d),
                "l"(make_desc(sa + kk * 32)), "l"(make_desc(sb + kk * 32)), "r"(idesc), "r"(acc));
          }
          umma_commit_pair(&empty_bar[stage]);
          if (++stage == kTnStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pair(&tfull_bar[as]);
        as ^= 1;
        if (as == 0) aphase ^= 1;
      }
    }
  } else {  // ------------------------------------------------------- epilogue (4 warps, both CTAs)
    const int quarter = warp & 3;
    const uint32_t tempty_leader[2] = {mapa_shared(smem_u32(&tempty_bar[0]), 0), mapa_shared(smem_u32(&tempty_bar[1]), 0)};
    int as = 0;
    uint32_t aphase = 0;
    int buf = 0;  // hand-off buffer: one barrier per chunk orders its reuse two chunks later
    const uint32_t xchg_s = smem_u32(xchg);
    if (p.ph[1].out_idx >= 0 && lane == 0)  // the y map (TMA stores)
      asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(p.maps + p.ph[1].out_idx) : "memory");
    __syncwarp();
    for (int t = pair; t < n_tiles; t += n_pairs) {
      const TnTile tc = tn_tile(S, t);
      const TnPhase& ph = p.ph[tc.phase];
      mbar_wait(&tfull_bar[as], aphase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + static_cast<uint32_t>(as * MAXN) + (static_cast<uint32_t>(quarter * 32) << 16);
      const int m_left = min(S.rows[tc.entry] - tc.tok0, tc.n);  // valid token columns of this tile
      const size_t row_base = static_cast<size_t>(S.row0[tc.entry] + tc.tok0);
      if (tc.phase == 0) {
        // quarters 0/1 hold gate, 2/3 up of features [32 (q & 1), +32) of this CTA's 64.
        // Per 32-token chunk the two warps of a feature group swap halves through shared
        // memory (gate sends tokens 16-31, up sends 0-15) and each computes 16 tokens of h.
        const bool is_gate = quarter < 2;
        const int f = tc.n_tile * 128 + static_cast<int>(rank) * 64 + (quarter & 1) * 32 + lane;
        uint16_t* out = static_cast<uint16_t*>(ph.out) + row_base * ph.out_ld + f;
        const int jb = is_gate ? 0 : 16;  // this warp's tokens in the chunk
#pragma unroll 1
        for (int c = 0; c < tc.n; c += 32, buf ^= 1) {  // buf alternates across tiles too
          uint32_t v[32];
          tmem_ld32(tbase + c, v);
          tmem_ld_wait();
          // xchg[buf][pair q&1][sender][16 tokens][32 lanes] (shared-window addresses: the
          // aligned smem pointer has lost its address space, so generic accesses would be used)
          const uint32_t xb = xchg_s + static_cast<uint32_t>(((buf * 2 + (quarter & 1)) * 2) * 16 * 32 * 4);
          const uint32_t mine = xb + (is_gate ? 0u : 16u * 32u * 4u) + lane * 4u;
          const uint32_t theirs = xb + (is_gate ? 16u * 32u * 4u : 0u) + lane * 4u;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(mine + j * 128u), "r"(is_gate ? v[16 + j] : v[j]) : "memory");
          named_bar_sync(1, 128);
          const int nj = min(16, m_left - c - jb);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            uint32_t ob;
            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(ob) : "r"(theirs + j * 128u) : "memory");
            const float o = __uint_as_float(ob);
            const float own = __uint_as_float(is_gate ? v[j] : v[16 + j]);
            const float g = is_gate ? own : o;
            const float u = is_gate ? o : own;
            // fast-math SiLU (ex2.approx + rcp.approx, ~2 ulp of fp32 before the bf16 rounding):
            // the IEEE expf / division slow paths made this epilogue longer than a tile's MMAs
            const float h = __fdividef(g, 1.0f + __expf(-g)) * u;
            if (j < nj) out[static_cast<size_t>(c + jb + j) * ph.out_ld] = f32_to_bf16_rne(h);
          }
        }
        // release this warp's h rows to the down tiles of the entry (TMA readers)
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __syncwarp();
        if (lane == 0)
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.done + tc.entry) : "memory");
      } else {
        // y rows leave through shared memory and one TMA store per 32x32 chunk and warp
        // (scalar global stores, 128 B per warp instruction, cost ~12 % of a DeepSeek-shape
        // launch): lane l writes feature column l of the warp's [32 tokens][32 features]
        // tile, lane 0 stores it. A chunk with fewer than 32 of the expert's rows (its last)
        // uses scalar stores: a full box would overwrite the next expert's rows.
        const CUtensorMap* ymap = p.maps + ph.out_idx;
        const int h0 = tc.n_tile * 256 + static_cast<int>(rank) * 128 + quarter * 32;
        const uint32_t ys = smem_u32(ystage) + static_cast<uint32_t>(quarter) * 32u * 32u * 4u;
        float* out = static_cast<float*>(ph.out) + row_base * ph.out_ld + h0 + lane;
#pragma unroll 1
        for (int c = 0; c < tc.n; c += 32) {
          uint32_t v[32];
          tmem_ld32(tbase + c, v);
          const int nj = min(32, m_left - c);
          if (nj < 32) {
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < nj) out[static_cast<size_t>(c + j) * ph.out_ld] = __uint_as_float(v[j]);
            continue;
          }
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // staging free
          __syncwarp();
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j)
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(ys + static_cast<uint32_t>(j * 128 + lane * 4)), "r"(v[j])
                         : "memory");
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(ymap), "r"(h0),
                "r"(static_cast<int>(row_base) + c), "r"(ys)
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
      }
      tc_fence_before();
      mbar_arrive_cluster(tempty_leader[as]);
      as ^= 1;
      if (as == 0) aphase ^= 1;
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // y stores complete
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
  }
}

// Device-side tile schedule (one CTA of kMaxExperts threads): thread i takes group entry
// i, reads its row count from K2's offsets, and block scans give the compacted entry
// index and both phases' tile prefixes; every gate_up tile comes first (the host path's
// default order). Also zeroes the active entries' gate_up counters (the slot's previous
// kernels are complete: the host reuses a ring slot only after its event).
struct TnSchedArgs {
  int maxn, even;  // largest token tile; equal-width tiles
  int n_group;
  int expert[kMaxExperts];
  int n0, n1;  // weight-row tiles per expert: gate_up, down
};

__global__ void __launch_bounds__(kMaxExperts)
tn_schedule_kernel(const int32_t* __restrict__ offsets, const __grid_constant__ TnSchedArgs a, TnSched* __restrict__ out,
                   unsigned* __restrict__ done) {
  __shared__ int s_scan[3][kMaxExperts / 32];
  const int i = threadIdx.x, lane = i & 31, warp = i >> 5;
  int m = 0;
  if (i < a.n_group) m = __ldg(offsets + a.expert[i] + 1) - __ldg(offsets + a.expert[i]);
  const int row0 = i < a.n_group ? __ldg(offsets + a.expert[i]) : 0;
  const int act = m > 0 ? 1 : 0;
  const int tt = (m + a.maxn - 1) / a.maxn;
  int v[3] = {act, tt * a.n0, tt * a.n1};
  int incl[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {  // inclusive warp scans, then warp totals
    incl[q] = v[q];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl[q], o);
      if (lane >= o) incl[q] += t;
    }
    if (lane == 31) s_scan[q][warp] = incl[q];
  }
  __syncthreads();
  int excl[3], total[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    int before = 0, tot = 0;
    for (int w = 0; w < kMaxExperts / 32; ++w) {
      if (w < warp) before += s_scan[q][w];
      tot += s_scan[q][w];
    }
    excl[q] = before + incl[q] - v[q];
    total[q] = tot;
  }
  const int n = total[0];
  if (act) {
    const int e = excl[0];
    out->gidx[e] = i;
    out->t_tiles[e] = tt;
    out->row0[e] = row0;
    out->rows[e] = m;
    out->target[e] = kTnSignalsPerTile * static_cast<unsigned>(tt * a.n0);
    out->seg_start[e] = excl[1];
    out->seg_code[e] = e;
    out->seg_start[n + e] = total[1] + excl[2];
    out->seg_code[n + e] = e | (1 << 16);
    done[e] = 0u;
  }
  if (i == 0) {
    out->maxn = a.maxn;
    out->even = a.even;
    out->n_experts = n;
    out->n_seg = 2 * n;
    out->seg_start[2 * n] = total[1] + total[2];
  }
}

// ------------------------------------------------------------------ host helpers
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  if (!fn) fail(PS_ECUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 2D bf16 row-major [rows, cols] tensor map with a {64, box_rows} box, 128B swizzle.
CUtensorMap encode_map(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(PS_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
  return m;
}

// Tensor maps are pure functions of (base, rows, cols, box): resident slabs, staging slots
// and the chunk buffers keep their addresses, so a prefill launch looks its 4 maps per
// expert up instead of encoding them (264 cuTensorMapEncodeTiled calls per DeepSeek layer
// kept the GPU idle ~100 us per layer). Callers hold the prefill mutex.
CUtensorMap make_map(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  struct Key {
    const void* base;
    uint64_t rows, cols;
    uint32_t box;
    bool operator==(const Key& o) const { return base == o.base && rows == o.rows && cols == o.cols && box == o.box; }
  };
  struct Hash {
    size_t operator()(const Key& k) const {
      return std::hash<const void*>()(k.base) ^ (k.rows * 0x9e3779b97f4a7c15ull) ^ (k.cols << 20) ^ k.box;
    }
  };
  static std::unordered_map<Key, CUtensorMap, Hash> cache;
  const Key key{base, rows, cols, box_rows};
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (cache.size() >= 16384) cache.clear();  // bounded: buffers of engines long gone
  const CUtensorMap m = encode_map(base, rows, cols, box_rows);
  cache.emplace(key, m);
  return m;
}

// fp32 row-major [rows, cols] map with a {box_cols, box_rows} box, no swizzle (the y
// output tiles of the token-N kernel, TMA-stored from shared memory; cached like make_map).
CUtensorMap make_map_f32(const void* base, uint64_t rows, uint64_t cols, uint32_t box_cols, uint32_t box_rows) {
  struct Key {
    const void* base;
    uint64_t rows, cols;
    uint32_t bc, br;
    bool operator==(const Key& o) const {
      return base == o.base && rows == o.rows && cols == o.cols && bc == o.bc && br == o.br;
    }
  };
  struct Hash {
    size_t operator()(const Key& k) const {
      return std::hash<const void*>()(k.base) ^ (k.rows * 0x9e3779b97f4a7c15ull) ^ (k.cols << 20) ^ (k.bc << 8) ^ k.br;
    }
  };
  static std::unordered_map<Key, CUtensorMap, Hash> cache;
  const Key key{base, rows, cols, box_cols, box_rows};
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (cache.size() >= 16384) cache.clear();
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 4};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(PS_ECUDA, "cuTensorMapEncodeTiled (f32) failed: " + std::to_string(static_cast<int>(r)));
  cache.emplace(key, m);
  return m;
}

// Persistent device table of tensor maps for the token-N kernel. A map is a pure function
// of (address, rows, cols, box, element size), so an entry is encoded once, copied to the
// device once (in stream order, before the first kernel that uses it) and never modified:
// launches pass indices. Capacity 32768 maps (4 MiB); a full table is emptied after a
// device synchronisation (the engines of a process use ~2 maps per resident slab plus a
// few dozen per chunk size).
struct MapKey {
  const void* base;
  uint64_t rows, cols;
  uint32_t box_cols, box_rows, esize;
  bool operator==(const MapKey& o) const {
    return base == o.base && rows == o.rows && cols == o.cols && box_cols == o.box_cols && box_rows == o.box_rows &&
           esize == o.esize;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    return std::hash<const void*>()(k.base) ^ (k.rows * 0x9e3779b97f4a7c15ull) ^ (k.cols << 20) ^
           (static_cast<size_t>(k.box_cols) << 40) ^ (static_cast<size_t>(k.box_rows) << 50) ^ k.esize;
  }
};
struct MapTable {
  // capacity (maps): PS_MAPTABLE_CAP for tests of the overflow path, else 32768
  const int kCap = [] {
    const char* v = std::getenv("PS_MAPTABLE_CAP");
    const int c = v ? std::atoi(v) : 32768;
    return c >= 64 ? c : 32768;
  }();
  CUtensorMap* dev = nullptr;
  CUtensorMap* host = nullptr;  // pinned mirror: entry i is written once, before its copy
  int used = 0;
  std::unordered_map<MapKey, int, MapKeyHash> index;
  // Called once per launch, before its get()s: room for `n` new entries. A full table
  // (engines come and go, chunk sizes vary) is emptied once every enqueued kernel has run —
  // launches happen under the caller's mutex, so every user of the table is enqueued —
  // and nothing references an entry any more.
  void reserve(int n) {
    if (used + n <= kCap) return;
    PS_CUDA(cudaDeviceSynchronize());
    index.clear();
    used = 0;
  }
  int get(const MapKey& k, cudaStream_t s) {
    auto it = index.find(k);
    if (it != index.end()) return it->second;
    if (!dev) {
      PS_CUDA(cudaMalloc(&dev, sizeof(CUtensorMap) * kCap));
      PS_CUDA(cudaHostAlloc(&host, sizeof(CUtensorMap) * kCap, cudaHostAllocDefault));
    }
    if (used >= kCap) fail(PS_ERUNTIME, "ps_expert_ffn_prefill: tensor-map table: reserve() missing");
    const int i = used++;
    host[i] = k.esize == 4 ? make_map_f32(k.base, k.rows, k.cols, k.box_cols, k.box_rows)
                           : encode_map(k.base, k.rows, k.cols, k.box_rows);
    PS_CUDA(cudaMemcpyAsync(dev + i, host + i, sizeof(CUtensorMap), cudaMemcpyHostToDevice, s));
    index.emplace(k, i);
    return i;
  }
};

// Ring of per-launch weight tensor-map slots (device array + pinned staging). A slot is
// rewritten only after the event recorded behind its last kernels has completed, so no
// launch ever waits on the host for the GPU (on-demand experts are launched while their
// copies are still in flight).
struct MapRing {
  static constexpr int kSlots = 64;
  static constexpr int kPerSlot = 2 * kMaxExperts + 2;  // [a_x, a_h, gate_up maps, down maps] (M-side kernels)
  CUtensorMap* dev = nullptr;
  CUtensorMap* host = nullptr;
  cudaEvent_t ev[kSlots] = {};
  bool used[kSlots] = {};
  int next = 0;
  int acquire() {
    if (!dev) {
      PS_CUDA(cudaMalloc(&dev, sizeof(CUtensorMap) * kSlots * kPerSlot));
      PS_CUDA(cudaHostAlloc(&host, sizeof(CUtensorMap) * kSlots * kPerSlot, cudaHostAllocDefault));
      for (auto& e : ev) PS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const int s = next;
    next = (next + 1) % kSlots;
    if (used[s]) PS_CUDA(cudaEventSynchronize(ev[s]));
    used[s] = true;
    return s;
  }
};

void launch_pair(PrefillParams& p, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    PS_CUDA(cudaFuncSetAttribute(ffn_prefill_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kPairSmemBytes));
    attr = true;
  }
  const int tiles = p.tile_start[p.n_experts];
  if (tiles == 0) return;
  const int grid = 2 * std::min(tiles, kNumSMs / 2);  // one CTA pair per TPC, persistent
  ffn_prefill_pair_kernel<<<grid, kThreads, kPairSmemBytes, s>>>(p);
  PS_LAUNCH_CHECK("ffn_prefill_pair_kernel");
}

// Largest token tile of the token-N kernel: 256 (default) or 128 (PS_TN_MAXN; read per
// call, A/B knob).
int tn_maxn() {
  const char* v = std::getenv("PS_TN_MAXN");
  return v && std::atoi(v) == 128 ? 128 : 256;
}

// Equal-width token tiles for experts with more than MAXN rows (default 1; PS_TN_EVEN=0
// restores MAXN-wide tiles + a remainder tile; read per call, A/B knob).
int tn_even() {
  const char* v = std::getenv("PS_TN_EVEN");
  return v && v[0] == '0' ? 0 : 1;
}

template <int MAXN>
void launch_tn_t(TnParams& p, cudaStream_t s) {
  using G = TnGeo<MAXN>;
  static int max_pairs = 0;
  if (!max_pairs) {
    PS_CUDA(cudaFuncSetAttribute(ffn_prefill_tn_kernel<MAXN>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::kSmem));
    // every pair must be co-resident (a down tile may wait on any pair's gate_up tile)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * (kNumSMs / 2));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = G::kSmem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int clusters = 0;
    PS_CUDA(cudaOccupancyMaxActiveClusters(&clusters, ffn_prefill_tn_kernel<MAXN>, &cfg));
    if (clusters < 1) fail(PS_ECUDA, "ffn_prefill_tn_kernel: no 2-CTA cluster fits on this device");
    max_pairs = std::min(clusters, kNumSMs / 2);
  }
  const int tiles = p.sched_dev ? max_pairs : p.sched.seg_start[p.sched.n_seg];  // device schedule: all pairs
  if (tiles == 0) return;
  const int grid = 2 * std::min(tiles, max_pairs);
  ffn_prefill_tn_kernel<MAXN><<<grid, kThreads, G::kSmem, s>>>(p);
  PS_LAUNCH_CHECK("ffn_prefill_tn_kernel");
}

void launch_tn(TnParams& p, cudaStream_t s, int maxn) {
  if (maxn == 128) launch_tn_t<128>(p, s);
  else launch_tn_t<256>(p, s);
}

// Kernel choice: 0 = single-CTA, 1 = CTA pairs, 2 = auto, 3 = token-N CTA pairs.
// Initial value from PS_PREFILL_PAIR, else auto.
std::atomic<int>& prefill_mode() {
  static std::atomic<int> mode{[] {
    const char* v = std::getenv("PS_PREFILL_PAIR");
    return v && v[0] >= '0' && v[0] <= '3' ? v[0] - '0' : 2;
  }()};
  return mode;
}

void launch(PrefillParams& p, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    PS_CUDA(cudaFuncSetAttribute(ffn_prefill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    attr = true;
  }
  const int tiles = p.tile_start[p.n_experts];
  if (tiles == 0) return;
  const int grid = std::min(tiles, kNumSMs);
  ffn_prefill_kernel<<<grid, kThreads, kSmemBytes, s>>>(p);
  PS_LAUNCH_CHECK("ffn_prefill_kernel");
}

}  // namespace

// Kernel launches one ps_expert_ffn_prefill call makes (engine launch statistics).
int prefill_launches_per_call() {
  const int mode = prefill_mode().load();
  const char* merge = std::getenv("PS_TN_MERGE");
  return (mode == 2 || mode == 3) && !(merge && merge[0] == '0') ? 1 : 2;
}

}  // namespace ps

using namespace ps;

extern "C" ps_status ps_expert_ffn_prefill(const ps_expert_group* group, const int32_t* counts_host,
                                           const int32_t* offsets_host, const uint16_t* x_perm, int total_rows,
                                           int H, int F, uint16_t* h_perm, float* y_perm, void* stream) {
  return guarded([&] {
    require(group && counts_host && offsets_host && x_perm && h_perm && y_perm, "ps_expert_ffn_prefill: null argument");
    require(H % 64 == 0 && F % 128 == 0 && H % 256 == 0,
            "ps_expert_ffn_prefill: needs H % 256 == 0 and F % 128 == 0");
    require(group->n <= kMaxExperts, "ps_expert_ffn_prefill: too many experts");
    cudaStream_t s = as_stream(stream);
    static MapRing ring;
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    const int slot = ring.acquire();
    CUtensorMap* maps_host = ring.host + slot * MapRing::kPerSlot;
    CUtensorMap* maps_dev = ring.dev + slot * MapRing::kPerSlot;

    // CTA pairs compute 256-row M tiles: an expert's last tile pads up to 255 rows
    // instead of 127, yet with ~6 % extra padding (Mixtral, 4096 tokens routed at random)
    // pairs are still 1.03x faster end to end (scripts/prefill_micro.py). Pairs unless
    // their extra padding exceeds 8 % of the routed rows.
    // auto (2) = the token-N kernel: no M padding, one launch for both phases; it matched
    // or beat the M-side kernels at every expert shape measured (profiles/r02_prefill_tn.md)
    const int mode = prefill_mode().load();
    if (mode == 3 || mode == 2) {
      static unsigned* done_dev = nullptr;  // [MapRing::kSlots][kMaxExperts] gate_up signals
      static std::vector<unsigned> done_host(MapRing::kSlots * kMaxExperts, 0u);  // their running targets
      if (!done_dev) {
        PS_CUDA(cudaMalloc(&done_dev, sizeof(unsigned) * MapRing::kSlots * kMaxExperts));
        PS_CUDA(cudaMemset(done_dev, 0, sizeof(unsigned) * MapRing::kSlots * kMaxExperts));
      }
      static MapTable table;
      table.reserve(2 * group->n + 2 * 17 + 1);
      TnParams tp{};
      tp.F = F;
      tp.H = H;
      tp.ph[0].K = H;
      tp.ph[1].K = F;
      tp.ph[0].n_tiles_n = F / 128;
      tp.ph[1].n_tiles_n = H / 256;
      unsigned* shadow = done_host.data() + slot * kMaxExperts;
      const int maxn = tn_maxn();
      tp.sched.maxn = maxn;
      tp.sched.even = tn_even();
      int n = 0;
      bool used_half[17] = {};
      for (int i = 0; i < group->n; ++i) {
        const int e = group->experts[i];
        const int m = counts_host[e];
        if (m == 0) continue;
        const uint16_t* slab = group->slabs[i];
        tp.ph[0].w_idx[n] = table.get(MapKey{slab, 2ull * F, static_cast<uint64_t>(H), 64, 64, 2}, s);
        tp.ph[1].w_idx[n] = table.get(MapKey{slab + 2ull * F * H, static_cast<uint64_t>(H), static_cast<uint64_t>(F),
                                             64, 128, 2}, s);
        const int tt = (m + maxn - 1) / maxn;
        const int ts = tn_tile_width(m, tt, tp.sched.even, maxn);
        const int rem = m - (tt - 1) * ts;
        used_half[((rem + 15) & ~15) / 16] = true;  // last tile: N/2 = 8j rows
        if (tt > 1) used_half[ts / 16] = true;
        tp.sched.gidx[n] = n;
        tp.sched.t_tiles[n] = tt;
        tp.sched.row0[n] = offsets_host[e];
        tp.sched.rows[n] = m;
        for (TnPhase& ph : tp.ph) ph.tile_start[n + 1] = ph.tile_start[n] + tt * ph.n_tiles_n;
        tp.sched.target[n] = shadow[n] + kTnSignalsPerTile * static_cast<unsigned>(tt * tp.ph[0].n_tiles_n);
        ++n;
      }
      if (n == 0) return;
      for (int j = 0; j <= 16; ++j) {
        tp.ph[0].tok_idx[j] = tp.ph[1].tok_idx[j] = -1;
        if (!used_half[j] || j == 0) continue;
        const uint32_t box = static_cast<uint32_t>(8 * j);
        tp.ph[0].tok_idx[j] = table.get(MapKey{x_perm, static_cast<uint64_t>(total_rows), static_cast<uint64_t>(H), 64,
                                               box, 2}, s);
        tp.ph[1].tok_idx[j] = table.get(MapKey{h_perm, static_cast<uint64_t>(total_rows), static_cast<uint64_t>(F), 64,
                                               box, 2}, s);
      }
      tp.ph[0].out_idx = -1;
      tp.ph[1].out_idx = table.get(MapKey{y_perm, static_cast<uint64_t>(total_rows), static_cast<uint64_t>(H), 32,
                                          32, 4}, s);
      tp.maps = table.dev;
      tp.sched.n_experts = n;
      tp.n_group = n;
      tp.done = done_dev + slot * kMaxExperts;
      // PS_TN_LAG: experts between a gate_up segment and its down segment. Default: all
      // gate_up tiles first (DeepSeek shape, same process: lag 10 277 us, all-first 283,
      // lag 6 296, lag 0 554 — the acquires wait; Mixtral: all-first best), knob kept for A/B.
      const int lag = [] {
        const char* v = std::getenv("PS_TN_LAG");
        const int d = v ? std::atoi(v) : kMaxExperts;
        return d < 0 ? 0 : d;
      }();
      // phases: 3 = both (interleaved with lag D), 1 = gate_up only, 2 = down only
      auto build_segments = [&](TnParams& q, int phases) {
        const int D = std::min(lag, n);
        int t = 0;
        TnSched& S = q.sched;
        S.n_seg = 0;
        auto seg = [&](int ph, int e) {
          if (!(phases & (1 << ph))) return;
          S.seg_start[S.n_seg] = t;
          S.seg_code[S.n_seg] = e | (ph << 16);
          t += q.ph[ph].tile_start[e + 1] - q.ph[ph].tile_start[e];
          ++S.n_seg;
        };
        for (int e = 0; e < n; ++e) {
          seg(0, e);
          if (e >= D) seg(1, e - D);
        }
        for (int e = n - D; e < n; ++e) seg(1, e);
        S.seg_start[S.n_seg] = t;
      };
      build_segments(tp, 3);
      tp.ph[0].out = h_perm;
      tp.ph[0].out_ld = F;
      tp.ph[1].out = y_perm;
      tp.ph[1].out_ld = H;
      const char* merge = std::getenv("PS_TN_MERGE");  // A/B knob: 0 runs the phases as two launches
      if (merge && merge[0] == '0') {
        TnParams second = tp;
        build_segments(tp, 1);
        build_segments(second, 2);
        launch_tn(tp, s, maxn);
        launch_tn(second, s, maxn);
      } else {
        launch_tn(tp, s, maxn);
      }
      // the slot's counters advance only once the launch is enqueued (a failed launch
      // leaves them where the next use of the slot expects them)
      for (int i = 0; i < n; ++i) shadow[i] = tp.sched.target[i];
      PS_CUDA(cudaEventRecord(ring.ev[slot], s));
      return;
    }
    const bool pair = mode == 1;
    PrefillParams gu{}, dn{};
    gu.mode = kSwiGLU;
    dn.mode = kStoreF32;
    gu.K = H;
    dn.K = F;
    gu.F = dn.F = F;
    gu.H = dn.H = H;
    gu.n_tiles_n = F / (kBN / 2);
    dn.n_tiles_n = H / kBN;
    int n = 0;
    for (int i = 0; i < group->n; ++i) {
      const int e = group->experts[i];
      const int m = counts_host[e];
      if (m == 0) continue;
      const uint16_t* slab = group->slabs[i];
      maps_host[2 + n] = make_map(slab, 2ull * F, H, kBN / 2);                                          // [Wg; Wu]
      maps_host[2 + group->n + n] = make_map(slab + 2ull * F * H, static_cast<uint64_t>(H), F, kBN / 2);  // Wd
      const int mt = pair ? (m + 2 * kBM - 1) / (2 * kBM) : (m + kBM - 1) / kBM;
      for (PrefillParams* p : {&gu, &dn}) {
        p->m_tiles[n] = mt;
        p->row0[n] = offsets_host[e];
        p->rows[n] = m;
        p->tile_start[n + 1] = p->tile_start[n] + mt * p->n_tiles_n;
      }
      ++n;
    }
    if (n == 0) return;
    gu.n_experts = dn.n_experts = n;
    maps_host[0] = make_map(x_perm, static_cast<uint64_t>(total_rows), H, kBM);
    maps_host[1] = make_map(h_perm, static_cast<uint64_t>(total_rows), F, kBM);
    PS_CUDA(cudaMemcpyAsync(maps_dev, maps_host, sizeof(CUtensorMap) * (2 + 2 * group->n), cudaMemcpyHostToDevice, s));
    gu.a_map = maps_dev;
    dn.a_map = maps_dev + 1;
    gu.b_maps = maps_dev + 2;
    dn.b_maps = maps_dev + 2 + group->n;
    gu.out = h_perm;
    gu.out_ld = F;
    dn.out = y_perm;
    dn.out_ld = H;
    if (pair) {
      launch_pair(gu, s);
      launch_pair(dn, s);
    } else {
      launch(gu, s);
      launch(dn, s);
    }
    PS_CUDA(cudaEventRecord(ring.ev[slot], s));
  });
}

extern "C" ps_status ps_expert_ffn_prefill_dev(const ps_expert_group* group, const int32_t* offsets_dev,
                                               const uint16_t* x_perm, int total_rows, int H, int F,
                                               uint16_t* h_perm, float* y_perm, void* stream) {
  return guarded([&] {
    require(group && offsets_dev && x_perm && h_perm && y_perm, "ps_expert_ffn_prefill_dev: null argument");
    require(H % 256 == 0 && F % 128 == 0, "ps_expert_ffn_prefill_dev: needs H % 256 == 0 and F % 128 == 0");
    require(group->n >= 0 && group->n <= kMaxExperts, "ps_expert_ffn_prefill_dev: too many experts");
    require(total_rows >= 1, "ps_expert_ffn_prefill_dev: total_rows >= 1");
    if (group->n == 0) return;
    cudaStream_t s = as_stream(stream);
    static MapRing ring;
    static MapTable table;
    static TnSched* sched_dev = nullptr;  // [MapRing::kSlots]
    static unsigned* done_dev = nullptr;  // [MapRing::kSlots][kMaxExperts]
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    if (!sched_dev) {
      PS_CUDA(cudaMalloc(&sched_dev, sizeof(TnSched) * MapRing::kSlots));
      PS_CUDA(cudaMalloc(&done_dev, sizeof(unsigned) * MapRing::kSlots * kMaxExperts));
    }
    const int slot = ring.acquire();
    table.reserve(2 * group->n + 2 * 17 + 1);
    TnParams tp{};
    tp.F = F;
    tp.H = H;
    tp.ph[0].K = H;
    tp.ph[1].K = F;
    tp.ph[0].n_tiles_n = F / 128;
    tp.ph[1].n_tiles_n = H / 256;
    TnSchedArgs sa{};
    sa.n_group = group->n;
    sa.maxn = tn_maxn();
    sa.even = tn_even();
    sa.n0 = tp.ph[0].n_tiles_n;
    sa.n1 = tp.ph[1].n_tiles_n;
    for (int i = 0; i < group->n; ++i) {
      const uint16_t* slab = group->slabs[i];
      sa.expert[i] = group->experts[i];
      tp.ph[0].w_idx[i] = table.get(MapKey{slab, 2ull * F, static_cast<uint64_t>(H), 64, 64, 2}, s);
      tp.ph[1].w_idx[i] = table.get(MapKey{slab + 2ull * F * H, static_cast<uint64_t>(H), static_cast<uint64_t>(F),
                                           64, 128, 2}, s);
    }
    tp.ph[0].tok_idx[0] = tp.ph[1].tok_idx[0] = -1;
    for (int j = 1; j <= 16; ++j) {  // every last-tile width: the counts are on the device
      const uint32_t box = static_cast<uint32_t>(8 * j);
      tp.ph[0].tok_idx[j] = table.get(MapKey{x_perm, static_cast<uint64_t>(total_rows), static_cast<uint64_t>(H), 64,
                                             box, 2}, s);
      tp.ph[1].tok_idx[j] = table.get(MapKey{h_perm, static_cast<uint64_t>(total_rows), static_cast<uint64_t>(F), 64,
                                             box, 2}, s);
    }
    tp.ph[0].out_idx = -1;
    tp.ph[1].out_idx = table.get(MapKey{y_perm, static_cast<uint64_t>(total_rows), static_cast<uint64_t>(H), 32, 32, 4}, s);
    tp.maps = table.dev;
    tp.n_group = group->n;
    tp.done = done_dev + slot * kMaxExperts;
    tp.sched_dev = sched_dev + slot;
    tp.ph[0].out = h_perm;
    tp.ph[0].out_ld = F;
    tp.ph[1].out = y_perm;
    tp.ph[1].out_ld = H;
    tn_schedule_kernel<<<1, kMaxExperts, 0, s>>>(offsets_dev, sa, sched_dev + slot, tp.done);
    PS_LAUNCH_CHECK("tn_schedule_kernel");
    launch_tn(tp, s, sa.maxn);
    PS_CUDA(cudaEventRecord(ring.ev[slot], s));
  });
}

extern "C" ps_status ps_set_prefill_kernel(int mode) {
  return guarded([&] {
    require(mode >= 0 && mode <= 3,
            "ps_set_prefill_kernel: mode 0 (single CTA), 1 (CTA pairs), 2 (auto) or 3 (token-N CTA pairs)");
    prefill_mode().store(mode);
  });
}
