// Lossless transfer format for host-resident expert slabs ("z-slabs").
//
// The non-resident experts cross PCIe (55 GB/s) while the GPU streams HBM at 6.5 TB/s,
// so every byte not sent over PCIe is worth ~100x its decode cost. bf16 weights of a
// trained (or, here, synthetic Gaussian) matrix use only a narrow band of the 8-bit
// exponent field: a slab is stored as
//   lo    [n]        u8   sign << 7 | 7-bit mantissa        (verbatim)
//   codes [n*bits/8]      `bits` = 3 or 4 per value (32 values = `bits` little-endian
//                         words per lane segment): code c < 2^bits - 1 means
//                         exponent = base + c; all ones is an escape
//   esc_off [nb + 1] u32  prefix of escapes per 1024-value block
//   esc   [n_esc]    u8   raw exponents of the escaped values, in value order
// i.e. 11-12 bits per value + 1 byte per escape (70-75 % of bf16; the encoder picks the
// code width with the smaller estimated size). Decoding is bit-exact
// (tests/test_gpu_zexpert.py), so every downstream result is identical to loading the
// raw slab. Encoder: host C++ (at engine create, multithreaded over blocks); decoder:
// one warp per 1024-value block, 32 values per lane, escape ranks by a warp scan, the
// block staged in shared memory and written as coalesced 512-byte warp stores (1.41 B
// read + 2 B written per value; v4 for 3-bit codes at 0.77 of HBM, v3 for 4-bit at 0.82).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "device_common.cuh"
#include "zslab_format.hpp"

namespace ps {
namespace {

// Escapes (all-ones codes) among a lane's 32 codes with word-level bit tricks.
template <int BITS>
__device__ __forceinline__ int z_count_esc(const uint32_t (&cw)[BITS + 1]) {
  if constexpr (BITS == 4) {
    int c = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) c += __popc(cw[q] & (cw[q] >> 1) & (cw[q] >> 2) & (cw[q] >> 3) & 0x11111111u);
    return c;
  } else {  // 96 bits: codes 0..20 in the low 64 bits, codes 21..31 from bit 63 on
    const uint64_t lo = static_cast<uint64_t>(cw[0]) | (static_cast<uint64_t>(cw[1]) << 32);
    const uint64_t hi = (static_cast<uint64_t>(cw[1]) >> 31) | (static_cast<uint64_t>(cw[2]) << 1);
    return __popcll(lo & (lo >> 1) & (lo >> 2) & 0x1249249249249249ull) +
           __popcll(hi & (hi >> 1) & (hi >> 2) & 0x49249249ull);
  }
}

constexpr int kZEscStage = 256;  // staged escapes per block (more: read from global)

// Two codes (values i, i+1; i even) as 16-bit lanes of one word: the 2*BITS bits at
// BITS*i of the lane's little-endian code words (funnel shift, constant after unrolling).
template <int BITS>
__device__ __forceinline__ uint32_t z_code_pair(const uint32_t (&cw)[BITS + 1], int i) {
  const int bit = BITS * i, w = bit >> 5, sh = bit & 31;
  const uint32_t t = __funnelshift_r(cw[w], cw[w + 1], sh);
  constexpr uint32_t m = (1u << BITS) - 1u;
  return (t & m) | ((t << (16 - BITS)) & (m << 16));
}

// Decoder (PS_ZDECODE=3, default): one warp per 1024-value block, 32 consecutive values
// per lane (2 x 16 B of lo bytes, BITS words of codes), branch-free: every value is
// assembled as if its code were not an escape, two bf16 at a time in 32-bit registers —
//   L = two lo bytes in 16-bit lanes (one byte permute), C = two codes (funnel shift,
//   masks), out = ((L << 8) & 0x80008000) | ((C + (base | base << 16)) << 7) | (L & 0x007f007f)
// — then the lane's escapes (all-ones codes, ~3 % of values at 3-bit codes, found with
// word-level bit tricks) are patched. The block is staged in shared memory (XOR-swizzled
// 16-byte chunks) and written out as whole sectors: 512 contiguous bytes per warp store
// (row-major) or 64 per 4 lanes (a tiled slab's 32-value tile rows). Per-lane 16-byte
// stores at a 64-byte stride made every write a half-sector request and the L1->XBAR
// request path the limiter (72 % busy, DRAM 40 %; profiles/r02_z_decode.md). The next
// block's loads are issued before the current block is assembled (software pipeline).
// Row-major start of the 32-value tile row at tiled index v, in 32-bit arithmetic
// (z_untile's 64-bit division is a ~100-instruction subroutine; the host checks
// n = 3HF < 2^32 for tiled slabs).
__device__ __forceinline__ uint32_t z_untile32(uint32_t v, uint32_t H, uint32_t F) {
  const uint32_t fh = F * H;
  const uint32_t base = v < fh ? 0u : (v < 2u * fh ? fh : 2u * fh);
  const uint32_t K = v < 2u * fh ? H : F;
  const uint32_t t = v - base, tile = t >> 9, i = (t >> 5) & 15u, nkb = K >> 5;
  const uint32_t rb = tile / nkb, kb = tile - rb * nkb;
  return base + (rb * 16u + i) * K + kb * 32u;
}

template <int BITS>
__global__ void __launch_bounds__(256, 4)
z_decode_kernel(const uint8_t* __restrict__ z, uint64_t n, uint32_t base, uint32_t nb, uint32_t tile_h,
                uint32_t tile_f, uint16_t* __restrict__ out) {
  __shared__ uint8_t s_esc[8][kZEscStage];
  __shared__ __align__(16) uint4 s_out[8][128];  // per warp: 32 lanes x 4 chunks of 8 bf16
  const uint64_t n_pad = static_cast<uint64_t>(nb) * kZBlock;
  const uint8_t* lo = z + z_lo_off();
  const uint32_t* codes = reinterpret_cast<const uint32_t*>(z + z_codes_off(n_pad));
  const uint32_t* esc_off = reinterpret_cast<const uint32_t*>(z + z_escoff_off(n_pad, BITS));
  const uint8_t* esc = z + z_esc_off(n_pad, nb, BITS);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t base2 = base | (base << 16);
  uint8_t* se = s_esc[warp];
  uint4* so = s_out[warp];
  // swizzled 16-byte slot: a quarter-warp's 16-byte stores (fixed q) hit 8 distinct bank groups
  auto chunk = [](int ln, int q) { return ln * 4 + (q ^ ((ln >> 1) & 3)); };
  struct Blk {
    uint4 l0, l1;
    uint32_t cw[BITS];
    uint32_t eoff, eend;
  };
  auto fetch = [&](uint32_t bb, Blk& k) {
    const uint64_t seg = static_cast<uint64_t>(bb) * 32 + lane;
    k.l0 = __ldg(reinterpret_cast<const uint4*>(lo + seg * 32));
    k.l1 = __ldg(reinterpret_cast<const uint4*>(lo + seg * 32 + 16));
#pragma unroll
    for (int q = 0; q < BITS; ++q) k.cw[q] = __ldg(codes + seg * BITS + q);
    k.eoff = __ldg(esc_off + bb);
    k.eend = __ldg(esc_off + bb + 1);
  };
  uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  Blk nxt{};
  if (b < nb) fetch(b, nxt);
  for (; b < nb; b += warps) {
    const Blk cur = nxt;
    if (b + warps < nb) fetch(b + warps, nxt);
    const uint64_t vb = static_cast<uint64_t>(b) * kZBlock;
    const uint64_t v0 = vb + 32u * lane;
    uint32_t cw[BITS + 1];
#pragma unroll
    for (int q = 0; q < BITS; ++q) cw[q] = cur.cw[q];
    cw[BITS] = 0;
    const uint32_t lw[8] = {cur.l0.x, cur.l0.y, cur.l0.z, cur.l0.w, cur.l1.x, cur.l1.y, cur.l1.z, cur.l1.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // 8 values -> one 16-byte chunk in shared memory
      uint32_t pk[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int p = 4 * q + h;  // values 2p, 2p+1
        const uint32_t L = __byte_perm(lw[p >> 1], 0u, (p & 1) ? 0x4342u : 0x4140u);
        pk[h] = ((L << 8) & 0x80008000u) | ((z_code_pair<BITS>(cw, 2 * p) + base2) << 7) | (L & 0x007f007fu);
      }
      so[chunk(lane, q)] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
    if (cur.eend != cur.eoff) {  // escapes in this block (warp-uniform): patch them in smem
      const uint32_t eoff = cur.eoff;
      const uint32_t n_stage = min(cur.eend - eoff, static_cast<uint32_t>(kZEscStage));
      for (uint32_t k = lane; k < n_stage; k += 32) se[k] = esc[eoff + k];
      __syncwarp();
      const int n_e = z_count_esc<BITS>(cw);
      int incl = n_e;  // warp exclusive scan of escape counts -> this lane's first rank
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      uint32_t e_at = eoff + static_cast<uint32_t>(incl - n_e);
      uint16_t* so16 = reinterpret_cast<uint16_t*>(so);
      auto patch = [&](int i) {  // value i of this lane, in value (= escape) order
        const uint32_t r = e_at - eoff;
        const uint32_t ex = r < static_cast<uint32_t>(kZEscStage) ? se[r] : esc[e_at];
        ++e_at;
        const uint32_t l = __ldg(lo + v0 + i);  // lo byte (L1 hit)
        so16[chunk(lane, i >> 3) * 8 + (i & 7)] = static_cast<uint16_t>(((l & 0x80u) << 8) | (ex << 7) | (l & 0x7fu));
      };
      if constexpr (BITS == 3) {
        const uint64_t A = static_cast<uint64_t>(cw[0]) | (static_cast<uint64_t>(cw[1]) << 32);
        const uint64_t B = (static_cast<uint64_t>(cw[1]) >> 31) | (static_cast<uint64_t>(cw[2]) << 1);
        uint64_t ma = A & (A >> 1) & (A >> 2) & 0x1249249249249249ull;  // codes 0..20: bit 3i
        uint64_t mb = B & (B >> 1) & (B >> 2) & 0x49249249ull;          // codes 21..31
        while (ma) {
          const int pos = __ffsll(static_cast<long long>(ma)) - 1;
          ma &= ma - 1;
          patch(pos / 3);
        }
        while (mb) {
          const int pos = __ffsll(static_cast<long long>(mb)) - 1;
          mb &= mb - 1;
          patch(21 + pos / 3);
        }
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t m = cw[q] & (cw[q] >> 1) & (cw[q] >> 2) & (cw[q] >> 3) & 0x11111111u;
          while (m) {
            const int pos = __ffs(m) - 1;
            m &= m - 1;
            patch(8 * q + pos / 4);
          }
        }
      }
    }
    __syncwarp();
    // write-out: 16-byte chunk c = lane + 32 r is values 8c..8c+7 of the block (segment
    // c / 4 = the lane that assembled it, quarter c % 4)
    if (vb + kZBlock <= n) {
      const uint64_t my_off = tile_h ? static_cast<uint64_t>(z_untile32(static_cast<uint32_t>(v0), tile_h, tile_f))
                                     : v0;  // this lane's segment start
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int c = lane + 32 * r, sl = c >> 2, q = c & 3;
        const uint64_t seg_off = __shfl_sync(0xffffffffu, my_off, sl);
        *reinterpret_cast<uint4*>(out + seg_off + 8 * q) = so[chunk(sl, q)];
      }
    } else {  // the last, partial block of a row-major slab (tiled slabs are whole blocks)
      const uint16_t* so16 = reinterpret_cast<const uint16_t*>(so);
      for (int i = 0; i < 32; ++i)
        if (v0 + i < n) out[v0 + i] = so16[chunk(lane, i >> 3) * 8 + (i & 7)];
    }
    __syncwarp();  // staging buffers are reused by the next block
  }
}

// v4 (default, PS_ZDECODE=3 selects v3): v3's structure with ~25 % fewer instructions —
//  * assembly per bf16 pair: one byte permute DUPLICATES each lo byte into both halves of
//    its 16-bit lane ([b b]: bit 15 = sign, bits 0-6 = mantissa), so the value is
//    (P & 0x807f807f) | ((C << 7) + (base << 7 | base << 23)) — PRMT, funnel shift, three
//    mask/shift ops, one IMAD, one LOP3 instead of eleven instructions;
//  * escapes: per-value 32-bit masks (codes 0-10 | 11-20 | 21-31), index by a multiply-high
//    division, and the patch rewrites only the exponent of the value already staged in
//    shared memory (no dependent global load of its lo byte). Requires base + 2^BITS - 1 <
//    256 (an escape code's provisional exponent must not carry into the sign); the host
//    falls back to v3 otherwise.
template <int BITS>
__global__ void __launch_bounds__(256, 4)
z_decode_kernel_v4(const uint8_t* __restrict__ z, uint64_t n, uint32_t base, uint32_t nb, uint32_t tile_h,
                   uint32_t tile_f, uint16_t* __restrict__ out) {
  const uint32_t mh = tile_h ? static_cast<uint32_t>((0x100000000ull + (tile_h >> 5) - 1) / (tile_h >> 5)) : 0u;
  const uint32_t mf = tile_f ? static_cast<uint32_t>((0x100000000ull + (tile_f >> 5) - 1) / (tile_f >> 5)) : 0u;
  __shared__ uint8_t s_esc[8][kZEscStage];
  __shared__ __align__(16) uint4 s_out[8][128];
  const uint64_t n_pad = static_cast<uint64_t>(nb) * kZBlock;
  const uint8_t* lo = z + z_lo_off();
  const uint32_t* codes = reinterpret_cast<const uint32_t*>(z + z_codes_off(n_pad));
  const uint32_t* esc_off = reinterpret_cast<const uint32_t*>(z + z_escoff_off(n_pad, BITS));
  const uint8_t* esc = z + z_esc_off(n_pad, nb, BITS);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t ebase = (base << 7) | (base << 23);
  uint8_t* se = s_esc[warp];
  uint4* so = s_out[warp];
  const uint32_t so_s = static_cast<uint32_t>(__cvta_generic_to_shared(so));
  auto chunk = [](int ln, int q) { return ln * 4 + (q ^ ((ln >> 1) & 3)); };
  // Software pipeline: block b is assembled while the lo/code words AND the first 64
  // escape bytes of block b + W are in flight, and the escape offsets of block b + 2W
  // (the escape loads need their block's offsets: a same-iteration dependent load
  // stalled on the offset, profiles/r02_z_decode.md).
  struct Blk {
    uint4 l0, l1;
    uint32_t cw[BITS];
    uint32_t eoff, eend;
    uint32_t e0, e1;  // escape bytes eoff + lane, eoff + 32 + lane (when present)
  };
  auto fetch = [&](uint32_t bb, uint32_t eo, uint32_t ee, Blk& k) {
    const uint64_t seg = static_cast<uint64_t>(bb) * 32 + lane;
    k.l0 = __ldg(reinterpret_cast<const uint4*>(lo + seg * 32));
    k.l1 = __ldg(reinterpret_cast<const uint4*>(lo + seg * 32 + 16));
#pragma unroll
    for (int q = 0; q < BITS; ++q) k.cw[q] = __ldg(codes + seg * BITS + q);
    k.eoff = eo;
    k.eend = ee;
    k.e0 = eo + lane < ee ? __ldg(esc + eo + lane) : 0u;
    k.e1 = eo + 32 + lane < ee ? __ldg(esc + eo + 32 + lane) : 0u;
  };
  uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  Blk nxt{};
  uint32_t o2_lo = 0, o2_hi = 0;  // escape offsets of block b + W (then of b + 2W)
  if (b < nb) {
    fetch(b, __ldg(esc_off + b), __ldg(esc_off + b + 1), nxt);
    if (b + warps < nb) {
      o2_lo = __ldg(esc_off + b + warps);
      o2_hi = __ldg(esc_off + b + warps + 1);
    }
  }
  for (; b < nb; b += warps) {
    const Blk cur = nxt;
    if (b + warps < nb) {
      fetch(b + warps, o2_lo, o2_hi, nxt);
      if (b + 2 * warps < nb) {
        o2_lo = __ldg(esc_off + b + 2 * warps);
        o2_hi = __ldg(esc_off + b + 2 * warps + 1);
      }
    }
    const uint64_t vb = static_cast<uint64_t>(b) * kZBlock;
    const uint64_t v0 = vb + 32u * lane;
    uint32_t cw[BITS + 1];
#pragma unroll
    for (int q = 0; q < BITS; ++q) cw[q] = cur.cw[q];
    cw[BITS] = 0;
    const uint32_t lw[8] = {cur.l0.x, cur.l0.y, cur.l0.z, cur.l0.w, cur.l1.x, cur.l1.y, cur.l1.z, cur.l1.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t pk[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int p = 4 * q + h;  // values 2p, 2p+1
        const uint32_t P = __byte_perm(lw[p >> 1], 0u, (p & 1) ? 0x3322u : 0x1100u);
        pk[h] = (P & 0x807f807fu) | (z_code_pair<BITS>(cw, 2 * p) * 128u + ebase);
      }
      so[chunk(lane, q)] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
    if (cur.eend != cur.eoff) {  // escapes in this block (warp-uniform)
      const uint32_t eoff = cur.eoff;
      const uint32_t n_stage = min(cur.eend - eoff, static_cast<uint32_t>(kZEscStage));
      se[lane] = static_cast<uint8_t>(cur.e0);  // prefetched with the block
      se[32 + lane] = static_cast<uint8_t>(cur.e1);
      for (uint32_t k = 64 + lane; k < n_stage; k += 32) se[k] = esc[eoff + k];  // > 64 escapes: rare
      __syncwarp();
      // per-value escape masks: m[0] codes 0-10 at bit 3i (BITS 3) ..., see v3's word tricks
      uint32_t m[3];
      int first[3];
      if constexpr (BITS == 3) {
        const uint64_t A = static_cast<uint64_t>(cw[0]) | (static_cast<uint64_t>(cw[1]) << 32);
        const uint64_t B = (static_cast<uint64_t>(cw[1]) >> 31) | (static_cast<uint64_t>(cw[2]) << 1);
        const uint64_t ma = A & (A >> 1) & (A >> 2) & 0x1249249249249249ull;  // codes 0..20: bit 3i
        m[0] = static_cast<uint32_t>(ma);         // codes 0..10 (bits 0..30)
        m[1] = static_cast<uint32_t>(ma >> 32);   // codes 11..20 (bits 1..28 = 3i - 32)
        m[2] = static_cast<uint32_t>(B & (B >> 1) & (B >> 2) & 0x49249249ull);  // codes 21..31: bit 3(i-21)
        first[0] = 0;
        first[1] = 32;
        first[2] = 63;  // (pos + 63) / 3 = 21 + pos / 3
      } else {
        m[0] = m[1] = m[2] = 0;
        first[0] = first[1] = first[2] = 0;
      }
      int n_e;
      if constexpr (BITS == 3) {
        n_e = __popc(m[0]) + __popc(m[1]) + __popc(m[2]);
      } else {
        n_e = z_count_esc<BITS>(cw);
      }
      int incl = n_e;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      uint32_t r = static_cast<uint32_t>(incl - n_e);  // this lane's first escape rank in the block
      const uint32_t key = (lane >> 1) & 3;
      auto patch = [&](int i, uint32_t ex) {
        const uint32_t addr = so_s + static_cast<uint32_t>(lane * 64) + ((static_cast<uint32_t>(i >> 3) ^ key) << 4) +
                              static_cast<uint32_t>((i & 7) * 2);
        uint32_t v;
        asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(addr));
        v = (v & 0x807fu) | (ex << 7);
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(static_cast<uint16_t>(v)));
      };
      if (cur.eend - eoff <= static_cast<uint32_t>(kZEscStage)) {  // all staged (the common case)
        if constexpr (BITS == 3) {
          // one loop over the three masks in value order (the warp runs max-over-lanes
          // iterations: one merged loop instead of three)
          while (m[0] | m[1] | m[2]) {
            const int w = m[0] ? 0 : (m[1] ? 1 : 2);
            const uint32_t mm = w == 0 ? m[0] : (w == 1 ? m[1] : m[2]);
            const uint32_t pos = static_cast<uint32_t>(__ffs(mm) - 1) + (w == 0 ? 0u : (w == 1 ? 32u : 63u));
            const uint32_t cleared = mm & (mm - 1);
            if (w == 0) m[0] = cleared;
            else if (w == 1) m[1] = cleared;
            else m[2] = cleared;
            patch(static_cast<int>(__umulhi(pos, 0x55555556u)), se[r++]);
          }
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t mm = cw[q] & (cw[q] >> 1) & (cw[q] >> 2) & (cw[q] >> 3) & 0x11111111u;
            while (mm) {
              const int pos = __ffs(mm) - 1;
              mm &= mm - 1;
              patch(8 * q + (pos >> 2), se[r++]);
            }
          }
        }
      } else {  // > kZEscStage escapes in the block: ranks past the staged ones read global memory
        auto ex_at = [&](uint32_t rk) {
          return rk < static_cast<uint32_t>(kZEscStage) ? static_cast<uint32_t>(se[rk]) : static_cast<uint32_t>(esc[eoff + rk]);
        };
        if constexpr (BITS == 3) {
#pragma unroll
          for (int w = 0; w < 3; ++w) {
            uint32_t mm = m[w];
            while (mm) {
              const int pos = __ffs(mm) - 1;
              mm &= mm - 1;
              patch(static_cast<int>(__umulhi(static_cast<uint32_t>(pos + first[w]), 0x55555556u)), ex_at(r++));
            }
          }
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t mm = cw[q] & (cw[q] >> 1) & (cw[q] >> 2) & (cw[q] >> 3) & 0x11111111u;
            while (mm) {
              const int pos = __ffs(mm) - 1;
              mm &= mm - 1;
              patch(8 * q + (pos >> 2), ex_at(r++));
            }
          }
        }
      }
    }
    __syncwarp();
    if (vb + kZBlock <= n) {
      if (tile_h) {
        // A tiled block is two 16x32 tiles of the same 16 weight rows, K-adjacent (K/64 is
        // whole, checked by the host): segment i and 16 + i are one 128 B run of output row
        // i. The block's (row, column) origin is computed once per block (warp-uniform);
        // each warp store writes 4 rows x 128 B (whole lines).
        const uint32_t vbl = static_cast<uint32_t>(vb), fh = tile_f * tile_h;
        const uint32_t mat = vbl < fh ? 0u : (vbl < 2u * fh ? 1u : 2u);
        const uint32_t K = mat < 2 ? tile_h : tile_f;
        const uint32_t T = (vbl - mat * fh) >> 9;  // even tile index within the matrix
        const uint32_t rb = __umulhi(T, mat < 2 ? mh : mf), kb = T - rb * (K >> 5);
        uint16_t* blk = out + mat * fh + rb * 16u * K + kb * 32u;
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          const int row = 4 * rr + (lane >> 3), j = lane & 7;
          const int sl = j < 4 ? row : 16 + row, q = j & 3;
          *reinterpret_cast<uint4*>(blk + static_cast<uint32_t>(row) * K + 8 * j) = so[chunk(sl, q)];
        }
      } else {
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          const int c = lane + 32 * rr, sl = c >> 2, q = c & 3;
          *reinterpret_cast<uint4*>(out + vb + 8 * c) = so[chunk(sl, q)];
        }
      }
    } else {
      const uint16_t* so16 = reinterpret_cast<const uint16_t*>(so);
      for (int i = 0; i < 32; ++i)
        if (v0 + i < n) out[v0 + i] = so16[chunk(lane, i >> 3) * 8 + (i & 7)];
    }
    __syncwarp();
  }
}

// Code i of a lane's 32 (v1 decoder): BITS bits at BITS*i of its little-endian words.
template <int BITS>
__device__ __forceinline__ uint32_t z_code(const uint32_t (&cw)[BITS + 1], int i) {
  const int bit = BITS * i, w = bit >> 5, sh = bit & 31;
  uint32_t c = cw[w] >> sh;
  if (sh + BITS > 32) c |= cw[w + 1] << (32 - sh);
  return c & ((1u << BITS) - 1u);
}

// v1 decoder (round 1; PS_ZDECODE=1): one warp per 1024-value block, 32 values per lane: lane L's codes are the BITS 32-bit
// words at BITS*L of the block's code region (bit BITS*i.. of a little-endian array).
// Codes are extracted twice (escape count for the warp scan, then the values) instead of
// kept in registers: <= 64 registers, 4 CTAs of 256 threads per SM for latency hiding.
// The block's escape bytes (contiguous, ~30 at 3-bit codes) are staged in shared memory
// by one coalesced warp load, so a lane's escapes cost a shared-memory read instead of a
// dependent global load after the scan.

template <int BITS>
__global__ void __launch_bounds__(256, 4)
z_decode_kernel_v1(const uint8_t* __restrict__ z, uint64_t n, uint32_t base, uint32_t nb, uint32_t tile_h,
                uint32_t tile_f, uint16_t* __restrict__ out) {
  constexpr uint32_t kEsc = (1u << BITS) - 1u;
  __shared__ uint8_t s_esc[8][kZEscStage];
  const uint64_t n_pad = static_cast<uint64_t>(nb) * kZBlock;
  const uint8_t* lo = z + z_lo_off();
  const uint32_t* codes = reinterpret_cast<const uint32_t*>(z + z_codes_off(n_pad));
  const uint32_t* esc_off = reinterpret_cast<const uint32_t*>(z + z_escoff_off(n_pad, BITS));
  const uint8_t* esc = z + z_esc_off(n_pad, nb, BITS);
  const int lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nb; b += warps) {
    const uint64_t seg = static_cast<uint64_t>(b) * 32 + lane;  // this lane's 32-value segment
    const uint64_t v0 = seg * 32;
    const uint4 l0 = *reinterpret_cast<const uint4*>(lo + v0);
    const uint4 l1 = *reinterpret_cast<const uint4*>(lo + v0 + 16);
    uint32_t cw[BITS + 1];
#pragma unroll
    for (int q = 0; q < BITS; ++q) cw[q] = codes[seg * BITS + q];
    cw[BITS] = 0;
    const uint32_t eoff = esc_off[b], eend = esc_off[b + 1];
    uint8_t* se = s_esc[threadIdx.x >> 5];
    const uint32_t n_stage = min(eend - eoff, static_cast<uint32_t>(kZEscStage));
    for (uint32_t k = lane; k < n_stage; k += 32) se[k] = esc[eoff + k];
    __syncwarp();
    const int n_e = z_count_esc<BITS>(cw);
    int incl = n_e;  // warp inclusive scan of escape counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    uint32_t e_at = eoff + static_cast<uint32_t>(incl - n_e);
    const uint32_t lw[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
    const bool full = v0 + 32 <= n;
    // tiled slabs (n = 3HF, a multiple of 1024, so always full): a lane's segment is one
    // 32-value tile row, 64 contiguous bytes of the row-major output
    uint16_t* dst = tile_h ? out + z_untile(v0, tile_h, tile_f) : out + v0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // 8 values -> one 16-byte store
      uint32_t pk[4];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = 8 * q + j;
        const uint32_t c = z_code<BITS>(cw, i);
        const uint32_t l = (lw[i >> 2] >> (8 * (i & 3))) & 0xffu;
        uint32_t ex = base + c;
        if (c == kEsc) {
          const uint32_t r = e_at - eoff;
          ex = r < static_cast<uint32_t>(kZEscStage) ? se[r] : esc[e_at];
          ++e_at;
        }
        const uint32_t v = ((l & 0x80u) << 8) | (ex << 7) | (l & 0x7fu);
        if (j & 1) pk[j >> 1] |= v << 16;
        else pk[j >> 1] = v;
      }
      if (full) {
        reinterpret_cast<uint4*>(dst)[q] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      } else {
        for (int j = 0; j < 8 && v0 + 8 * q + j < n; ++j)
          out[v0 + 8 * q + j] = static_cast<uint16_t>(pk[j >> 1] >> (16 * (j & 1)));
      }
    }
    __syncwarp();  // every lane done with s_esc before the next block restages it
  }
}

// One 1024-value block: lo bytes, packed `bits`-bit codes; returns the escape count.
uint32_t z_encode_block(const uint16_t* __restrict__ src, uint8_t* __restrict__ lo, uint8_t* __restrict__ codes,
                        uint32_t base, uint32_t bits) {
  // separate simple loops (auto-vectorised): sign+mantissa bytes, codes, escapes
  const uint32_t esc = z_escape(bits);
  uint8_t cd[kZBlock];
  for (int k = 0; k < kZBlock; ++k) {
    const uint32_t v = src[k];
    lo[k] = static_cast<uint8_t>(((v >> 8) & 0x80u) | (v & 0x7fu));
    const uint32_t d = ((v >> 7) & 0xffu) - base;  // wraps below base
    cd[k] = static_cast<uint8_t>(d < esc ? d : esc);
  }
  uint32_t c = 0;
  for (int k = 0; k < kZBlock; ++k) c += cd[k] == esc;
  if (bits == 4) {
    for (int k = 0; k < kZBlock / 2; ++k) codes[k] = static_cast<uint8_t>(cd[2 * k] | (cd[2 * k + 1] << 4));
  } else {  // 3 bits: 32 values -> 3 little-endian words per segment
    uint32_t* w = reinterpret_cast<uint32_t*>(codes);
    for (int sgm = 0; sgm < kZBlock / 32; ++sgm) {
      uint64_t acc[2] = {0, 0};
#pragma GCC unroll 32
      for (int i = 0; i < 32; ++i) {
        const int bit = 3 * i;
        if (bit < 64) {
          acc[0] |= static_cast<uint64_t>(cd[32 * sgm + i]) << bit;
          if (bit + 3 > 64) acc[1] |= static_cast<uint64_t>(cd[32 * sgm + i]) >> (64 - bit);
        } else {
          acc[1] |= static_cast<uint64_t>(cd[32 * sgm + i]) << (bit - 64);
        }
      }
      w[3 * sgm] = static_cast<uint32_t>(acc[0]);
      w[3 * sgm + 1] = static_cast<uint32_t>(acc[0] >> 32);
      w[3 * sgm + 2] = static_cast<uint32_t>(acc[1]);
    }
  }
  return c;
}

template <typename F>
void parallel_blocks(uint32_t nb, int threads, F&& f) {
  threads = std::max(1, std::min<int>(threads, static_cast<int>(nb)));
  std::vector<std::thread> ts;
  for (int t = 0; t < threads; ++t)
    ts.emplace_back([&, t] {
      for (uint32_t b = static_cast<uint32_t>(static_cast<uint64_t>(nb) * t / threads);
           b < static_cast<uint64_t>(nb) * (t + 1) / threads; ++b)
        f(b);
    });
  for (auto& th : ts) th.join();
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" {

uint64_t ps_zslab_bound(uint64_t n) {
  const uint64_t nb = (n + kZBlock - 1) / kZBlock, n_pad = nb * kZBlock;
  return z_esc_off(n_pad, static_cast<uint32_t>(nb), 4) + n_pad;  // worst case: 4-bit codes, every value escaped
}

ps_status ps_zslab_encode(const uint16_t* slab, uint64_t n, uint8_t* out, uint64_t cap, uint64_t* out_bytes,
                          int threads) {
  return guarded([&] {
    require(slab && out && out_bytes && n > 0, "ps_zslab_encode: bad arguments");
    const uint32_t nb = static_cast<uint32_t>((n + kZBlock - 1) / kZBlock);
    const uint64_t n_pad = static_cast<uint64_t>(nb) * kZBlock;
    require(cap >= z_esc_off(n_pad, nb, 3), "ps_zslab_encode: output too small");
    threads = threads > 0 ? threads : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    // exponent histogram (sampled every 61st value) -> for code widths 3 and 4, the
    // window of 2^bits - 1 exponents with most mass; the width with the smaller
    // estimated size (codes + one byte per escape) wins.
    std::vector<uint64_t> hist(256, 0);
    uint64_t samples = 0;
    for (uint64_t i = 0; i < n; i += 61, ++samples) hist[(slab[i] >> 7) & 0xff]++;
    uint32_t bits = 4, base = 0;
    double best_size = 1e300;
    for (uint32_t bw : {3u, 4u}) {
      const uint32_t win = z_escape(bw);
      uint32_t bb = 0;
      uint64_t best = 0;
      for (uint32_t b = 0; b + win <= 256; ++b) {
        uint64_t s = 0;
        for (uint32_t j = 0; j < win; ++j) s += hist[b + j];
        if (s > best) {
          best = s;
          bb = b;
        }
      }
      const double esc_frac = samples ? 1.0 - static_cast<double>(best) / samples : 0.0;
      const double size = bw / 8.0 + esc_frac;  // bytes per value beyond the lo byte
      if (size < best_size) {
        best_size = size;
        bits = bw;
        base = bb;
      }
    }
    if (const char* v = std::getenv("PS_ZSLAB_BITS")) {  // tests pin the width
      const uint32_t forced = static_cast<uint32_t>(std::atoi(v));
      if (forced == 3 || forced == 4) {
        bits = forced;
        uint64_t best = 0;
        for (uint32_t b = 0; b + z_escape(bits) <= 256; ++b) {
          uint64_t s = 0;
          for (uint32_t j = 0; j < z_escape(bits); ++j) s += hist[b + j];
          if (s > best) {
            best = s;
            base = b;
          }
        }
      }
    }
    const uint32_t escv = z_escape(bits);
    require(cap >= z_esc_off(n_pad, nb, bits), "ps_zslab_encode: output too small");
    uint8_t* lo = out + z_lo_off();
    uint8_t* codes = out + z_codes_off(n_pad);
    uint32_t* esc_off = reinterpret_cast<uint32_t*>(out + z_escoff_off(n_pad, bits));
    auto exp_of = [&](uint64_t i) { return i < n ? static_cast<uint32_t>((slab[i] >> 7) & 0xff) : base; };
    auto escaped = [&](uint32_t e) { return e < base || e >= base + escv; };
    // pass 1: lo bytes, codes, escape count per block (the ragged tail is padded with
    // code-0 values)
    std::vector<uint32_t> cnt(nb);
    parallel_blocks(nb, threads, [&](uint32_t b) {
      const uint64_t i0 = static_cast<uint64_t>(b) * kZBlock;
      uint16_t tmp[kZBlock];
      const uint16_t* src = slab + i0;
      if (i0 + kZBlock > n) {
        for (int k = 0; k < kZBlock; ++k) tmp[k] = i0 + k < n ? slab[i0 + k] : static_cast<uint16_t>(base << 7);
        src = tmp;
      }
      cnt[b] = z_encode_block(src, lo + i0, codes + i0 * bits / 8, base, bits);
    });
    esc_off[0] = 0;
    for (uint32_t b = 0; b < nb; ++b) esc_off[b + 1] = esc_off[b] + cnt[b];
    const uint64_t n_esc = esc_off[nb];
    const uint64_t bytes = (z_esc_off(n_pad, nb, bits) + n_esc + 15) / 16 * 16;
    require(cap >= bytes, "ps_zslab_encode: output too small for the escapes");
    uint8_t* esc = out + z_esc_off(n_pad, nb, bits);
    // pass 2: escaped exponents in value order
    parallel_blocks(nb, threads, [&](uint32_t b) {
      if (cnt[b] == 0) return;  // most blocks of a weight slab have no escape
      uint32_t at = esc_off[b];
      for (uint64_t i = static_cast<uint64_t>(b) * kZBlock; i < static_cast<uint64_t>(b + 1) * kZBlock; ++i) {
        const uint32_t e = exp_of(i);
        if (escaped(e)) esc[at++] = static_cast<uint8_t>(e);
      }
    });
    ZHeader h{};
    h.magic = kZMagic;
    h.n = n;
    h.base = base;
    h.nb = nb;
    h.n_esc = n_esc;
    h.bytes = bytes;
    h.code_bits = bits;
    std::memcpy(out, &h, sizeof(h));
    *out_bytes = bytes;
  });
}

ps_status ps_zslab_info(const uint8_t* z_host, uint64_t* n, uint64_t* bytes, uint64_t* n_esc) {
  return guarded([&] {
    require(z_host != nullptr, "ps_zslab_info: null");
    ZHeader h;
    std::memcpy(&h, z_host, sizeof(h));
    require(h.magic == kZMagic, "ps_zslab_info: not a z-slab");
    if (n) *n = h.n;
    if (bytes) *bytes = h.bytes;
    if (n_esc) *n_esc = h.n_esc;
  });
}

// z-slab of an expert slab in the host lane's tile layout (ps_host_slab_tile): the same
// encoding of the tiled values, header marked so ps_zslab_decode emits row-major order and
// the lane's z path reads tiles as sequential streams.
ps_status ps_zslab_encode_tiled(const uint16_t* slab_tiled, int H, int F, uint8_t* out, uint64_t cap,
                                uint64_t* out_bytes, int threads) {
  const uint64_t n = 3ull * static_cast<uint64_t>(H) * static_cast<uint64_t>(F);
  if (!(H > 0 && F > 0 && H % 32 == 0 && F % 32 == 0)) {
    set_last_error("ps_zslab_encode_tiled: H, F must be positive multiples of 32");
    return PS_EINVAL;
  }
  const ps_status st = ps_zslab_encode(slab_tiled, n, out, cap, out_bytes, threads);
  if (st != PS_OK) return st;
  ZHeader h;
  std::memcpy(&h, out, sizeof(h));
  h.tiled = 1;
  h.tile_h = static_cast<uint32_t>(H);
  h.tile_f = static_cast<uint32_t>(F);
  std::memcpy(out, &h, sizeof(h));
  return PS_OK;
}

// Device decode: z (device copy of the z-slab) -> out [n] bf16. The header fields are
// passed from the host (the caller keeps the host z-slab), so no device read-back.
ps_status ps_zslab_decode(const uint8_t* z_dev, const uint8_t* z_host_header, uint16_t* out, void* stream) {
  return guarded([&] {
    require(z_dev && z_host_header && out, "ps_zslab_decode: null argument");
    ZHeader h;
    std::memcpy(&h, z_host_header, sizeof(h));
    require(h.magic == kZMagic, "ps_zslab_decode: not a z-slab");
    const int threads = 256;
    const int grid = static_cast<int>(std::min<uint64_t>((static_cast<uint64_t>(h.nb) * 32 + threads - 1) / threads,
                                                         4 * 148));
    require(h.code_bits == 3 || h.code_bits == 4, "ps_zslab_decode: bad code width");
    const uint32_t th = h.tiled ? h.tile_h : 0, tf = h.tiled ? h.tile_f : 0;
    require(!h.tiled || (th % 32 == 0 && tf % 32 == 0 && th && tf && h.n == 3ull * th * tf && h.n < (1ull << 32)),
            "ps_zslab_decode: bad tiled header");
    const int version = [] {  // PS_ZDECODE=1 / 3: the round-1 / v3 decoders (A/B), else v4
      const char* v = std::getenv("PS_ZDECODE");
      return v && (v[0] == '1' || v[0] == '3') ? v[0] - '0' : 4;
    }();
    if (version == 1) {
      const int grid1 = static_cast<int>(std::min<uint64_t>((static_cast<uint64_t>(h.nb) * 32 + threads - 1) / threads,
                                                            4 * 148));
      if (h.code_bits == 3)
        z_decode_kernel_v1<3><<<grid1, threads, 0, as_stream(stream)>>>(z_dev, h.n, h.base, h.nb, th, tf, out);
      else
        z_decode_kernel_v1<4><<<grid1, threads, 0, as_stream(stream)>>>(z_dev, h.n, h.base, h.nb, th, tf, out);
    } else if (version == 4 && h.code_bits == 3 && h.base + z_escape(h.code_bits) < 256 &&
               (!h.tiled || (th % 64 == 0 && tf % 64 == 0))) {
      // v4 for 3-bit codes (151 -> 119 us per Mixtral expert); 4-bit codes (0.01 % escapes)
      // gain nothing from its escape path and stay on v3 (113-116 us either way)
      z_decode_kernel_v4<3><<<grid, threads, 0, as_stream(stream)>>>(z_dev, h.n, h.base, h.nb, th, tf, out);
    } else if (h.code_bits == 3) {
      z_decode_kernel<3><<<grid, threads, 0, as_stream(stream)>>>(z_dev, h.n, h.base, h.nb, th, tf, out);
    } else {
      z_decode_kernel<4><<<grid, threads, 0, as_stream(stream)>>>(z_dev, h.n, h.base, h.nb, th, tf, out);
    }
    PS_LAUNCH_CHECK("z_decode_kernel");
  });
}

}  // extern "C"
