// K3 (decode path) — grouped SwiGLU expert FFN as one persistent HBM-streaming kernel.
//
// No reference code exists for the expert FFN; the op is
// y = W_down(SiLU(W_gate x) * (W_up x)) over the experts a
// decode step activates, with per-expert token counts m_e <= 64 per pass.
//
// Design (HBM-bound: algorithmic bytes = sum_e 3*H*F*2):
//  * One launch does gate_up AND down. Work items are 32 weight rows x a K range:
//    gate_up = (expert, 16-row F tile: 16 gate + 16 up rows, K = H); down = (expert,
//    split of F, 32-row H tile). All gate_up items precede all down items; CTA b takes
//    items b, b+G, b+2G, ... (G = one CTA per SM; cooperative launch, all resident).
//  * Per CTA one producer lane streams the weight tiles through a 6-stage ring of
//    32 KiB shared-memory stages with 2D TMA boxes (cp.async.bulk.tensor, {256 cols x 16
//    or 32 rows} = 8-16 KiB per op, mbarrier complete_tx, out-of-bounds rows/cols
//    zero-filled). Measured on B200 (scripts/probes): TMA ops of >= 8 KiB stream at the
//    HBM roofline, 1-2 KiB ops are op-rate bound at 50-60% of it; >= 128 KiB must be in
//    flight per SM. The ring keeps 192 KiB in flight and streams across item and phase
//    boundaries.
//  * 8 consumer warps split each stage's 16 K blocks (2 each). Tokens are the 8-wide N
//    side of mma.sync.m16n8k16 (bf16 in, fp32 accumulate): a dot product is invariant
//    under a common permutation of K, so a lane's A fragment is one 16-byte LDS (rows g
//    and g+8, elements 8t..8t+7 of a 32-wide K block) and its B fragment the matching 16
//    bytes of the activation row, loaded from L1/L2 one stage ahead. (Decode is
//    HBM-bound at m_e <= 64: mma.sync keeps up with the stream; tcgen05 is used on the
//    prefill path where the op is tensor-bound.)
//  * Partials of the 8 warps are reduced through shared memory per item; epilogues:
//    gate_up h = SiLU(g) * u -> bf16 [perm_row, F]; down -> fp32 y_part[split][row][H]
//    (summed in fixed order by K2's combine). Deterministic (no float atomics).
//  * gate_up -> down dependency without a second launch or a grid barrier: each gate_up
//    item bumps a per-(expert, split) counter after its h stores (release); a down item
//    waits (acquire) until every F tile of its split is done, then reads h from L2.
//    Items run in increasing index order per CTA and every gate_up index is below every
//    down index, so a wait never blocks a producer of h; the producer keeps prefetching
//    down weights meanwhile. Counters live in a per-stream workspace of two sets used
//    in alternation: block 0 of a launch zeroes the other set for the next launch (the
//    stream's previous launch, which used it, is complete); a failed launch re-zeroes it
//    on the host side.
//  * Weight tensor maps are encoded on the host once per slab and kept in a device table
//    (immutable entries; the kernel acquire-fences them before first use).
#include <cuda.h>

#include <algorithm>
#include <mutex>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "device_common.cuh"
#include "zslab_format.hpp"

// Timeline hooks for scripts/probes/ffn_trace.cu (which includes this file with
// PS_FFN_TRACE defined); compiled out of the product.
#ifndef PS_FFN_TRACE
#define PS_TRACE(ord, k)
#define PS_STAGE_CHECK(it, k0, hf, kl, mt, a0, a8)
#endif

namespace ps {
namespace {

constexpr int kMaxSplit = 8;
constexpr int kSyncEntries = 64;                 // max entries per launch (sync workspace rows)
constexpr int kCWarps = 8;                       // consumer warps
constexpr int kThreads = (kCWarps + 2) * 32;     // + TMA producer warp + release signaler warp
constexpr int kMailbox = 8;                      // consumer -> signaler queue of finished gate_up items
constexpr int kBarBytes = 2048;                  // mbarriers + per-entry tables; keeps the ring 1 KiB aligned
constexpr int kMaxTokens = 64;                   // tokens per expert per launch (8 * NT, NT <= 8)
constexpr int kHalf = 256;                       // TMA box width (cols)
constexpr int kTileBytes = 16 * kHalf * 2;       // one (16-row m-tile, 256-col half) = 8 KiB
constexpr int kStageBytes = 4 * kTileBytes;      // 32 KiB: MT m-tiles x (4 / MT) halves
constexpr int kMaps = 3;                         // per slab: gate_up {256,16}, gate_up {256,32}, down {256,32}

// smem header: full[8] | empty[8] | posted[kMailbox] | freed[kMailbox] | row0[64] | m[64] | mailbox slots |
// active entries[64] | n_active
static_assert(256 + 3 * kSyncEntries * 4 + kMailbox * 4 + 4 <= kBarBytes, "smem header");

// NT = 8-token groups per expert, MT = 16-row m-tiles per stage (and per item). A stage
// is always 32 KiB: MT = 2 -> 32 rows x 512 cols, MT = 4 -> 64 rows x 256 cols. Activation
// bytes per stage scale with tokens / rows, so more tokens use taller items (MT = 4): the
// activations are re-read from L2 once per item and would otherwise approach the L2
// bandwidth at 16+ tokens per expert.
template <int NT, int MT, bool ZS = false> struct Geo {
  static constexpr int kCols = 2 * 512 / MT;          // K elements per stage
  static constexpr int kKb = 2;                       // K blocks per consumer warp and stage
  static constexpr int kWarpsPerStage = kCols / 64;   // 8 (MT = 2) or 4 (MT = 4)
  static constexpr int kGroups = kCWarps / kWarpsPerStage;  // warp groups taking alternate stages
  static constexpr int kRows = 16 * MT;               // weight rows per item and stage
  static constexpr int kRedBytes = kCWarps * MT * NT * 4 * 32 * 4;
  static constexpr int kStages = (227 * 1024 - kBarBytes - kRedBytes) / kStageBytes > 6
                                     ? 6 : (227 * 1024 - kBarBytes - kRedBytes) / kStageBytes;
  // ZS (z-slab source): no ring; the small footprint lets 2 CTAs share an SM
  static constexpr int kSmem = kBarBytes + (ZS ? 0 : kStages * kStageBytes) + kRedBytes;
  static_assert(kStages >= 3 && kSmem <= 227 * 1024, "decode FFN smem budget");
};

template <int CAP>
struct DecodeParams {
  const CUtensorMap* maps;        // device map table, kMaps per slab: [Wg; Wu] as [2F, H] box {256, 16}
                                  //   and box {256, 32}; Wd as [H, F] box {256, 32}
  int map_idx[CAP];               // table index of entry i's slab
  int n;                          // entries (experts with host-side m_e > tok_base; the
                                  // resident group is launched before the host knows the
                                  // counts, so entries with device-side m_e = 0 are dropped
                                  // in the kernel prologue: only active entries get items)
  int gu_per;                     // gate_up items per entry (F / (8 MT))
  int dn_per;                     // down items per entry (n_split * H / (16 MT))
  int expert[CAP];
  int H, F, k, n_split, kchunk, dn_tiles, tok_base;
  const int32_t* offsets;
  const int32_t* perm_src;
  const uint16_t* x;
  uint16_t* h;
  float* y_part;
  size_t split_stride;
  int* sync;                      // this launch's [kSyncEntries * kMaxSplit] gate_up-items-done counters
  int* sync_next;                 // the other parity's set: zeroed here for the next launch
  const uint8_t* z[CAP];          // ZS: entry i's z-slab (device; lane tile layout of an [H, F] expert)
};

struct Item {
  bool down;
  int i, r0, split, kbeg, kend;
};

// gate_up items: 8*MT F rows (8*MT gate + 8*MT up weight rows) x all of H; down items:
// 16*MT H rows x one split of F. Items enumerate the ACTIVE entries act[0..n_act).
template <int MT, class P>
__device__ __forceinline__ Item item_at(const P& p, const int* act, int n_act, int idx) {
  Item it;
  const int gu_total = n_act * p.gu_per;
  if (idx < gu_total) {
    it.down = false;
    const int j = idx / p.gu_per;
    it.i = act[j];
    it.r0 = (idx - j * p.gu_per) * 8 * MT;
    it.split = it.r0 / p.kchunk;
    it.kbeg = 0;
    it.kend = p.H;
  } else {
    idx -= gu_total;
    it.down = true;
    const int j = idx / p.dn_per;
    it.i = act[j];
    const int local = idx - j * p.dn_per;
    it.split = local / p.dn_tiles;
    it.r0 = (local % p.dn_tiles) * 16 * MT;
    it.kbeg = min(p.F, it.split * p.kchunk);
    it.kend = min(p.F, it.split * p.kchunk + p.kchunk);
  }
  return it;
}

// gate_up items of split s (the down items of that split wait for all of them).
template <int MT, class P>
__device__ __forceinline__ int split_items(const P& p, int s) {
  const int b = min(p.F, s * p.kchunk), e = min(p.F, s * p.kchunk + p.kchunk);
  return (e - b + 8 * MT - 1) / (8 * MT);
}

// Weights are streamed exactly once per launch: load them with an L2 evict-first policy
// so they do not push the small per-layer tensors (router gate, hidden states, ids,
// LLaPor components) out of L2 between layers.
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                       uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// h is produced inside this launch by other SMs: read it from L2 (never a stale L1 line).
__device__ __forceinline__ uint4 ld_cg(const void* p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

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

__device__ __forceinline__ uint4 zero4() { return make_uint4(0u, 0u, 0u, 0u); }

__device__ __forceinline__ uint4 lds128(const uint8_t* p) { return *reinterpret_cast<const uint4*>(p); }

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kCWarps * 32) : "memory"); }

// Activation fragments of this lane for one stage: KB K blocks x NT token groups.
// kw = the warp's first column in this stage.
template <int NT, int KB>
__device__ __forceinline__ void load_act(uint4 (&xv)[KB][NT], const uint16_t* const (&xr)[NT], bool down, int kw,
                                         int kend, int, int tig) {
#pragma unroll
  for (int u = 0; u < KB; ++u) {
    const int kg = kw + u * 32 + 8 * tig;
    const bool kin = kg < kend;
#pragma unroll
    for (int j = 0; j < NT; ++j)
      xv[u][j] = kin && xr[j] ? (down ? ld_cg(xr[j] + kg) : ldg_keep(xr[j] + kg)) : zero4();
  }
}


// ------------------------------------------------------------------ z-slab source (ZS)
// The consumer warps read the experts' weights as z-slabs (zexpert.cu: lossless 11-12 bit
// format, lane tile layout: 16 x 32 tiles) and decode their MMA A fragments in registers —
// no shared-memory ring, no decode pass, no bf16 copy. A consumer warp's share of a ring
// stage (64 K columns x 16 rows of one m-tile) is exactly one 1024-value z block: tile u
// of the block is the warp's K block u, and lane (g, t) needs values 8t..8t+7 of tile rows
// g and g + 8 — 8 lo bytes and 24 (3-bit) or 32 (4-bit) code bits per fragment. Escapes
// (all-ones codes) are ranked by a warp scan in the block's value order (tile, row, lane
// quarter) and patched from the block's escape bytes. The fragments are the bytes a TMA
// load of the decoded slab would deliver, so every partial sum is bitwise the bf16 path's.
struct ZSrc {
  const uint8_t* lo;
  const uint32_t* codes;
  const uint32_t* esc_off;
  const uint8_t* esc;
  uint32_t base, bits, n_esc;
};

__device__ __forceinline__ ZSrc z_src(const uint8_t* z, int H, int F) {
  const uint32_t* h32 = reinterpret_cast<const uint32_t*>(z);
  const uint32_t base = __ldg(h32 + 4), nb = __ldg(h32 + 5), n_esc = __ldg(h32 + 6);
  const uint32_t bits = __ldg(h32 + 10), tiled = __ldg(h32 + 11), th = __ldg(h32 + 12), tf = __ldg(h32 + 13);
  if (!tiled || th != static_cast<uint32_t>(H) || tf != static_cast<uint32_t>(F) || (bits != 3 && bits != 4)) __trap();
  const uint64_t n_pad = static_cast<uint64_t>(nb) * kZBlock;
  ZSrc r;
  r.lo = z + z_lo_off();
  r.codes = reinterpret_cast<const uint32_t*>(z + z_codes_off(n_pad));
  r.esc_off = reinterpret_cast<const uint32_t*>(z + z_escoff_off(n_pad, bits));
  r.esc = z + z_esc_off(n_pad, nb, bits);
  r.base = base;
  r.bits = bits;
  r.n_esc = n_esc;
  return r;
}

// One lane's raw share of a z block: fragments f = 2u + r (tile u, row gid + 8r).
struct ZRaw {
  uint2 lo[4];
  uint32_t c0[4], c1[4];  // the code words holding the fragment's field
  uint32_t eoff, eend;
  bool valid;
};

template <int BITS>
__device__ __forceinline__ void z_fetch(const ZSrc& zs, int b, int gid, int tig, ZRaw& r) {
  r.valid = b >= 0;
  if (!r.valid) return;
  // fragment f = 2u + rr is segment 16u + gid + 8rr of the block: constant offsets from
  // this lane's first fragment
  const uint8_t* lo = zs.lo + static_cast<size_t>(b) * 1024 + gid * 32 + 8 * tig;
  const uint32_t* cw = zs.codes + static_cast<size_t>(b) * (32 * BITS) + gid * BITS;
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const int so = (f >> 1) * 16 + 8 * (f & 1);  // segment offset of fragment f
    r.lo[f] = __ldg(reinterpret_cast<const uint2*>(lo + so * 32));
    if constexpr (BITS == 3) {
      const uint32_t* w = cw + so * 3 + ((24 * tig) >> 5);
      r.c0[f] = __ldg(w);
      r.c1[f] = tig == 3 ? 0u : __ldg(w + 1);
    } else {
      r.c0[f] = __ldg(cw + so * 4 + tig);
      r.c1[f] = 0u;
    }
  }
  r.eoff = __ldg(zs.esc_off + b);
  r.eend = __ldg(zs.esc_off + b + 1);
}

// Decode the 4 fragments of a fetched block (zeros for a block past the K range).
template <int BITS>
__device__ __forceinline__ void z_frags(const ZSrc& zs, const ZRaw& r, int lane, int tig, uint4 (&a)[4]) {
  if (!r.valid) {
#pragma unroll
    for (int f = 0; f < 4; ++f) a[f] = zero4();
    return;
  }
  constexpr bool b3 = BITS == 3;
  const uint32_t base2 = zs.base | (zs.base << 16);
  uint32_t fld[4], em[4];
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    fld[f] = b3 ? __funnelshift_r(r.c0[f], r.c1[f], (24u * tig) & 31u) & 0xffffffu : r.c0[f];
    em[f] = b3 ? fld[f] & (fld[f] >> 1) & (fld[f] >> 2) & 0x249249u
               : fld[f] & (fld[f] >> 1) & (fld[f] >> 2) & (fld[f] >> 3) & 0x11111111u;
#pragma unroll
    for (int pq = 0; pq < 4; ++pq) {  // values 2pq, 2pq + 1
      const uint32_t lw = pq < 2 ? r.lo[f].x : r.lo[f].y;
      const uint32_t L = __byte_perm(lw, 0u, (pq & 1) ? 0x4342u : 0x4140u);
      uint32_t C;
      if (b3) {
        const uint32_t t = fld[f] >> (6 * pq);
        C = (t & 7u) | ((t << 13) & (7u << 16));
      } else {
        const uint32_t t = fld[f] >> (8 * pq);
        C = (t & 15u) | ((t << 12) & (15u << 16));
      }
      const uint32_t v = ((L << 8) & 0x80008000u) | (((C + base2) << 7) & 0x7f807f80u) | (L & 0x007f007fu);
      if (pq == 0) a[f].x = v;
      else if (pq == 1) a[f].y = v;
      else if (pq == 2) a[f].z = v;
      else a[f].w = v;
    }
  }
  if (r.eend == r.eoff) return;  // warp-uniform: no escapes in this block
  // ranks: fragment class f holds keys [32 f, 32 f + 32) of the block's value order in lane order
  int cnt[4];
#pragma unroll
  for (int f = 0; f < 4; ++f) cnt[f] = __popc(em[f]);
  uint32_t S = static_cast<uint32_t>(cnt[0]) | (static_cast<uint32_t>(cnt[1]) << 16);
  uint32_t T = static_cast<uint32_t>(cnt[2]) | (static_cast<uint32_t>(cnt[3]) << 16);
  const uint32_t S0 = S, T0 = T;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t s2 = __shfl_up_sync(0xffffffffu, S, o), t2 = __shfl_up_sync(0xffffffffu, T, o);
    if (lane >= o) {
      S += s2;
      T += t2;
    }
  }
  const uint32_t St = __shfl_sync(0xffffffffu, S, 31), Tt = __shfl_sync(0xffffffffu, T, 31);
  const uint32_t eS = S - S0, eT = T - T0;
  const uint32_t tot0 = St & 0xffffu, tot1 = St >> 16, tot2 = Tt & 0xffffu;
  uint32_t pre[4] = {eS & 0xffffu, tot0 + (eS >> 16), tot0 + tot1 + (eT & 0xffffu), tot0 + tot1 + tot2 + (eT >> 16)};
  uint32_t eb[4];
#pragma unroll
  for (int f = 0; f < 4; ++f) {  // up to 4 escape bytes per fragment in one register
    eb[f] = 0u;
    if (cnt[f] > 0) {
      const uint32_t at = r.eoff + pre[f], a4 = at & ~3u;
      const uint32_t w0 = __ldg(reinterpret_cast<const uint32_t*>(zs.esc + a4));
      const uint32_t w1 = a4 + 4u < zs.n_esc ? __ldg(reinterpret_cast<const uint32_t*>(zs.esc + a4 + 4)) : 0u;
      eb[f] = __funnelshift_r(w0, w1, (at & 3u) * 8u);
    }
  }
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    uint32_t m = em[f];
    uint32_t rk = 0;
    while (m) {
      const int pos = __ffs(m) - 1;
      m &= m - 1;
      const int v = b3 ? pos / 3 : pos / 4;  // value 0..7 of the fragment
      const uint32_t ex = rk < 4 ? (eb[f] >> (8 * rk)) & 0xffu : static_cast<uint32_t>(zs.esc[r.eoff + pre[f] + rk]);
      ++rk;
      const uint32_t sh = 7u + 16u * (v & 1), keep = ~(0xffu << sh), put = ex << sh;
      const int w = v >> 1;
      if (w == 0) a[f].x = (a[f].x & keep) | put;
      else if (w == 1) a[f].y = (a[f].y & keep) | put;
      else if (w == 2) a[f].z = (a[f].z & keep) | put;
      else a[f].w = (a[f].w & keep) | put;
    }
  }
}

template <int NT, int MT, int CAP, bool ZS>
__global__ void __launch_bounds__(kThreads, ZS ? 2 : 1) ffn_decode_kernel(const __grid_constant__ DecodeParams<CAP> p) {
  using G = Geo<NT, MT, ZS>;
  constexpr int KB = G::kKb;
  constexpr int kHalves = 4 / MT;  // 256-col halves per stage
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 8;
  uint64_t* posted = full + 16;                               // gate_up item done (consumer -> signaler)
  uint64_t* freed = full + 16 + kMailbox;                     // mailbox entry free (signaler -> consumer)
  int* s_row0 = reinterpret_cast<int*>(smem + 256);           // per-entry first row of this pass
  int* s_m = s_row0 + kSyncEntries;                           // per-entry rows of this pass (<= 8*NT)
  int* s_mb = s_m + kSyncEntries;                             // mailbox: counter slot of the finished item
  int* s_act = s_mb + kMailbox;                               // active entries (device m_e > 0), in order
  int* s_nact = s_act + kSyncEntries;
  uint8_t* ring = smem + kBarBytes;
  float* red = reinterpret_cast<float*>(ring + (ZS ? 0 : G::kStages * kStageBytes));  // [warp][mt][j][q][lane]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < G::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], G::kWarpsPerStage);
    }
    for (int b = 0; b < kMailbox; ++b) {
      mbar_init(&posted[b], 1);
      mbar_init(&freed[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < p.n; i += blockDim.x) {
    const int e = p.expert[i];
    const int r0 = p.offsets[e] + p.tok_base;
    s_row0[i] = r0;
    s_m[i] = min(8 * NT, p.offsets[e + 1] - r0);
  }
  if (blockIdx.x == 0)  // counters of the next launch (other parity); this stream's previous launch is done
    for (int i = threadIdx.x; i < kSyncEntries * kMaxSplit; i += blockDim.x) p.sync_next[i] = 0;
  __syncthreads();
  if (warp == 0) {  // compact the active entries (ballot + popc, order preserved)
    int na = 0;
    for (int i0 = 0; i0 < p.n; i0 += 32) {
      const int i = i0 + lane;
      const bool on = i < p.n && s_m[i] > 0;
      const unsigned mask = __ballot_sync(0xffffffffu, on);
      if (on) s_act[na + __popc(mask & ((1u << lane) - 1u))] = i;
      na += __popc(mask);
    }
    if (lane == 0) *s_nact = na;
  }
  __syncthreads();
  const int n_act = *s_nact;
  const int total = n_act * (p.gu_per + p.dn_per);

  if (ZS && warp == kCWarps + 1) return;  // ZS: consumer thread 0 publishes (a polling lane costs issue slots)
  if (warp == kCWarps + 1) {
    // ---------------------------------------------------------------- signaler lane
    // Publishes finished gate_up items to the down items of their split: acquire the
    // consumers' mailbox post (which follows their h stores and a CTA barrier), then a
    // gpu-scope fence + counter increment. The fence stalls only this lane, not the
    // consumer warps that feed the ring.
    if (lane != 0) return;
    const int gu_total = n_act * p.gu_per;
    const int mine = gu_total > static_cast<int>(blockIdx.x)
                         ? (gu_total - static_cast<int>(blockIdx.x) + gridDim.x - 1) / gridDim.x : 0;
    for (int q = 0; q < mine; ++q) {
      const int b = q % kMailbox;
      mbar_wait(&posted[b], (q / kMailbox) & 1);
      const int slot = s_mb[b];
      __threadfence();
      atomicAdd(p.sync + slot, 1);
      mbar_arrive(&freed[b]);
    }
    return;
  }

  if (ZS && warp == kCWarps) return;  // z-slab source: the consumers fetch their own weights
  if (warp == kCWarps) {
    // ---------------------------------------------------------------- producer lane
    // Table maps are written by host copies: order them before tensormap-proxy use
    // (also drops any cached descriptor at a reused table slot).
    for (int i = lane; i < kMaps * p.n; i += 32) {
      const CUtensorMap* m = p.maps + kMaps * p.map_idx[i / kMaps] + i % kMaps;
      asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(m) : "memory");
    }
    __syncwarp();
    if (lane != 0) return;
    const uint64_t pol = evict_first_policy();
    uint32_t n = 0;
    int ord = 0;
    for (int idx = blockIdx.x; idx < total; idx += gridDim.x, ++ord) {
      PS_TRACE(ord, 4);
      const Item it = item_at<MT>(p, s_act, n_act, idx);
      const CUtensorMap* maps = p.maps + kMaps * p.map_idx[it.i];
      for (int k0 = it.kbeg; k0 < it.kend; k0 += G::kCols, ++n) {
        const int s = n % G::kStages;
        mbar_wait(&empty[s], ((n / G::kStages) & 1) ^ 1);
        uint8_t* dst = ring + s * kStageBytes;
        mbar_expect_tx(&full[s], kStageBytes);
        // smem tile (m-tile mt, half hf) at (hf * MT + mt) * 8 KiB; a box of 16*b rows
        // fills b consecutive m-tiles.
#pragma unroll
        for (int hf = 0; hf < kHalves; ++hf) {
          uint8_t* d = dst + hf * MT * kTileBytes;
          const int c = k0 + hf * kHalf;
          if (!it.down) {  // m-tiles [0, MT/2): gate rows; [MT/2, MT): up rows
            const CUtensorMap* gm = MT == 2 ? &maps[0] : &maps[1];
            tma_2d(d, gm, &full[s], c, it.r0, pol);
            tma_2d(d + (MT / 2) * kTileBytes, gm, &full[s], c, p.F + it.r0, pol);
          } else {         // MT m-tiles of W_down rows, boxes of 32 rows
#pragma unroll
            for (int b = 0; b < MT / 2; ++b) tma_2d(d + 2 * b * kTileBytes, &maps[2], &full[s], c, it.r0 + 32 * b, pol);
          }
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumer warps
  // Warp w always covers K columns [512 s + 64 w, +64) of every 512-wide window s: with
  // MT = 4 (256-col stages) warp group w/4 takes alternate stages. The per-warp partial
  // sums, and so the results, are bitwise independent of MT (i.e. of the launch's token
  // counts) and of the split of experts into launches.
  const int gid = lane >> 2, tig = lane & 3;
  const int grp = warp / G::kWarpsPerStage;                      // stages st with st % kGroups == grp
  const int wcol = 64 * (warp % G::kWarpsPerStage);              // this warp's columns inside its stage
  const int hf = wcol / kHalf;                                   // its 256-col half
  const int kl0 = wcol % kHalf + 8 * tig;                        // element offset inside the half
  uint32_t n = 0;
  int ord = 0, gu_done = 0;
  for (int idx = blockIdx.x; idx < total; idx += gridDim.x, ++ord) {
    if (threadIdx.x == 0) PS_TRACE(ord, 0);
    const Item it = item_at<MT>(p, s_act, n_act, idx);
    const int row0 = s_row0[it.i], m = s_m[it.i];
    const int slot = it.i * kMaxSplit + it.split;
    if (it.down) {
      if (threadIdx.x == 0) {
        const int need = split_items<MT>(p, it.split);
        while (ld_acquire(p.sync + slot) < need) __nanosleep(32);
      }
      consumer_sync();
    }
    if (threadIdx.x == 0) PS_TRACE(ord, 1);
    const uint16_t* xr[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int t = 8 * j + gid;
      xr[j] = t >= m ? nullptr
              : it.down ? p.h + static_cast<size_t>(row0 + t) * p.F
                        : p.x + static_cast<size_t>(p.perm_src[row0 + t] / p.k) * p.H;
    }
    float acc[MT][NT][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[mt][j][q] = 0.f;

    const int nst = (it.kend - it.kbeg + G::kCols - 1) / G::kCols;
    const int kcol0 = it.kbeg + wcol;  // this warp's first column of stage 0
    // One ring stage st of this item: wait for the TMA fill, 2 K blocks x (MT m-tiles x NT)
    // MMAs, release.
    auto consume = [&](int st, const uint4 (&xv)[KB][NT]) {
      const uint32_t q = n + st;
      const int s = q % G::kStages;
      mbar_wait(&full[s], (q / G::kStages) & 1);
      const uint8_t* sp = ring + s * kStageBytes + hf * MT * kTileBytes;
#pragma unroll
      for (int u = 0; u < KB; ++u) {
        const int off = (kl0 + 32 * u) * 2;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const uint4 a0 = lds128(sp + mt * kTileBytes + gid * (kHalf * 2) + off);
          const uint4 a8 = lds128(sp + mt * kTileBytes + (gid + 8) * (kHalf * 2) + off);
          PS_STAGE_CHECK(it, it.kbeg + st * G::kCols, hf, kl0 + 32 * u, mt, a0, a8);
#pragma unroll
          for (int j = 0; j < NT; ++j) mma_block(acc[mt][j], a0, a8, xv[u][j]);
        }
      }
      // The slot is refilled by TMA (async proxy) after this arrive: order this lane's
      // generic-proxy reads before it (without this fence, refills raced the reads:
      // scripts/probes/ffn_check.cu, non-deterministic h/y).
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    };
    auto load = [&](uint4 (&xv)[KB][NT], int st) {
      load_act<NT, KB>(xv, xr, it.down, kcol0 + st * G::kCols, it.kend, 0, tig);
    };
    constexpr int GS = G::kGroups;
    if constexpr (ZS) {
      // z-slab weights: this warp's z block per m-tile and stage (one stage of raw z data
      // and activations in flight ahead of the decode + MMAs)
      const ZSrc zs = z_src(p.z[it.i], p.H, p.F);
      auto blk = [&](int st, int mt) -> int {
        const int col = kcol0 + st * G::kCols;
        if (col >= it.kend) return -1;
        int r0m, K;
        uint32_t vb;
        if (!it.down) {
          r0m = it.r0 + 16 * (mt < MT / 2 ? mt : mt - MT / 2);
          vb = mt < MT / 2 ? 0u : static_cast<uint32_t>(p.F) * p.H;
          K = p.H;
        } else {
          r0m = it.r0 + 16 * mt;
          vb = 2u * static_cast<uint32_t>(p.F) * p.H;
          K = p.F;
        }
        return static_cast<int>(vb / kZBlock + (((r0m >> 4) * (K >> 5) + (col >> 5)) >> 1));
      };
      // no register prefetch: 2 CTAs per SM (20 warps) hide the load latency instead
      auto run = [&](auto bits_tag) {
        constexpr int BITS = decltype(bits_tag)::value;
        for (int st = grp; st < nst; st += GS) {
          ZRaw ra[MT];
          uint4 xa[KB][NT];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) z_fetch<BITS>(zs, blk(st, mt), gid, tig, ra[mt]);
          load(xa, st);
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            uint4 a[4];
            z_frags<BITS>(zs, ra[mt], lane, tig, a);
#pragma unroll
            for (int u = 0; u < KB; ++u)
#pragma unroll
              for (int j = 0; j < NT; ++j) mma_block(acc[mt][j], a[2 * u], a[2 * u + 1], xa[u][j]);
          }
        }
      };
      if (zs.bits == 3) run(std::integral_constant<int, 3>{});
      else run(std::integral_constant<int, 4>{});
    } else if constexpr (NT >= 8) {  // 64 tokens: no registers for a second activation buffer
      uint4 xa[KB][NT];
      for (int st = grp; st < nst; st += GS) {
        load(xa, st);
        consume(st, xa);
      }
    } else {
      // Activations for this warp's next stage are loaded during the current one (L1/L2
      // latency overlaps the weight stream).
      uint4 xa[KB][NT], xb[KB][NT];
      if (grp < nst) load(xa, grp);
      for (int st = grp; st < nst; st += 2 * GS) {
        if (st + GS < nst) load(xb, st + GS);
        consume(st, xa);
        if (st + GS >= nst) break;
        if (st + 2 * GS < nst) load(xa, st + 2 * GS);
        consume(st + GS, xb);
      }
    }
    n += nst;

    if (threadIdx.x == 0) PS_TRACE(ord, 2);
    // Cross-warp reduction through shared memory + epilogue.
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) red[(((warp * MT + mt) * NT + j) * 4 + q) * 32 + lane] = acc[mt][j][q];
    consumer_sync();
    // Value v = (mt, j, q, lane): c0,c1 -> row gid, tokens 2*tig+{0,1}; c2,c3 -> row gid+8.
    // gate_up pairs gate m-tile mt with up m-tile mt + MT/2.
    const int n_mt = it.down ? MT : MT / 2;
    for (int v = threadIdx.x; v < n_mt * NT * 4 * 32; v += kCWarps * 32) {
      const int ln = v & 31, q = (v >> 5) & 3, j = (v >> 7) % NT, mt = (v >> 7) / NT;
      const int t = 8 * j + 2 * (ln & 3) + (q & 1);
      const int r = 16 * mt + (ln >> 2) + (q >> 1) * 8;
      float s0 = 0.f, s1 = 0.f;
#pragma unroll
      for (int w = 0; w < kCWarps; ++w) {
        s0 += red[(((w * MT + mt) * NT + j) * 4 + q) * 32 + ln];
        if (!it.down) s1 += red[(((w * MT + mt + MT / 2) * NT + j) * 4 + q) * 32 + ln];
      }
      if (t < m) {
        if (!it.down) {
          const int f = it.r0 + r;
          if (f < p.F) {
            const float hv = s0 / (1.0f + expf(-s0)) * s1;
            p.h[static_cast<size_t>(row0 + t) * p.F + f] = f32_to_bf16_rne(hv);
          }
        } else {
          const int d = it.r0 + r;
          if (d < p.H) p.y_part[it.split * p.split_stride + static_cast<size_t>(row0 + t) * p.H + d] = s0;
        }
      }
    }
    consumer_sync();  // red reusable; every h store of this item issued
    if (threadIdx.x == 0) PS_TRACE(ord, 3);
    if (ZS && !it.down) {  // publish this F tile to the down items of its split
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(p.sync + slot, 1);
      }
    } else if (!it.down) {  // hand this F tile to the signaler (mbarrier arrive = release.cta)
      if (threadIdx.x == 0) {
        const int b = gu_done % kMailbox;
        mbar_wait(&freed[b], ((gu_done / kMailbox) & 1) ^ 1);
        s_mb[b] = slot;
        mbar_arrive(&posted[b]);
      }
      ++gu_done;
    }
  }
}

// ------------------------------------------------------------------ host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(ptr);
  });
  if (!fn) fail(PS_ECUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// Row-major bf16 [rows, cols], box {256 cols, box_rows}, no swizzle, OOB -> zeros.
CUtensorMap encode_rows(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kHalf), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(PS_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
  return m;
}

// Device table of weight tensor maps, kMaps per (slab, H, F), uploaded once on first use
// (stream-ordered before the launch) and read by the kernel through a global pointer:
// keeps the launch parameter block small (64 experts x 3 maps would be 24 KiB) and
// costs no host encode or copy in steady state (engine slabs are fixed pool slots).
int slab_map_index(const uint16_t* slab, int H, int F, cudaStream_t s, const CUtensorMap** table) {
  struct Key {
    int dev;
    const void* p;
    int H, F;
    bool operator==(const Key& o) const { return dev == o.dev && p == o.p && H == o.H && F == o.F; }
  };
  struct Hash {
    size_t operator()(const Key& k) const {
      return std::hash<const void*>()(k.p) ^ (static_cast<size_t>(k.H) * 0x9e3779b97f4a7c15ull) ^
             (static_cast<size_t>(k.F) << 20) ^ static_cast<size_t>(k.dev);
    }
  };
  struct Table {
    CUtensorMap* dev = nullptr;
    int used = 0;
  };
  constexpr int kCap = 8192;  // slabs per device (kMaps maps each, 3 MiB)
  static std::mutex mu;
  static std::unordered_map<Key, int, Hash> index;
  static std::unordered_map<int, Table> tables;
  int dev = 0;
  PS_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  Table& t = tables[dev];
  if (!t.dev) PS_CUDA(cudaMalloc(&t.dev, sizeof(CUtensorMap) * kMaps * kCap));
  *table = t.dev;
  auto it = index.find(Key{dev, slab, H, F});
  if (it != index.end()) return it->second;
  if (t.used == kCap) {  // full: start over (the kernel's acquire fence drops stale descriptors)
    PS_CUDA(cudaStreamSynchronize(s));
    for (auto i = index.begin(); i != index.end();) i = i->first.dev == dev ? index.erase(i) : std::next(i);
    t.used = 0;
  }
  CUtensorMap m[kMaps];
  m[0] = encode_rows(slab, 2ull * F, static_cast<uint64_t>(H), 16);
  m[1] = encode_rows(slab, 2ull * F, static_cast<uint64_t>(H), 32);
  m[2] = encode_rows(slab + 2ull * F * H, static_cast<uint64_t>(H), static_cast<uint64_t>(F), 32);
  const int idx = t.used++;
  PS_CUDA(cudaMemcpyAsync(t.dev + kMaps * idx, m, sizeof(m), cudaMemcpyHostToDevice, s));  // pageable: staged now
  index.emplace(Key{dev, slab, H, F}, idx);
  return idx;
}

struct DeviceInfo {
  int sms = 0;
  std::unordered_map<const void*, int> blocks_per_sm;
};

DeviceInfo& device_info() {
  static std::mutex mu;
  static std::unordered_map<int, DeviceInfo> m;
  int dev = 0;
  PS_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  DeviceInfo& d = m[dev];
  if (d.sms == 0) PS_CUDA(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev));
  return d;
}

// Two counter sets per (device, stream), used by alternate launches: launch L counts in
// set L&1 and zeroes set (L+1)&1, which the previous launch on this stream (ordered
// before it) used. No reset atomics on the critical path.
struct SyncSets {
  int* cur;
  int* next;
};
SyncSets sync_workspace(cudaStream_t s) {
  struct Ws {
    int* base = nullptr;
    uint64_t launches = 0;
  };
  static std::mutex mu;
  static std::unordered_map<uint64_t, Ws> ws;
  int dev = 0;
  PS_CUDA(cudaGetDevice(&dev));
  const uint64_t key = (static_cast<uint64_t>(dev) << 56) ^ reinterpret_cast<uint64_t>(s);
  std::lock_guard<std::mutex> g(mu);
  Ws& w = ws[key];
  const size_t set = static_cast<size_t>(kSyncEntries) * kMaxSplit;
  if (!w.base) {
    PS_CUDA(cudaMalloc(&w.base, sizeof(int) * 2 * set));
    PS_CUDA(cudaMemset(w.base, 0, sizeof(int) * 2 * set));
  }
  const int par = static_cast<int>(w.launches++ & 1);
  return SyncSets{w.base + par * set, w.base + (par ^ 1) * set};
}

template <int NT, int MT, int CAP, bool ZS>
void launch(const DecodeParams<CAP>& p, cudaStream_t s) {
  DeviceInfo& d = device_info();
  const size_t smem = Geo<NT, MT, ZS>::kSmem;
  const void* fn = reinterpret_cast<const void*>(ffn_decode_kernel<NT, MT, CAP, ZS>);
  int& bps = d.blocks_per_sm[fn];
  if (bps == 0) {
    PS_CUDA(cudaFuncSetAttribute(ffn_decode_kernel<NT, MT, CAP, ZS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    PS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, ffn_decode_kernel<NT, MT, CAP, ZS>, kThreads, smem));
    require(bps >= 1, "ffn_decode_kernel: does not fit on an SM");
  }
  const int total = p.n * (p.gu_per + p.dn_per);  // upper bound (entries with m_e = 0 are dropped on device)
  const int grid = std::min(total, bps * d.sms);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // co-residency: the h dependency spins
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;  // measured cost of the attribute: ~1.5 us per launch
  PS_CUDA(cudaLaunchKernelEx(&cfg, ffn_decode_kernel<NT, MT, CAP, ZS>, p));
}

struct Shape {
  int H, F, k, n_split, kchunk;
};

// Items per entry for m-tiles-per-item MT: gate_up F/(8 MT), down n_split * H/(16 MT).
constexpr int mt_for(int NT) { return NT == 1 || NT == 8 ? 2 : 4; }

template <int CAP>
void run_group(const ps_expert_group* group, int base, int count, const int32_t* counts_host, const Shape& sh,
               int tok_base, int NT, const int32_t* offsets, const int32_t* perm_src, const uint16_t* x, uint16_t* h,
               float* y_part, size_t split_stride, cudaStream_t s, const uint8_t* const* zslabs = nullptr) {
  DecodeParams<CAP> p;
  p.n = 0;
  p.H = sh.H;
  p.F = sh.F;
  p.k = sh.k;
  p.n_split = sh.n_split;
  p.kchunk = sh.kchunk;
  const int MT = mt_for(NT);
  p.gu_per = (sh.F + 8 * MT - 1) / (8 * MT);
  p.dn_tiles = (sh.H + 16 * MT - 1) / (16 * MT);
  p.dn_per = p.dn_tiles * sh.n_split;
  p.tok_base = tok_base;
  p.offsets = offsets;
  p.perm_src = perm_src;
  p.x = x;
  p.h = h;
  p.y_part = y_part;
  p.split_stride = split_stride;
  for (int i = base; i < base + count; ++i) {
    const int e = group->experts[i];
    if (counts_host[e] <= tok_base) continue;
    if (zslabs) {
      p.z[p.n] = zslabs[i];
      p.map_idx[p.n] = 0;
      p.maps = nullptr;
    } else {
      p.map_idx[p.n] = slab_map_index(group->slabs[i], sh.H, sh.F, s, &p.maps);
      p.z[p.n] = nullptr;
    }
    p.expert[p.n] = e;
    ++p.n;
  }
  if (p.n == 0) return;
  const SyncSets ss = sync_workspace(s);  // one parity flip per launch
  p.sync = ss.cur;
  p.sync_next = ss.next;
  try {
    if (zslabs) {  // z-slab source: decode batches of <= 8 tokens per expert
      launch<1, mt_for(1), CAP, true>(p, s);
    } else {
      switch (NT) {
        case 1: launch<1, mt_for(1), CAP, false>(p, s); break;
        case 2: launch<2, mt_for(2), CAP, false>(p, s); break;
        case 4: launch<4, mt_for(4), CAP, false>(p, s); break;
        default: launch<8, mt_for(8), CAP, false>(p, s); break;
      }
    }
  } catch (...) {
    // The failed launch never zeroed the next launch's counter set: do it here, so the
    // next launch on this stream does not count on top of stale values.
    cudaMemsetAsync(ss.next, 0, sizeof(int) * kSyncEntries * kMaxSplit, s);
    throw;
  }
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" {

int ps_ffn_down_splits(int H, int F) {
  // Down items are (split of F) x (16*MT rows of H), gate_up items (16*MT weight rows) x
  // H; splitting F into ~F/H parts keeps both item kinds about the same size, which
  // balances the persistent CTAs (Mixtral F=14336, H=4096: 4 splits of 3584).
  const int s = (F + H / 2) / std::max(H, 1);
  return std::min(std::max(s, 1), kMaxSplit);
}

ps_status ps_expert_ffn(const ps_expert_group* group, const int32_t* counts_host, const int32_t* offsets,
                        const int32_t* perm_src, int k, const uint16_t* x, int H, int F, uint16_t* h,
                        float* y_part, int n_split, int total_rows, void* stream) {
  return guarded([&] {
    require(group && counts_host && offsets && perm_src && x && h && y_part, "ps_expert_ffn: null argument");
    require(H >= 8 && F >= 8 && H % 8 == 0 && F % 8 == 0, "ps_expert_ffn: H and F must be multiples of 8");
    require(n_split >= 1 && n_split <= kMaxSplit && group->n >= 0 && group->n <= PS_MAX_GROUP,
            "ps_expert_ffn: bad group/split");
    cudaStream_t s = as_stream(stream);
    int max_m = 0;
    for (int i = 0; i < group->n; ++i) {
      require(group->slabs[i] != nullptr, "ps_expert_ffn: null slab");
      max_m = std::max(max_m, counts_host[group->experts[i]]);
    }
    if (max_m == 0) return;
    require(total_rows >= max_m, "ps_expert_ffn: total_rows smaller than an expert's rows");
    Shape sh{H, F, k, n_split, 0};
    sh.kchunk = (F + n_split - 1) / n_split;
    sh.kchunk = (sh.kchunk + 31) / 32 * 32;  // gate_up items (8*MT <= 32 F rows) never straddle a split
    const size_t split_stride = static_cast<size_t>(total_rows) * H;

    // Token passes of <= 64 rows per expert (decode has m_e <= 64: one pass).
    for (int tok_base = 0; tok_base < max_m; tok_base += kMaxTokens) {
      const int pass_m = std::min(kMaxTokens, max_m - tok_base);
      const int NT = pass_m <= 8 ? 1 : pass_m <= 16 ? 2 : pass_m <= 32 ? 4 : 8;
      for (int base = 0; base < group->n; base += kSyncEntries) {
        const int count = std::min(kSyncEntries, group->n - base);
        if (count <= 8)
          run_group<8>(group, base, count, counts_host, sh, tok_base, NT, offsets, perm_src, x, h, y_part,
                       split_stride, s);
        else
          run_group<kSyncEntries>(group, base, count, counts_host, sh, tok_base, NT, offsets, perm_src, x, h, y_part,
                                  split_stride, s);
      }
    }
  });
}

ps_status ps_expert_ffn_zslab(const ps_expert_group* group, const void* const* zslabs, const int32_t* counts_host,
                              const int32_t* offsets, const int32_t* perm_src, int k, const uint16_t* x, int H, int F,
                              uint16_t* h, float* y_part, int n_split, int total_rows, void* stream) {
  return guarded([&] {
    require(group && zslabs && counts_host && offsets && perm_src && x && h && y_part,
            "ps_expert_ffn_zslab: null argument");
    require(H % 64 == 0 && F % 64 == 0 && H >= 64 && F >= 64, "ps_expert_ffn_zslab: H and F must be multiples of 64");
    require(n_split >= 1 && n_split <= kMaxSplit && group->n >= 0 && group->n <= PS_MAX_GROUP,
            "ps_expert_ffn_zslab: bad group/split");
    require(3ull * H * F < (1ull << 32), "ps_expert_ffn_zslab: expert too large");
    cudaStream_t s = as_stream(stream);
    int max_m = 0;
    for (int i = 0; i < group->n; ++i) {
      require(zslabs[i] != nullptr, "ps_expert_ffn_zslab: null z-slab");
      max_m = std::max(max_m, counts_host[group->experts[i]]);
    }
    if (max_m == 0) return;
    require(max_m <= 8, "ps_expert_ffn_zslab: more than 8 tokens for an expert (decode batches only)");
    require(total_rows >= max_m, "ps_expert_ffn_zslab: total_rows smaller than an expert's rows");
    Shape sh{H, F, k, n_split, 0};
    sh.kchunk = (F + n_split - 1) / n_split;
    sh.kchunk = (sh.kchunk + 31) / 32 * 32;
    require(sh.kchunk % 64 == 0, "ps_expert_ffn_zslab: the down split width must be a multiple of 64");
    const size_t split_stride = static_cast<size_t>(total_rows) * H;
    const auto* z = reinterpret_cast<const uint8_t* const*>(zslabs);
    for (int base = 0; base < group->n; base += kSyncEntries) {
      const int count = std::min(kSyncEntries, group->n - base);
      if (count <= 8)
        run_group<8>(group, base, count, counts_host, sh, 0, 1, offsets, perm_src, x, h, y_part, split_stride, s, z);
      else
        run_group<kSyncEntries>(group, base, count, counts_host, sh, 0, 1, offsets, perm_src, x, h, y_part,
                                split_stride, s, z);
    }
  });
}

}  // extern "C"
