// Host expert lane — the reference's Resource::Cpu (simulator.cpp:139-146; cpu_cost =
// beta*m + C, cost_model.cpp:34-37) made real: a SwiGLU expert FFN computed by the host
// cores straight from the pinned host copy of a non-resident expert, so PreSched's
// cpu_set runs concurrently with the PCIe loads of its ondemand_seq instead of being
// loaded too. Opt-in (ps_engine_config.host_threads); the GPU
// path never falls back to it.
//
// Bound: host DRAM bandwidth (every weight byte is read once per expert; m <= 64
// tokens reuse it from registers/L1), so the kernel is an AVX512-BF16 GEMV:
// VDPBF16PS multiplies bf16 pairs into fp32 accumulators, one weight vector (32 bf16)
// feeds up to 8 tokens. Phase 1 (gate_up): each thread owns a contiguous range of the
// F rows of W_gate and W_up, h = bf16(SiLU(g) * u) (the same bf16 rounding point as
// the GPU path, k3_ffn_decode.cu). Phase 2 (down): each thread owns a range of the H
// rows of W_down, y fp32. Numerics: fp32 accumulation in a different order than the
// GPU -> compared with the f64 oracle at the bf16 tolerance (tests/test_host_lane.py).
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <thread>
#include <vector>

#include <pthread.h>
#include <sched.h>
#include <sys/syscall.h>
#include <unistd.h>

#include "common.hpp"
#include "zslab_format.hpp"

namespace ps {
namespace {

// CPUs for the lane: the LAST `n` CPUs of the process's affinity set, so the engine and
// I/O threads (and the Python caller) keep the first ones. Empty = no pinning
// (PS_HOST_LANE_PIN=0 or fewer CPUs than threads).
std::vector<int> lane_cpus(int n) {
  const char* v = std::getenv("PS_HOST_LANE_PIN");
  if (v && v[0] == '0') return {};
  cpu_set_t set;
  CPU_ZERO(&set);
  if (sched_getaffinity(0, sizeof(set), &set) != 0) return {};
  std::vector<int> cpus;
  for (int c = 0; c < CPU_SETSIZE; ++c)
    if (CPU_ISSET(c, &set)) cpus.push_back(c);
  if (static_cast<int>(cpus.size()) < n + 2) return {};
  return std::vector<int>(cpus.end() - n, cpus.end());
}

void pin_self(int cpu) {
  cpu_set_t set;
  CPU_ZERO(&set);
  CPU_SET(cpu, &set);
  pthread_setaffinity_np(pthread_self(), sizeof(set), &set);
}

// Persistent pool: the caller is worker 0; workers wait on a generation counter
// (C++20 atomic wait = futex), run their share, count down. Workers are pinned to
// lane_cpus() (one CPU each); the caller pins itself with pin_caller().
class Pool {
 public:
  explicit Pool(int threads) : n_(std::max(1, threads)), cpus_(lane_cpus(n_)) {
    for (int i = 1; i < n_; ++i)
      workers_.emplace_back([this, i] {
        if (!cpus_.empty()) pin_self(cpus_[i]);
        loop(i);
      });
  }
  void pin_caller() const {
    if (!cpus_.empty()) pin_self(cpus_[0]);
  }
  ~Pool() {
    stop_ = true;
    gen_.fetch_add(1, std::memory_order_release);
    gen_.notify_all();
    for (auto& t : workers_) t.join();
  }
  int size() const { return n_; }
  // fn(tid) on every thread; returns when all are done.
  void run(const std::function<void(int)>& fn) {
    fn_ = &fn;
    remaining_.store(n_ - 1, std::memory_order_relaxed);
    gen_.fetch_add(1, std::memory_order_release);
    gen_.notify_all();
    fn(0);
    for (int r = remaining_.load(std::memory_order_acquire); r != 0; r = remaining_.load(std::memory_order_acquire))
      remaining_.wait(r, std::memory_order_acquire);
  }

 private:
  void loop(int tid) {
    uint64_t seen = 0;
    while (true) {
      gen_.wait(seen, std::memory_order_acquire);
      seen = gen_.load(std::memory_order_acquire);
      if (stop_) return;
      (*fn_)(tid);
      if (remaining_.fetch_sub(1, std::memory_order_acq_rel) == 1) remaining_.notify_one();
    }
  }
  int n_;
  std::vector<int> cpus_;
  std::vector<std::thread> workers_;
  std::atomic<uint64_t> gen_{0};
  std::atomic<int> remaining_{0};
  const std::function<void(int)>* fn_ = nullptr;
  std::atomic<bool> stop_{false};
};

#define as_bh(v) ((__m512bh)(v))

inline uint16_t f32_to_bf16_rn(float f) {  // round-to-nearest-even (finite values)
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

// One row of W_gate / W_up against MT tokens starting at x (row stride H):
// h[t*F] = bf16(SiLU(g) * u) (h points at column r of token 0).
template <int MT>
__attribute__((target("avx512f,avx512bf16,avx512bw,avx512vl")))
inline void gate_up_row(const uint16_t* g_row, const uint16_t* u_row, const uint16_t* x, int H, int F,
                        uint16_t* h) {
  __m512 ag[MT], au[MT];
#pragma GCC unroll 8
  for (int t = 0; t < MT; ++t) {
    ag[t] = _mm512_setzero_ps();
    au[t] = _mm512_setzero_ps();
  }
  for (int d = 0; d < H; d += 32) {
    const __m512i vg = _mm512_loadu_si512(g_row + d);
    const __m512i vu = _mm512_loadu_si512(u_row + d);
#pragma GCC unroll 8
    for (int t = 0; t < MT; ++t) {
      const __m512i vx = _mm512_loadu_si512(x + static_cast<size_t>(t) * H + d);
      ag[t] = _mm512_dpbf16_ps(ag[t], as_bh(vg), as_bh(vx));
      au[t] = _mm512_dpbf16_ps(au[t], as_bh(vu), as_bh(vx));
    }
  }
#pragma GCC unroll 8
  for (int t = 0; t < MT; ++t) {
    const float g = _mm512_reduce_add_ps(ag[t]), u = _mm512_reduce_add_ps(au[t]);
    h[static_cast<size_t>(t) * F] = f32_to_bf16_rn(g / (1.0f + std::exp(-g)) * u);
  }
}

// One row of W_down against MT rows of h (row stride F): y[t*H] (column r of token 0).
template <int MT>
__attribute__((target("avx512f,avx512bf16,avx512bw,avx512vl")))
inline void down_row(const uint16_t* d_row, const uint16_t* h, int H, int F, float* y) {
  __m512 a[MT];
#pragma GCC unroll 8
  for (int t = 0; t < MT; ++t) a[t] = _mm512_setzero_ps();
  for (int f = 0; f < F; f += 32) {
    const __m512i vw = _mm512_loadu_si512(d_row + f);
#pragma GCC unroll 8
    for (int t = 0; t < MT; ++t)
      a[t] = _mm512_dpbf16_ps(a[t], as_bh(vw), as_bh(_mm512_loadu_si512(h + static_cast<size_t>(t) * F + f)));
  }
#pragma GCC unroll 8
  for (int t = 0; t < MT; ++t) y[static_cast<size_t>(t) * H] = _mm512_reduce_add_ps(a[t]);
}

// ---- AMX-BF16 path (TDPBF16PS: C[16x16] f32 += A[16x32] bf16 * B[32x16] bf16) --------
// A = 16 weight rows x 32 columns straight from the row-major slab (tile row stride =
// the weight row pitch); B = 16 tokens in the VNNI pair layout [K/2][16][2], packed once
// per expert (x) or written in that layout by phase 1 (h). One tile op consumes 1 KiB of
// weights in ~16 cycles, so the lane is bound by DRAM, not by the dot products, at any
// m <= 16 (the AVX512-BF16 GEMV above becomes compute-bound from m ~ 4).
constexpr int kTok = 16;  // tokens per B tile (padded)

struct alignas(64) TileConfig {
  uint8_t palette_id = 1, start_row = 0, reserved[14] = {};
  uint16_t colsb[16] = {};
  uint8_t rows[16] = {};
};

bool amx_enabled() {
  static const bool ok = [] {
    __builtin_cpu_init();
    if (!__builtin_cpu_supports("amx-bf16") || !__builtin_cpu_supports("amx-tile")) return false;
    // Linux: request permission for the AMX tile data state (ARCH_REQ_XCOMP_PERM 0x1023,
    // XFEATURE_XTILEDATA 18) once per process.
    return syscall(SYS_arch_prctl, 0x1023, 18) == 0;
  }();
  return ok;
}

__attribute__((target("amx-tile,amx-bf16")))
void amx_config() {
  TileConfig c;
  for (int t = 0; t < 5; ++t) {  // 0,1: C (16 x 16 f32); 2,3: A (16 x 32 bf16); 4: B (16 x 32 bf16)
    c.rows[t] = 16;
    c.colsb[t] = 64;
  }
  _tile_loadconfig(&c);
}

// Phase 1 on 16 rows [r, r+16) of W_gate/W_up and one group of 16 tokens:
// xb = packed x of the group [H/2][16][2]; writes h (VNNI layout hb [F/2][16][2]) for
// those rows. kTiled: the slab is in the lane's tile layout (ps_host_slab_tile): the 16-row
// block occupies the same bytes as in row-major order, but as consecutive 16x32 tiles of
// 1 KiB (column tile kb at + kb*512 values), so a block is two sequential streams instead
// of 32 row streams — the hardware prefetchers keep far more lines in flight per core.
template <bool kTiled>
__attribute__((target("amx-tile,amx-bf16,avx512f")))
void amx_gate_up_block(const uint16_t* wg, const uint16_t* wu, const uint16_t* xb, int H, int r, uint16_t* hb,
                       int mt) {
  alignas(64) float cg[16 * 16], cu[16 * 16];
  const size_t pitch = kTiled ? 64 : static_cast<size_t>(H) * 2;
  const uint16_t* ag = wg + static_cast<size_t>(r) * H;
  const uint16_t* au = wu + static_cast<size_t>(r) * H;
  _tile_zero(0);
  _tile_zero(1);
  for (int k = 0; k < H; k += 32) {
    const size_t o = kTiled ? static_cast<size_t>(k) * 16 : static_cast<size_t>(k);
    if (kTiled) {
      if (k + 256 < H)
        for (int q = 0; q < 16; ++q) {
          _mm_prefetch(reinterpret_cast<const char*>(ag + o + 8 * 512) + 64 * q, _MM_HINT_T0);
          _mm_prefetch(reinterpret_cast<const char*>(au + o + 8 * 512) + 64 * q, _MM_HINT_T0);
        }
    } else if (k + 512 < H) {
      for (int i = 0; i < 16; ++i) {
        _mm_prefetch(reinterpret_cast<const char*>(ag + static_cast<size_t>(i) * H + k + 512), _MM_HINT_T0);
        _mm_prefetch(reinterpret_cast<const char*>(au + static_cast<size_t>(i) * H + k + 512), _MM_HINT_T0);
      }
    }
    _tile_loadd(2, ag + o, pitch);
    _tile_loadd(3, au + o, pitch);
    _tile_loadd(4, xb + static_cast<size_t>(k) * kTok, 64);
    _tile_dpbf16ps(0, 2, 4);
    _tile_dpbf16ps(1, 3, 4);
  }
  _tile_stored(0, cg, 64);
  _tile_stored(1, cu, 64);
  // C[i][t] = row r+i, token t -> hb[((r+i)/2)*16 + t][(r+i)%2]. Only the group's mt real
  // tokens: a padded column of hb only feeds its own (discarded) output column in phase 2.
  for (int i = 0; i < 16; ++i)
    for (int t = 0; t < mt; ++t) {
      const float g = cg[i * 16 + t], u = cu[i * 16 + t];
      hb[(static_cast<size_t>((r + i) >> 1) * kTok + t) * 2 + ((r + i) & 1)] = f32_to_bf16_rn(g / (1.0f + std::exp(-g)) * u);
    }
}

// Phase 2 on 16 rows [r, r+16) of W_down against hb (VNNI [F/2][16][2]); y[t*H + r+i]
// for the first m tokens of the group.
template <bool kTiled>
__attribute__((target("amx-tile,amx-bf16,avx512f")))
void amx_down_block(const uint16_t* wd, const uint16_t* hb, int H, int F, int r, int m, float* y) {
  alignas(64) float c[16 * 16];
  const size_t pitch = kTiled ? 64 : static_cast<size_t>(F) * 2;
  const uint16_t* a = wd + static_cast<size_t>(r) * F;
  _tile_zero(0);
  for (int k = 0; k < F; k += 32) {
    const size_t o = kTiled ? static_cast<size_t>(k) * 16 : static_cast<size_t>(k);
    if (kTiled) {
      if (k + 256 < F)
        for (int q = 0; q < 16; ++q) _mm_prefetch(reinterpret_cast<const char*>(a + o + 8 * 512) + 64 * q, _MM_HINT_T0);
    } else if (k + 512 < F) {
      for (int i = 0; i < 16; ++i)
        _mm_prefetch(reinterpret_cast<const char*>(a + static_cast<size_t>(i) * F + k + 512), _MM_HINT_T0);
    }
    _tile_loadd(2, a + o, pitch);
    _tile_loadd(4, hb + static_cast<size_t>(k) * kTok, 64);
    _tile_dpbf16ps(0, 2, 4);
  }
  _tile_stored(0, c, 64);
  for (int t = 0; t < m; ++t)
    for (int i = 0; i < 16; ++i) y[static_cast<size_t>(t) * H + r + i] = c[i * 16 + t];
}

void untile_matrix_inplace(uint16_t* w, int R, int K, std::vector<uint16_t>& tmp) {
  tmp.resize(static_cast<size_t>(16) * K);
  for (int rb = 0; rb < R / 16; ++rb) {
    uint16_t* blk = w + static_cast<size_t>(rb) * 16 * K;
    std::memcpy(tmp.data(), blk, sizeof(uint16_t) * 16 * K);
    for (int kb = 0; kb < K / 32; ++kb)
      for (int i = 0; i < 16; ++i)
        std::memcpy(blk + static_cast<size_t>(i) * K + kb * 32, tmp.data() + static_cast<size_t>(kb) * 512 + i * 32, 64);
  }
}

// In-place re-layout of one [R][K] matrix into 16x32 tiles, block by block (a 16-row block
// keeps its byte range).
void tile_matrix_inplace(uint16_t* w, int R, int K, std::vector<uint16_t>& tmp) {
  tmp.resize(static_cast<size_t>(16) * K);
  for (int rb = 0; rb < R / 16; ++rb) {
    uint16_t* blk = w + static_cast<size_t>(rb) * 16 * K;
    std::memcpy(tmp.data(), blk, sizeof(uint16_t) * 16 * K);
    for (int kb = 0; kb < K / 32; ++kb)
      for (int i = 0; i < 16; ++i)
        std::memcpy(blk + static_cast<size_t>(kb) * 512 + i * 32, tmp.data() + static_cast<size_t>(i) * K + kb * 32, 64);
  }
}

__attribute__((target("amx-tile"))) void amx_release() { _tile_release(); }
// ---- z-slab path: the lane reads the transfer format instead of bf16 -----------------
// Host DRAM is the lane's bound, so reading 1.41-1.5 B instead of 2 B per weight is worth a
// few vector ops: each 16-row x 32-column A tile is decoded from the z-slab into a 1 KiB
// scratch and loaded from there. Per 32-value row segment (AVX-512 VBMI/VBMI2, branch-free):
// sign/mantissa bytes widened to 16 bit; the 3- or 4-bit exponent codes (a little-endian
// bit stream) pulled into 16-bit lanes with one byte permute + variable shift and rebased;
// escaped lanes patched with an expand-load from the block's escape list. Each row keeps a
// running escape pointer, so no per-segment rank scan.

bool z_isa_ok() {
  static const bool ok = [] {
    __builtin_cpu_init();
    return __builtin_cpu_supports("avx512vbmi") && __builtin_cpu_supports("avx512vbmi2") &&
           __builtin_cpu_supports("avx512bw") && __builtin_cpu_supports("avx512vl");
  }();
  return ok;
}

inline uint32_t z_code_at(const ZView& z, uint64_t u) {  // scalar code of value u
  const uint64_t bit = u * z.bits;
  const uint32_t w = z.codes[bit >> 3] | (static_cast<uint32_t>(z.codes[(bit >> 3) + 1]) << 8);
  return (w >> (bit & 7)) & z_escape(z.bits);
}

// Escape-list position of value v: the block's first escape + escapes in the block before v.
inline const uint8_t* z_esc_ptr(const ZView& z, uint64_t v) {
  const uint64_t b = v / kZBlock;
  const uint32_t esc = z_escape(z.bits);
  uint32_t rank = 0;
  for (uint64_t u = b * kZBlock; u < v; ++u) rank += z_code_at(z, u) == esc;
  return z.esc + z.esc_off[b] + rank;
}

struct alignas(64) ZDec {  // per-slab constants of the vector decoder (plain data)
  uint8_t perm[64];   // byte permute: qword q (values 8q..8q+7) <- code bytes q*bits .. q*bits+7
  uint8_t shift[64];  // multishift: byte j of each qword <- bits j*bits .. j*bits+7 of it
  uint8_t cmask, base;
  uint32_t seg_bytes;  // code bytes per 64-value segment
};

ZDec z_dec(const ZView& z) {
  ZDec d{};
  for (int q = 0; q < 8; ++q)
    for (int b = 0; b < 8; ++b) {
      d.perm[8 * q + b] = static_cast<uint8_t>(q * static_cast<int>(z.bits) + b);
      d.shift[8 * q + b] = static_cast<uint8_t>(b * static_cast<int>(z.bits));
    }
  d.cmask = static_cast<uint8_t>(z_escape(z.bits));
  d.base = static_cast<uint8_t>(z.base);
  d.seg_bytes = 8 * z.bits;
  return d;
}

struct ZRegs {
  __m512i perm, shift, cmask, base, m80, lo_idx, hi_idx;
};

__attribute__((target("avx512f,avx512bw,avx512vl,avx512vbmi")))
inline ZRegs z_regs(const ZDec& d) {
  // bf16 values 0-31 / 32-63 from the in-lane byte interleaves u0 = unpacklo(lo, hi)
  // (values 0-7 | 16-23 | 32-39 | 48-55) and u1 = unpackhi (8-15 | 24-31 | ...)
  return {_mm512_loadu_si512(d.perm), _mm512_loadu_si512(d.shift), _mm512_set1_epi8(static_cast<char>(d.cmask)),
          _mm512_set1_epi8(static_cast<char>(d.base)), _mm512_set1_epi8(static_cast<char>(0x80)),
          _mm512_set_epi64(11, 10, 3, 2, 9, 8, 1, 0), _mm512_set_epi64(15, 14, 7, 6, 13, 12, 5, 4)};
}

// 64 values at v (v % 64 == 0) -> seg[0..31], seg[512..543] (the same row of two
// consecutive 16x32 tiles); ep = this row's escape pointer. Byte-wide throughout (64
// values per op; 512-bit ALU work has two ports): codes pulled out of the bit stream with
// one byte permute + multishift, escapes merged by an expand-load, then the two bf16
// bytes (sign|exp>>1, exp<<7|mantissa) built with bit-selects and interleaved.
__attribute__((target("avx512f,avx512bw,avx512vl,avx512vbmi,avx512vbmi2")))
inline void z_decode64(const ZView& z, const ZRegs& r, uint32_t seg_bytes, uint64_t v, const uint8_t*& ep,
                       uint16_t* seg, uint16_t* seg2) {
  const __m512i L = _mm512_loadu_si512(z.lo + v);
  const __m512i cb = _mm512_zextsi256_si512(
      _mm256_loadu_si256(reinterpret_cast<const __m256i*>(z.codes + (v / 64) * seg_bytes)));
  const __m512i code = _mm512_and_si512(_mm512_multishift_epi64_epi8(r.shift, _mm512_permutexvar_epi8(r.perm, cb)),
                                        r.cmask);
  const __mmask64 em = _mm512_cmpeq_epi8_mask(code, r.cmask);
  const __m512i ex = _mm512_mask_expandloadu_epi8(_mm512_add_epi8(code, r.base), em, ep);
  ep += _mm_popcnt_u64(em);
  // hi byte: sign (bit 7 of L) | exp >> 1 ; lo byte: exp bit 0 -> bit 7 | mantissa (L & 0x7f)
  const __m512i hi = _mm512_ternarylogic_epi32(r.m80, L, _mm512_srli_epi16(ex, 1), 0xCA);
  const __m512i lo = _mm512_ternarylogic_epi32(r.m80, _mm512_slli_epi16(ex, 7), L, 0xCA);
  const __m512i u0 = _mm512_unpacklo_epi8(lo, hi), u1 = _mm512_unpackhi_epi8(lo, hi);
  _mm512_storeu_si512(seg, _mm512_permutex2var_epi64(u0, r.lo_idx, u1));
  _mm512_storeu_si512(seg2, _mm512_permutex2var_epi64(u0, r.hi_idx, u1));
}

// Tiled z-slab: the 1024 values at v (one z block, v % 1024 == 0) are two consecutive
// 16x32 A tiles in order -> out[1024]. Two sequential streams (lo bytes, codes),
// prefetched 4 blocks ahead.
__attribute__((target("avx512f,avx512bw,avx512vl,avx512vbmi,avx512vbmi2")))
inline void z_run1024(const ZView& z, const ZRegs& r, uint32_t seg_bytes, uint64_t v, uint64_t vend, uint16_t* out) {
  // Prefetch 4 blocks ahead, across the unit's end too: a thread's next unit is usually the
  // adjacent 16-row block of the same slab, and small units (Qwen3's W_down: 12 blocks)
  // otherwise start cold on every unit. (Prefetches never fault; past the slab they only
  // touch other host memory.)
  static const bool unit_only = [] {  // PS_LANE_PF_UNIT=1: round 1's within-unit prefetch (A/B)
    const char* e = std::getenv("PS_LANE_PF_UNIT");
    return e && e[0] == '1';
  }();
  static const uint64_t ahead = [] {  // PS_LANE_PF_BLOCKS: prefetch distance in 1024-value blocks (A/B)
    const char* e = std::getenv("PS_LANE_PF_BLOCKS");
    const int b = e ? std::atoi(e) : 4;
    return static_cast<uint64_t>(b >= 1 && b <= 64 ? b : 4) * 1024;
  }();
  if (!unit_only || v + ahead < vend) {
    const char* pl = reinterpret_cast<const char*>(z.lo + v + ahead);
    for (int q = 0; q < 16; ++q) _mm_prefetch(pl + 64 * q, _MM_HINT_T0);
    const char* pc = reinterpret_cast<const char*>(z.codes + (v + ahead) / 64 * seg_bytes);
    for (uint32_t q = 0; q < seg_bytes / 4; ++q) _mm_prefetch(pc + 64 * q, _MM_HINT_T0);  // 16 x seg_bytes
  }
  const uint8_t* ep = z.esc + z.esc_off[v / kZBlock];
  for (int g = 0; g < 16; ++g) z_decode64(z, r, seg_bytes, v + 64 * g, ep, out + 64 * g, out + 64 * g + 32);
}

// Two consecutive A tiles (16 rows x 64 cols) of the row-major matrix whose row r starts at
// value `rowv`, row length `ld` values, columns [k, k+64) -> scratch [2][16][32]. The 16
// rows are 32 streams (sign/mantissa bytes and codes) — too many for the hardware
// prefetchers — so every row's lines are prefetched 1 KiB of values ahead. ep[16]: the
// rows' escape pointers, set at k == 0 and at every block start.
__attribute__((target("avx512f,avx512bw,avx512vl,avx512vbmi,avx512vbmi2")))
inline void z_tile2(const ZView& z, const ZRegs& r, uint32_t seg_bytes, uint64_t rowv, uint64_t ld, int k, int kend,
                    const uint8_t** ep, uint16_t* scratch) {
  const int kp = k + 512;
  if (kp < kend)
    for (int i = 0; i < 16; ++i) {
      const uint64_t v = rowv + static_cast<uint64_t>(i) * ld + kp;
      _mm_prefetch(reinterpret_cast<const char*>(z.lo + v), _MM_HINT_T1);
      if ((k & 127) == 0) _mm_prefetch(reinterpret_cast<const char*>(z.codes + (v / 64) * seg_bytes), _MM_HINT_T1);
    }
  for (int i = 0; i < 16; ++i) {
    const uint64_t v = rowv + static_cast<uint64_t>(i) * ld + k;
    if (k == 0)
      ep[i] = z_esc_ptr(z, v);
    else if (v % kZBlock == 0)
      ep[i] = z.esc + z.esc_off[v / kZBlock];
    z_decode64(z, r, seg_bytes, v, ep[i], scratch + i * 32, scratch + 512 + i * 32);
  }
}

__attribute__((target("amx-tile,amx-bf16,avx512f,avx512bw,avx512vl,avx512vbmi,avx512vbmi2")))
void amx_gate_up_block_z(const ZView& z, const ZDec& d, int H, int F, const uint16_t* xb, int r, uint16_t* hb,
                         int mt) {
  alignas(64) float cg[16 * 16], cu[16 * 16];
  // two scratch sets, alternated per step: the next step's decode stores do not wait for
  // this step's tile loads (write-after-read on one buffer serialises decode and AMX)
  alignas(64) uint16_t sgb[2][2 * 16 * 32], sub[2][2 * 16 * 32];
  const uint8_t* eg[16];
  const uint8_t* eu[16];
  const ZRegs R = z_regs(d);
  const uint64_t gv = static_cast<uint64_t>(r) * H, uv = (static_cast<uint64_t>(F) + r) * H;
  _tile_zero(0);
  _tile_zero(1);
  for (int k = 0; k < H; k += 64) {
    uint16_t* sg = sgb[(k >> 6) & 1];
    uint16_t* su = sub[(k >> 6) & 1];
    if (z.tiled) {  // block rows [r, r+16), tiles k/32 and k/32+1: 1024 contiguous values
      z_run1024(z, R, d.seg_bytes, gv + static_cast<uint64_t>(k) * 16, gv + 16ull * H, sg);
      z_run1024(z, R, d.seg_bytes, uv + static_cast<uint64_t>(k) * 16, uv + 16ull * H, su);
    } else {
      z_tile2(z, R, d.seg_bytes, gv, H, k, H, eg, sg);
      z_tile2(z, R, d.seg_bytes, uv, H, k, H, eu, su);
    }
    for (int h = 0; h < 2; ++h) {
      _tile_loadd(2, sg + h * 512, 64);
      _tile_loadd(3, su + h * 512, 64);
      _tile_loadd(4, xb + static_cast<size_t>(k + 32 * h) * kTok, 64);
      _tile_dpbf16ps(0, 2, 4);
      _tile_dpbf16ps(1, 3, 4);
    }
  }
  _tile_stored(0, cg, 64);
  _tile_stored(1, cu, 64);
  for (int i = 0; i < 16; ++i)  // the group's mt real tokens only (see amx_gate_up_block)
    for (int t = 0; t < mt; ++t) {
      const float g = cg[i * 16 + t], u = cu[i * 16 + t];
      hb[(static_cast<size_t>((r + i) >> 1) * kTok + t) * 2 + ((r + i) & 1)] = f32_to_bf16_rn(g / (1.0f + std::exp(-g)) * u);
    }
}

__attribute__((target("amx-tile,amx-bf16,avx512f,avx512bw,avx512vl,avx512vbmi,avx512vbmi2")))
void amx_down_block_z(const ZView& z, const ZDec& d, const uint16_t* hb, int H, int F, int r, int m, float* y) {
  alignas(64) float c[16 * 16];
  alignas(64) uint16_t sdb[2][2 * 16 * 32];
  const uint8_t* ed[16];
  const ZRegs R = z_regs(d);
  const uint64_t dv = 2ull * F * H + static_cast<uint64_t>(r) * F;
  _tile_zero(0);
  for (int k = 0; k < F; k += 64) {
    uint16_t* sd = sdb[(k >> 6) & 1];
    if (z.tiled)
      z_run1024(z, R, d.seg_bytes, dv + static_cast<uint64_t>(k) * 16, dv + 16ull * F, sd);
    else
      z_tile2(z, R, d.seg_bytes, dv, F, k, F, ed, sd);
    for (int h = 0; h < 2; ++h) {
      _tile_loadd(2, sd + h * 512, 64);
      _tile_loadd(4, hb + static_cast<size_t>(k + 32 * h) * kTok, 64);
      _tile_dpbf16ps(0, 2, 4);
    }
  }
  _tile_stored(0, c, 64);
  for (int t = 0; t < m; ++t)
    for (int i = 0; i < 16; ++i) y[static_cast<size_t>(t) * H + r + i] = c[i * 16 + t];
}

template <typename Fn>
void by_token_chunks(int m, Fn&& fn) {  // fn(template MT, t0)
  int t0 = 0;
  for (; t0 + 8 <= m; t0 += 8) fn(std::integral_constant<int, 8>{}, t0);
  switch (m - t0) {
    case 7: fn(std::integral_constant<int, 7>{}, t0); break;
    case 6: fn(std::integral_constant<int, 6>{}, t0); break;
    case 5: fn(std::integral_constant<int, 5>{}, t0); break;
    case 4: fn(std::integral_constant<int, 4>{}, t0); break;
    case 3: fn(std::integral_constant<int, 3>{}, t0); break;
    case 2: fn(std::integral_constant<int, 2>{}, t0); break;
    case 1: fn(std::integral_constant<int, 1>{}, t0); break;
    default: break;
  }
}

// Guided self-scheduling of (expert, 16-row block) units: a pool pass ends at its
// slowest thread, and DRAM contention makes equal static ranges finish unevenly. Each
// grab takes remaining/(2T) units (>= 2): long contiguous weight streams early, single
// ~25 us units at the end, so the pass tail is about one unit. Units write disjoint
// outputs, so results do not depend on the assignment.
template <typename Fn>
void for_units(int64_t U, int T, std::atomic<int64_t>& next, Fn&& fn) {
  // A/B runs: PS_HOST_LANE_CHUNKS=1 one chunk per thread, =2 fixed chunks of U/(8T)
  static const int mode = [] {
    const char* v = std::getenv("PS_HOST_LANE_CHUNKS");
    return v ? std::atoi(v) : 0;
  }();
  const int64_t fixed = mode == 1 ? (U + T - 1) / T : std::max<int64_t>(1, (U + 8 * T - 1) / (8 * T));
  int64_t cur = next.load(std::memory_order_relaxed);
  while (cur < U) {
    const int64_t c = mode ? fixed : std::max<int64_t>(2, (U - cur) / (2 * static_cast<int64_t>(T)));
    if (!next.compare_exchange_weak(cur, cur + c, std::memory_order_relaxed)) continue;
    for (int64_t u = cur, e = std::min(U, cur + c); u < e; ++u) fn(u);
    cur = next.load(std::memory_order_relaxed);
  }
}

}  // namespace
}  // namespace ps

struct ps_host_lane_s {
  std::unique_ptr<ps::Pool> pool;
  bool amx = false;            // AMX-BF16 tiles available (else the AVX512-BF16 GEMV)
  std::vector<uint16_t> h;     // [m, F] bf16 activations (AVX512 path)
  std::vector<uint16_t> xb, hb;  // VNNI-packed x / h per 16-token group (AMX path)
};

using namespace ps;

extern "C" {

ps_status ps_host_lane_create(int threads, ps_host_lane* out) {
  return guarded([&] {
    require(out != nullptr && threads >= 1 && threads <= 1024, "ps_host_lane_create: threads in [1, 1024]");
    __builtin_cpu_init();
    if (!__builtin_cpu_supports("avx512bf16"))
      fail(PS_ERUNTIME, "ps_host_lane_create: the host CPU lacks AVX512_BF16 (the host lane's GEMV instruction)");
    auto l = std::make_unique<ps_host_lane_s>();
    l->pool = std::make_unique<Pool>(threads);
    const char* force = std::getenv("PS_HOST_LANE_ISA");  // "avx512" forces the GEMV path (tests)
    l->amx = amx_enabled() && !(force && std::strcmp(force, "avx512") == 0);
    *out = l.release();
  });
}

ps_status ps_host_lane_destroy(ps_host_lane l) {
  delete l;
  return PS_OK;
}

int ps_host_lane_threads(ps_host_lane l) { return l ? l->pool->size() : 0; }

int ps_host_lane_isa(ps_host_lane l) { return l ? (l->amx ? 2 : 1) : 0; }
int ps_host_lane_reads_z(ps_host_lane l) { return l && l->amx && z_isa_ok() ? 1 : 0; }

ps_status ps_host_lane_bind_caller(ps_host_lane l) {
  return guarded([&] {
    require(l != nullptr, "ps_host_lane_bind_caller: null lane");
    l->pool->pin_caller();
  });
}

// A batch of experts (PreSched's cpu_set of one layer) in two pool passes: phase 1 over
// all (expert, 16-row block of W_gate/W_up) units, phase 2 over all (expert, 16-row
// block of W_down) units; each thread streams a contiguous range of units. One pass pair
// per layer instead of per expert keeps small experts (Qwen3: 9 MiB) off the pool's
// wake-up latency.
namespace ps {
namespace {
ps_status expert_ffn_batch(ps_host_lane l, int n, const uint16_t* const* slabs, const int32_t* m, const int32_t* row0,
                           int H, int F, const uint16_t* x, float* y, bool tiled) {
  return guarded([&] {
    if (tiled && !(l && l->amx)) fail(PS_ERUNTIME, "ps_host_expert_ffn_batch_tiled: needs AMX-BF16");
    require(l && n >= 0 && (n == 0 || (slabs && m && row0 && x && y)), "ps_host_expert_ffn_batch: null argument");
    require(H > 0 && F > 0 && H % 32 == 0 && F % 32 == 0, "ps_host_expert_ffn: H and F must be multiples of 32");
    for (int j = 0; j < n; ++j) {
      require(slabs[j] != nullptr, "ps_host_expert_ffn: null slab");
      require(m[j] >= 0 && m[j] <= 4096 && row0[j] >= 0, "ps_host_expert_ffn: m out of range");
    }
    const int T = l->pool->size();
    const int nb1 = F / 16, nb2 = H / 16;
    const int64_t U1 = static_cast<int64_t>(n) * nb1, U2 = static_cast<int64_t>(n) * nb2;
    auto range = [&](int64_t U, int tid, int64_t& u0, int64_t& u1) {
      u0 = U * tid / T;
      u1 = U * (tid + 1) / T;
    };
    if (l->amx) {
      // AMX path: per expert, token groups of 16 (zero-padded), x packed into the VNNI
      // pair layout; h written by phase 1 in the same layout.
      std::vector<size_t> xo(n + 1, 0), ho(n + 1, 0);
      for (int j = 0; j < n; ++j) {
        const size_t G = (m[j] + kTok - 1) / kTok;
        xo[j + 1] = xo[j] + G * H * kTok;
        ho[j + 1] = ho[j] + G * F * kTok;
      }
      if (l->xb.size() < xo[n]) l->xb.resize(xo[n]);
      if (l->hb.size() < ho[n]) l->hb.resize(ho[n]);
      uint16_t* xb = l->xb.data();
      uint16_t* hb = l->hb.data();
      std::memset(xb, 0, sizeof(uint16_t) * xo[n]);
      for (int j = 0; j < n; ++j)
        for (int t = 0; t < m[j]; ++t) {
          const uint16_t* xr = x + static_cast<size_t>(row0[j] + t) * H;
          uint16_t* d = xb + xo[j] + static_cast<size_t>(t / kTok) * H * kTok + (t % kTok) * 2;
          for (int k = 0; k < H; k += 2) {
            d[static_cast<size_t>(k >> 1) * kTok * 2] = xr[k];
            d[static_cast<size_t>(k >> 1) * kTok * 2 + 1] = xr[k + 1];
          }
        }
      // PS_HOST_LANE_ONEPASS=1: one pool pass (below). Opt-in: alternating engine runs
      // show no measurable difference to two passes (profiles/r01_bench_lane_onepass.jsonl),
      // and its spin-waits burn a core when lane threads oversubscribe the host.
      static const bool two_pass = [] {
        const char* v = std::getenv("PS_HOST_LANE_ONEPASS");
        return !(v && v[0] == '1');
      }();
      if (!two_pass) {
        // One pool pass: gate_up units (expert-major) then down units; a down unit of
        // expert j waits (release/acquire counter) until all nb1 gate_up units of j have
        // written h. All gate_up units are handed out before any down unit and never
        // wait, so the spin always ends; threads that finish early start on the down
        // projections instead of idling at a phase barrier.
        std::unique_ptr<std::atomic<int>[]> done(new std::atomic<int>[n]);
        for (int j = 0; j < n; ++j) done[j].store(0, std::memory_order_relaxed);
        std::atomic<int64_t> next{0};
        l->pool->run([&](int) {
          amx_config();
          for_units(U1 + U2, T, next, [&](int64_t u) {
            if (u < U1) {
              const int j = static_cast<int>(u / nb1), blk = static_cast<int>(u % nb1);
              const uint16_t* wg = slabs[j];
              const uint16_t* wu = wg + static_cast<size_t>(F) * H;
              for (int g = 0; g * kTok < m[j]; ++g)
                (tiled ? amx_gate_up_block<true> : amx_gate_up_block<false>)(
                    wg, wu, xb + xo[j] + static_cast<size_t>(g) * H * kTok, H, blk * 16,
                    hb + ho[j] + static_cast<size_t>(g) * F * kTok, std::min(kTok, m[j] - g * kTok));
              done[j].fetch_add(1, std::memory_order_release);
            } else {
              const int64_t v = u - U1;
              const int j = static_cast<int>(v / nb2), blk = static_cast<int>(v % nb2);
              while (done[j].load(std::memory_order_acquire) < nb1) _mm_pause();
              const uint16_t* wd = slabs[j] + static_cast<size_t>(2) * F * H;
              for (int g = 0; g * kTok < m[j]; ++g)
                (tiled ? amx_down_block<true> : amx_down_block<false>)(
                    wd, hb + ho[j] + static_cast<size_t>(g) * F * kTok, H, F, blk * 16,
                    std::min(kTok, m[j] - g * kTok), y + static_cast<size_t>(row0[j] + g * kTok) * H);
            }
          });
          amx_release();
        });
        return;
      }
      std::atomic<int64_t> next1{0}, next2{0};
      l->pool->run([&](int) {
        amx_config();
        for_units(U1, T, next1, [&](int64_t u) {
          const int j = static_cast<int>(u / nb1), blk = static_cast<int>(u % nb1);
          const uint16_t* wg = slabs[j];
          const uint16_t* wu = wg + static_cast<size_t>(F) * H;
          for (int g = 0; g * kTok < m[j]; ++g)
            (tiled ? amx_gate_up_block<true> : amx_gate_up_block<false>)(
                wg, wu, xb + xo[j] + static_cast<size_t>(g) * H * kTok, H, blk * 16,
                hb + ho[j] + static_cast<size_t>(g) * F * kTok, std::min(kTok, m[j] - g * kTok));
        });
        amx_release();
      });
      l->pool->run([&](int) {
        amx_config();
        for_units(U2, T, next2, [&](int64_t u) {
          const int j = static_cast<int>(u / nb2), blk = static_cast<int>(u % nb2);
          const uint16_t* wd = slabs[j] + static_cast<size_t>(2) * F * H;
          for (int g = 0; g * kTok < m[j]; ++g)
            (tiled ? amx_down_block<true> : amx_down_block<false>)(
                wd, hb + ho[j] + static_cast<size_t>(g) * F * kTok, H, F, blk * 16, std::min(kTok, m[j] - g * kTok),
                y + static_cast<size_t>(row0[j] + g * kTok) * H);
        });
        amx_release();
      });
      return;
    }
    // AVX512-BF16 GEMV path. Rows outer, token chunks inner: a weight row (8 KiB at
    // H = 4096) is read from DRAM once and re-read from L1 by the next chunk of 8 tokens.
    std::vector<size_t> hoff(n + 1, 0);
    for (int j = 0; j < n; ++j) hoff[j + 1] = hoff[j] + static_cast<size_t>(m[j]) * F;
    if (l->h.size() < hoff[n]) l->h.resize(hoff[n]);
    uint16_t* h = l->h.data();
    l->pool->run([&](int tid) {
      int64_t u0, u1;
      range(U1, tid, u0, u1);
      for (int64_t u = u0; u < u1; ++u) {
        const int j = static_cast<int>(u / nb1), blk = static_cast<int>(u % nb1);
        const uint16_t* wg = slabs[j];
        const uint16_t* wu = wg + static_cast<size_t>(F) * H;
        const uint16_t* xj = x + static_cast<size_t>(row0[j]) * H;
        for (int r = blk * 16; r < blk * 16 + 16; ++r)
          by_token_chunks(m[j], [&](auto mt, int t0) {
            gate_up_row<decltype(mt)::value>(wg + static_cast<size_t>(r) * H, wu + static_cast<size_t>(r) * H,
                                             xj + static_cast<size_t>(t0) * H, H, F,
                                             h + hoff[j] + static_cast<size_t>(t0) * F + r);
          });
      }
    });
    l->pool->run([&](int tid) {
      int64_t u0, u1;
      range(U2, tid, u0, u1);
      for (int64_t u = u0; u < u1; ++u) {
        const int j = static_cast<int>(u / nb2), blk = static_cast<int>(u % nb2);
        const uint16_t* wd = slabs[j] + static_cast<size_t>(2) * F * H;
        for (int r = blk * 16; r < blk * 16 + 16; ++r)
          by_token_chunks(m[j], [&](auto mt, int t0) {
            down_row<decltype(mt)::value>(wd + static_cast<size_t>(r) * F, h + hoff[j] + static_cast<size_t>(t0) * F,
                                          H, F, y + static_cast<size_t>(row0[j] + t0) * H + r);
          });
      }
    });
  });
}
}  // namespace
}  // namespace ps

ps_status ps_host_expert_ffn_batch(ps_host_lane l, int n, const uint16_t* const* slabs, const int32_t* m,
                                   const int32_t* row0, int H, int F, const uint16_t* x, float* y) {
  return ps::expert_ffn_batch(l, n, slabs, m, row0, H, F, x, y, false);
}

ps_status ps_host_expert_ffn_batch_tiled(ps_host_lane l, int n, const uint16_t* const* slabs, const int32_t* m,
                                         const int32_t* row0, int H, int F, const uint16_t* x, float* y) {
  return ps::expert_ffn_batch(l, n, slabs, m, row0, H, F, x, y, true);
}

ps_status ps_host_slab_untile(uint16_t* slab, int H, int F) {
  return guarded([&] {
    require(slab && H > 0 && F > 0 && H % 32 == 0 && F % 32 == 0, "ps_host_slab_untile: bad argument");
    std::vector<uint16_t> tmp;
    untile_matrix_inplace(slab, F, H, tmp);
    untile_matrix_inplace(slab + static_cast<size_t>(F) * H, F, H, tmp);
    untile_matrix_inplace(slab + static_cast<size_t>(2) * F * H, H, F, tmp);
  });
}

ps_status ps_host_slab_tile(uint16_t* slab, int H, int F) {
  return guarded([&] {
    require(slab && H > 0 && F > 0 && H % 32 == 0 && F % 32 == 0, "ps_host_slab_tile: bad argument");
    std::vector<uint16_t> tmp;
    tile_matrix_inplace(slab, F, H, tmp);                                      // W_gate [F][H]
    tile_matrix_inplace(slab + static_cast<size_t>(F) * H, F, H, tmp);         // W_up   [F][H]
    tile_matrix_inplace(slab + static_cast<size_t>(2) * F * H, H, F, tmp);     // W_down [H][F]
  });
}

// Same as ps_host_expert_ffn_batch, weights read from z-slabs (AMX path only).
ps_status ps_host_expert_ffn_batch_z(ps_host_lane l, int n, const uint8_t* const* zslabs, const int32_t* m,
                                     const int32_t* row0, int H, int F, const uint16_t* x, float* y) {
  return guarded([&] {
    require(l && n >= 0 && (n == 0 || (zslabs && m && row0 && x && y)), "ps_host_expert_ffn_batch_z: null argument");
    require(H > 0 && F > 0 && H % 64 == 0 && F % 64 == 0, "ps_host_expert_ffn_batch_z: H, F % 64 == 0");
    if (!l->amx || !z_isa_ok())
      fail(PS_ERUNTIME, "ps_host_expert_ffn_batch_z: needs AMX-BF16 and AVX-512 VBMI2 (use the raw slabs)");
    std::vector<ZView> zv;
    std::vector<ZDec> zd;
    for (int j = 0; j < n; ++j) {
      require(zslabs[j] != nullptr && m[j] >= 0 && m[j] <= 4096 && row0[j] >= 0, "ps_host_expert_ffn_batch_z: bad job");
      const ZHeader* h = reinterpret_cast<const ZHeader*>(zslabs[j]);
      require(h->magic == kZMagic && h->n == 3ull * H * F, "ps_host_expert_ffn_batch_z: not a z-slab of this shape");
      require(h->code_bits == 3 || h->code_bits == 4, "ps_host_expert_ffn_batch_z: bad code width");
      require(!h->tiled || (h->tile_h == static_cast<uint32_t>(H) && h->tile_f == static_cast<uint32_t>(F)),
              "ps_host_expert_ffn_batch_z: tiled z-slab of another shape");
      zv.emplace_back(zslabs[j]);
      zd.push_back(z_dec(zv.back()));
    }
    const int T = l->pool->size();
    const int nb1 = F / 16, nb2 = H / 16;
    const int64_t U1 = static_cast<int64_t>(n) * nb1, U2 = static_cast<int64_t>(n) * nb2;
    std::vector<size_t> xo(n + 1, 0), ho(n + 1, 0);
    for (int j = 0; j < n; ++j) {
      const size_t G = (m[j] + kTok - 1) / kTok;
      xo[j + 1] = xo[j] + G * H * kTok;
      ho[j + 1] = ho[j] + G * F * kTok;
    }
    if (l->xb.size() < xo[n]) l->xb.resize(xo[n]);
    if (l->hb.size() < ho[n]) l->hb.resize(ho[n]);
    uint16_t* xb = l->xb.data();
    uint16_t* hb = l->hb.data();
    std::memset(xb, 0, sizeof(uint16_t) * xo[n]);
    for (int j = 0; j < n; ++j)
      for (int t = 0; t < m[j]; ++t) {
        const uint16_t* xr = x + static_cast<size_t>(row0[j] + t) * H;
        uint16_t* d = xb + xo[j] + static_cast<size_t>(t / kTok) * H * kTok + (t % kTok) * 2;
        for (int k = 0; k < H; k += 2) {
          d[static_cast<size_t>(k >> 1) * kTok * 2] = xr[k];
          d[static_cast<size_t>(k >> 1) * kTok * 2 + 1] = xr[k + 1];
        }
      }
    std::atomic<int64_t> next1{0}, next2{0};
    std::atomic<int> arrived{0};
    auto phase2 = [&] {
      for_units(U2, T, next2, [&](int64_t u) {
        const int j = static_cast<int>(u / nb2), blk = static_cast<int>(u % nb2);
        for (int g = 0; g * kTok < m[j]; ++g)
          amx_down_block_z(zv[j], zd[j], hb + ho[j] + static_cast<size_t>(g) * F * kTok, H, F, blk * 16,
                           std::min(kTok, m[j] - g * kTok), y + static_cast<size_t>(row0[j] + g * kTok) * H);
      });
    };
    // One pool run per phase (default). PS_HOST_LANE_SPLITRUN=0: both phases in one run
    // with a spin barrier between them (saves a futex wake per batch, but in the engine a
    // descheduled lane thread — the engine and I/O threads share the cores — holds 15
    // spinning threads: Qwen3 host lane 900 -> 400-560 tok/s, r02_configs_qwen3_splitrun.jsonl).
    static const bool split_runs = [] {
      const char* v = std::getenv("PS_HOST_LANE_SPLITRUN");
      return !(v && v[0] == '0');
    }();
    l->pool->run([&](int) {
      amx_config();
      for_units(U1, T, next1, [&](int64_t u) {
        const int j = static_cast<int>(u / nb1), blk = static_cast<int>(u % nb1);
        for (int g = 0; g * kTok < m[j]; ++g)
          amx_gate_up_block_z(zv[j], zd[j], H, F, xb + xo[j] + static_cast<size_t>(g) * H * kTok, blk * 16,
                              hb + ho[j] + static_cast<size_t>(g) * F * kTok, std::min(kTok, m[j] - g * kTok));
      });
      if (split_runs) {
        amx_release();
        return;
      }
      // phase barrier: every h row written (release) before any down unit reads it (acquire)
      arrived.fetch_add(1, std::memory_order_acq_rel);
      while (arrived.load(std::memory_order_acquire) < T) _mm_pause();
      phase2();
      amx_release();
    });
    if (split_runs)
      l->pool->run([&](int) {
        amx_config();
        phase2();
        amx_release();
      });
  });
}

ps_status ps_host_expert_ffn(ps_host_lane l, const uint16_t* slab, int H, int F, const uint16_t* x, int m, float* y) {
  const int32_t zero = 0;
  return ps_host_expert_ffn_batch(l, 1, &slab, &m, &zero, H, F, x, y);
}

}  // extern "C"
