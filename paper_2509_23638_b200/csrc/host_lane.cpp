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
// those rows.
__attribute__((target("amx-tile,amx-bf16,avx512f")))
void amx_gate_up_block(const uint16_t* wg, const uint16_t* wu, const uint16_t* xb, int H, int r, uint16_t* hb) {
  alignas(64) float cg[16 * 16], cu[16 * 16];
  const size_t pitch = static_cast<size_t>(H) * 2;
  const uint16_t* ag = wg + static_cast<size_t>(r) * H;
  const uint16_t* au = wu + static_cast<size_t>(r) * H;
  _tile_zero(0);
  _tile_zero(1);
  for (int k = 0; k < H; k += 32) {
    if (k + 512 < H)
      for (int i = 0; i < 16; ++i) {
        _mm_prefetch(reinterpret_cast<const char*>(ag + static_cast<size_t>(i) * H + k + 512), _MM_HINT_T0);
        _mm_prefetch(reinterpret_cast<const char*>(au + static_cast<size_t>(i) * H + k + 512), _MM_HINT_T0);
      }
    _tile_loadd(2, ag + k, pitch);
    _tile_loadd(3, au + k, pitch);
    _tile_loadd(4, xb + static_cast<size_t>(k) * kTok, 64);
    _tile_dpbf16ps(0, 2, 4);
    _tile_dpbf16ps(1, 3, 4);
  }
  _tile_stored(0, cg, 64);
  _tile_stored(1, cu, 64);
  // C[i][t] = row r+i, token t -> hb[((r+i)/2)*16 + t][(r+i)%2]
  for (int i = 0; i < 16; ++i)
    for (int t = 0; t < kTok; ++t) {
      const float g = cg[i * 16 + t], u = cu[i * 16 + t];
      hb[(static_cast<size_t>((r + i) >> 1) * kTok + t) * 2 + ((r + i) & 1)] = f32_to_bf16_rn(g / (1.0f + std::exp(-g)) * u);
    }
}

// Phase 2 on 16 rows [r, r+16) of W_down against hb (VNNI [F/2][16][2]); y[t*H + r+i]
// for the first m tokens of the group.
__attribute__((target("amx-tile,amx-bf16,avx512f")))
void amx_down_block(const uint16_t* wd, const uint16_t* hb, int H, int F, int r, int m, float* y) {
  alignas(64) float c[16 * 16];
  const size_t pitch = static_cast<size_t>(F) * 2;
  const uint16_t* a = wd + static_cast<size_t>(r) * F;
  _tile_zero(0);
  for (int k = 0; k < F; k += 32) {
    if (k + 512 < F)
      for (int i = 0; i < 16; ++i)
        _mm_prefetch(reinterpret_cast<const char*>(a + static_cast<size_t>(i) * F + k + 512), _MM_HINT_T0);
    _tile_loadd(2, a + k, pitch);
    _tile_loadd(4, hb + static_cast<size_t>(k) * kTok, 64);
    _tile_dpbf16ps(0, 2, 4);
  }
  _tile_stored(0, c, 64);
  for (int t = 0; t < m; ++t)
    for (int i = 0; i < 16; ++i) y[static_cast<size_t>(t) * H + r + i] = c[i * 16 + t];
}

__attribute__((target("amx-tile"))) void amx_release() { _tile_release(); }
// ---- z-slab path: the lane reads the 12-bit transfer format instead of bf16 --------
// Host DRAM is the lane's bound, so reading 1.5 B instead of 2 B per weight is worth a
// few vector ops: each 16-row x 32-column A tile is decoded from the z-slab into a 1 KiB
// scratch (AVX-512: sign/mantissa bytes widened to 16 bit, 4-bit exponent codes unpacked
// and rebased, escapes patched from the block's escape list) and loaded from there.

// Escaped exponents of the 32-value segment at value index v (v % 32 == 0, so the
// segment lies in one 1024-value block): rank of the first one = escapes in the block
// before v.
inline void z_patch_escapes(const ZView& z, uint64_t v, uint16_t* seg) {
  const uint64_t b = v / kZBlock;
  uint32_t rank = 0;
  for (uint64_t u = b * kZBlock; u < v; u += 2) {
    const uint8_t c = z.codes[u / 2];
    rank += (c & 15) == kZEscape;
    rank += (c >> 4) == kZEscape;
  }
  const uint8_t* e = z.esc + z.esc_off[b] + rank;
  for (int i = 0; i < 32; ++i) {
    const uint8_t c = (z.codes[(v + i) / 2] >> (4 * ((v + i) & 1))) & 15;
    if (c == kZEscape) seg[i] = static_cast<uint16_t>((seg[i] & 0x807fu) | (static_cast<uint32_t>(*e++) << 7));
  }
}

// 32 values at v -> seg[32] bf16.
__attribute__((target("avx512f,avx512bw,avx512vl")))
inline void z_decode32(const ZView& z, uint64_t v, uint16_t* seg) {
  const __m512i lo16 = _mm512_cvtepu8_epi16(_mm256_loadu_si256(reinterpret_cast<const __m256i*>(z.lo + v)));
  const __m128i cb = _mm_loadu_si128(reinterpret_cast<const __m128i*>(z.codes + v / 2));
  const __m128i nib = _mm_set1_epi8(0x0f);
  const __m128i ev = _mm_and_si128(cb, nib), od = _mm_and_si128(_mm_srli_epi16(cb, 4), nib);
  const __m256i codes8 = _mm256_set_m128i(_mm_unpackhi_epi8(ev, od), _mm_unpacklo_epi8(ev, od));
  const __m512i code16 = _mm512_cvtepu8_epi16(codes8);
  const __m512i exp16 = _mm512_add_epi16(code16, _mm512_set1_epi16(static_cast<short>(z.base)));
  const __m512i val = _mm512_or_si512(
      _mm512_or_si512(_mm512_slli_epi16(_mm512_and_si512(lo16, _mm512_set1_epi16(0x80)), 8),
                      _mm512_slli_epi16(exp16, 7)),
      _mm512_and_si512(lo16, _mm512_set1_epi16(0x7f)));
  _mm512_storeu_si512(seg, val);
  if (_mm512_cmpeq_epi16_mask(code16, _mm512_set1_epi16(kZEscape))) z_patch_escapes(z, v, seg);
}

// A tile (16 rows x 32 cols) of the row-major matrix whose row r starts at value `rowv`,
// row length `ld` values, column k -> scratch [16][32]. The 16 rows are 32 streams (sign/
// mantissa bytes and codes) — too many for the hardware prefetchers — so every row's
// lines are prefetched 1 KiB of values ahead.
__attribute__((target("avx512f,avx512bw,avx512vl")))
inline void z_tile(const ZView& z, uint64_t rowv, uint64_t ld, int k, int kend, uint16_t* scratch) {
  const int kp = k + 1024;
  if (kp < kend)
    for (int i = 0; i < 16; ++i) {
      const uint64_t v = rowv + static_cast<uint64_t>(i) * ld + kp;
      if ((k & 63) == 0) _mm_prefetch(reinterpret_cast<const char*>(z.lo + v), _MM_HINT_T0);
      if ((k & 127) == 0) _mm_prefetch(reinterpret_cast<const char*>(z.codes + v / 2), _MM_HINT_T0);
    }
  for (int i = 0; i < 16; ++i) z_decode32(z, rowv + static_cast<uint64_t>(i) * ld + k, scratch + i * 32);
}

__attribute__((target("amx-tile,amx-bf16,avx512f,avx512bw,avx512vl")))
void amx_gate_up_block_z(const ZView& z, int H, int F, const uint16_t* xb, int r, uint16_t* hb) {
  alignas(64) float cg[16 * 16], cu[16 * 16];
  alignas(64) uint16_t sg[16 * 32], su[16 * 32];
  const uint64_t gv = static_cast<uint64_t>(r) * H, uv = (static_cast<uint64_t>(F) + r) * H;
  _tile_zero(0);
  _tile_zero(1);
  for (int k = 0; k < H; k += 32) {
    z_tile(z, gv, H, k, H, sg);
    z_tile(z, uv, H, k, H, su);
    _tile_loadd(2, sg, 64);
    _tile_loadd(3, su, 64);
    _tile_loadd(4, xb + static_cast<size_t>(k) * kTok, 64);
    _tile_dpbf16ps(0, 2, 4);
    _tile_dpbf16ps(1, 3, 4);
  }
  _tile_stored(0, cg, 64);
  _tile_stored(1, cu, 64);
  for (int i = 0; i < 16; ++i)
    for (int t = 0; t < kTok; ++t) {
      const float g = cg[i * 16 + t], u = cu[i * 16 + t];
      hb[(static_cast<size_t>((r + i) >> 1) * kTok + t) * 2 + ((r + i) & 1)] = f32_to_bf16_rn(g / (1.0f + std::exp(-g)) * u);
    }
}

__attribute__((target("amx-tile,amx-bf16,avx512f,avx512bw,avx512vl")))
void amx_down_block_z(const ZView& z, const uint16_t* hb, int H, int F, int r, int m, float* y) {
  alignas(64) float c[16 * 16];
  alignas(64) uint16_t sd[16 * 32];
  const uint64_t dv = 2ull * F * H + static_cast<uint64_t>(r) * F;
  _tile_zero(0);
  for (int k = 0; k < F; k += 32) {
    z_tile(z, dv, F, k, F, sd);
    _tile_loadd(2, sd, 64);
    _tile_loadd(4, hb + static_cast<size_t>(k) * kTok, 64);
    _tile_dpbf16ps(0, 2, 4);
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
ps_status ps_host_expert_ffn_batch(ps_host_lane l, int n, const uint16_t* const* slabs, const int32_t* m,
                                   const int32_t* row0, int H, int F, const uint16_t* x, float* y) {
  return guarded([&] {
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
      l->pool->run([&](int tid) {
        int64_t u0, u1;
        range(U1, tid, u0, u1);
        if (u0 == u1) return;
        amx_config();
        for (int64_t u = u0; u < u1; ++u) {
          const int j = static_cast<int>(u / nb1), blk = static_cast<int>(u % nb1);
          const uint16_t* wg = slabs[j];
          const uint16_t* wu = wg + static_cast<size_t>(F) * H;
          for (int g = 0; g * kTok < m[j]; ++g)
            amx_gate_up_block(wg, wu, xb + xo[j] + static_cast<size_t>(g) * H * kTok, H, blk * 16,
                              hb + ho[j] + static_cast<size_t>(g) * F * kTok);
        }
        amx_release();
      });
      l->pool->run([&](int tid) {
        int64_t u0, u1;
        range(U2, tid, u0, u1);
        if (u0 == u1) return;
        amx_config();
        for (int64_t u = u0; u < u1; ++u) {
          const int j = static_cast<int>(u / nb2), blk = static_cast<int>(u % nb2);
          const uint16_t* wd = slabs[j] + static_cast<size_t>(2) * F * H;
          for (int g = 0; g * kTok < m[j]; ++g)
            amx_down_block(wd, hb + ho[j] + static_cast<size_t>(g) * F * kTok, H, F, blk * 16,
                           std::min(kTok, m[j] - g * kTok), y + static_cast<size_t>(row0[j] + g * kTok) * H);
        }
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

// Same as ps_host_expert_ffn_batch, weights read from z-slabs (AMX path only).
ps_status ps_host_expert_ffn_batch_z(ps_host_lane l, int n, const uint8_t* const* zslabs, const int32_t* m,
                                     const int32_t* row0, int H, int F, const uint16_t* x, float* y) {
  return guarded([&] {
    require(l && n >= 0 && (n == 0 || (zslabs && m && row0 && x && y)), "ps_host_expert_ffn_batch_z: null argument");
    require(H > 0 && F > 0 && H % 32 == 0 && F % 32 == 0, "ps_host_expert_ffn_batch_z: H, F % 32 == 0");
    if (!l->amx) fail(PS_ERUNTIME, "ps_host_expert_ffn_batch_z: needs AMX-BF16 (use the raw slabs)");
    std::vector<ZView> zv;
    for (int j = 0; j < n; ++j) {
      require(zslabs[j] != nullptr && m[j] >= 0 && m[j] <= 4096 && row0[j] >= 0, "ps_host_expert_ffn_batch_z: bad job");
      const ZHeader* h = reinterpret_cast<const ZHeader*>(zslabs[j]);
      require(h->magic == kZMagic && h->n == 3ull * H * F, "ps_host_expert_ffn_batch_z: not a z-slab of this shape");
      require(h->code_bits == 4, "ps_host_expert_ffn_batch_z: the lane decodes 4-bit z-slabs only");
      zv.emplace_back(zslabs[j]);
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
    l->pool->run([&](int tid) {
      const int64_t u0 = U1 * tid / T, u1 = U1 * (tid + 1) / T;
      if (u0 == u1) return;
      amx_config();
      for (int64_t u = u0; u < u1; ++u) {
        const int j = static_cast<int>(u / nb1), blk = static_cast<int>(u % nb1);
        for (int g = 0; g * kTok < m[j]; ++g)
          amx_gate_up_block_z(zv[j], H, F, xb + xo[j] + static_cast<size_t>(g) * H * kTok, blk * 16,
                              hb + ho[j] + static_cast<size_t>(g) * F * kTok);
      }
      amx_release();
    });
    l->pool->run([&](int tid) {
      const int64_t u0 = U2 * tid / T, u1 = U2 * (tid + 1) / T;
      if (u0 == u1) return;
      amx_config();
      for (int64_t u = u0; u < u1; ++u) {
        const int j = static_cast<int>(u / nb2), blk = static_cast<int>(u % nb2);
        for (int g = 0; g * kTok < m[j]; ++g)
          amx_down_block_z(zv[j], hb + ho[j] + static_cast<size_t>(g) * F * kTok, H, F, blk * 16,
                           std::min(kTok, m[j] - g * kTok), y + static_cast<size_t>(row0[j] + g * kTok) * H);
      }
      amx_release();
    });
  });
}

ps_status ps_host_expert_ffn(ps_host_lane l, const uint16_t* slab, int H, int F, const uint16_t* x, int m, float* y) {
  const int32_t zero = 0;
  return ps_host_expert_ffn_batch(l, 1, &slab, &m, &zero, H, F, x, y);
}

}  // extern "C"
