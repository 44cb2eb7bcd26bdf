// z-slab layout (lossless 12-bit transfer format of an expert slab; see zexpert.cu),
// shared by the CUDA decoder and the host expert lane's AMX z-path.
#pragma once
#include <cstddef>
#include <cstdint>

#ifdef __CUDACC__
#define PS_HD __host__ __device__
#else
#define PS_HD
#endif

namespace ps {

constexpr int kZBlock = 1024;  // values per block (escape prefix granularity)
constexpr int kZEscape = 15;   // escape code of the 4-bit format (the 3-bit format uses 7)
PS_HD inline uint32_t z_escape(uint32_t bits) { return (1u << bits) - 1u; }

struct ZHeader {  // at the start of every z-slab (64 bytes, keeps the streams 16-B aligned)
  uint64_t magic;  // "PSZSLAB1"
  uint64_t n;      // values (bf16 count)
  uint32_t base;   // exponent of code 0
  uint32_t nb;     // blocks
  uint64_t n_esc;  // escaped values
  uint64_t bytes;  // total z-slab bytes
  uint32_t code_bits;  // 3 or 4: exponent code width (escape = all ones)
  uint32_t tiled;      // 1: the values are an expert slab in the host lane's tile layout
  uint32_t tile_h, tile_f;  // H, F of that slab (tiled == 1); decoders emit row-major
  uint64_t pad;
};
static_assert(sizeof(ZHeader) == 64, "z header");
constexpr uint64_t kZMagic = 0x31424c534c5a5350ull;  // "PSZSLAB1"

PS_HD inline size_t z_lo_off() { return sizeof(ZHeader); }
PS_HD inline size_t z_codes_off(uint64_t n_pad) { return z_lo_off() + n_pad; }
// codes: `bits` per value, 32 values = 4*bits bytes (a lane's segment), little endian
PS_HD inline size_t z_escoff_off(uint64_t n_pad, uint32_t bits) { return z_codes_off(n_pad) + n_pad * bits / 8; }
PS_HD inline size_t z_esc_off(uint64_t n_pad, uint32_t nb, uint32_t bits) {
  return z_escoff_off(n_pad, bits) + 4ull * (nb + 1);
}

// Pointers into a z-slab (host view).
struct ZView {
  const uint8_t* lo;
  const uint8_t* codes;
  const uint32_t* esc_off;
  const uint8_t* esc;
  uint32_t base, bits, tiled;
  explicit ZView(const uint8_t* z) {
    const ZHeader* h = reinterpret_cast<const ZHeader*>(z);
    tiled = h->tiled;
    const uint64_t n_pad = static_cast<uint64_t>(h->nb) * kZBlock;
    bits = h->code_bits;
    lo = z + z_lo_off();
    codes = z + z_codes_off(n_pad);
    esc_off = reinterpret_cast<const uint32_t*>(z + z_escoff_off(n_pad, bits));
    esc = z + z_esc_off(n_pad, h->nb, bits);
    base = h->base;
  }
};

// Lane tile layout (ps_host_slab_tile): W_gate [F][H], W_up [F][H], W_down [H][F], each
// 16-row block stored as consecutive 16x32 tiles (1 KiB, row-major inside). Row-major index
// of the 32-value tile row that starts at tiled index v (v % 32 == 0).
PS_HD inline uint64_t z_untile(uint64_t v, uint32_t H, uint32_t F) {
  const uint64_t fh = static_cast<uint64_t>(F) * H;
  const uint64_t base = v < fh ? 0 : (v < 2 * fh ? fh : 2 * fh);
  const uint32_t K = v < 2 * fh ? H : F;
  const uint64_t t = v - base, tile = t >> 9;
  const uint32_t i = static_cast<uint32_t>(t >> 5) & 15u, nkb = K / 32;
  const uint64_t rb = tile / nkb, kb = tile - rb * nkb;
  return base + (rb * 16 + i) * K + kb * 32;
}

}  // namespace ps
