// Deterministic synthetic expert weights: bf16 ~ N(0, 1/sqrt(fan_in)),
// keyed by (seed, layer, expert, element index), so the device can materialise the
// resident experts in HBM and the host the offloaded ones without moving 90 GB.
//
// value = (u0+u1+u2+u3 - 2*65535) * c, ui the four 16-bit lanes of mix64(base + i),
// c = 1/(sigma_IH * sqrt(fan_in)) rounded once to f32. The integer sum is exact in f32
// and the product is one IEEE rounding, so host and device produce identical bits.
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

#include "device_common.cuh"

namespace ps {
namespace {

// Std-dev of the sum of four independent uniform integers in [0, 65535].
constexpr double kIrwinHallSigma = 37837.226631;  // sqrt(4 * (65536^2 - 1) / 12)

__host__ __device__ inline uint64_t slab_base(uint64_t seed, int layer, int expert) {
  return mix64(seed ^ mix64((static_cast<uint64_t>(static_cast<uint32_t>(layer)) << 32) |
                            static_cast<uint32_t>(expert)));
}

__host__ __device__ inline float hashed_value(uint64_t base, uint64_t i, float c) {
  const uint64_t r = mix64(base + i);
  const int s = static_cast<int>(r & 0xffff) + static_cast<int>((r >> 16) & 0xffff) +
                static_cast<int>((r >> 32) & 0xffff) + static_cast<int>((r >> 48) & 0xffff) - 2 * 65535;
  return static_cast<float>(s) * c;
}

inline uint16_t host_bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x40);
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

void scales(int H, int F, float* c_in, float* c_down) {
  *c_in = static_cast<float>(1.0 / (kIrwinHallSigma * std::sqrt(static_cast<double>(H))));
  *c_down = static_cast<float>(1.0 / (kIrwinHallSigma * std::sqrt(static_cast<double>(F))));
}

__global__ void init_slab_kernel(uint16_t* __restrict__ slab, uint64_t n, uint64_t n_in, uint64_t base,
                                 float c_in, float c_down) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x * 8;
  for (uint64_t i = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 8; i < n; i += stride) {
    uint32_t packed[4];
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      const float a = hashed_value(base, i + j, i + j < n_in ? c_in : c_down);
      const float b = hashed_value(base, i + j + 1, i + j + 1 < n_in ? c_in : c_down);
      packed[j / 2] = static_cast<uint32_t>(f32_to_bf16_rne(a)) | (static_cast<uint32_t>(f32_to_bf16_rne(b)) << 16);
    }
    *reinterpret_cast<uint4*>(slab + i) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
  }
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" {

ps_status ps_init_expert_slab(uint16_t* slab, int H, int F, uint64_t seed, int layer, int expert, void* stream) {
  return guarded([&] {
    require(slab && H > 0 && F > 0 && (static_cast<uint64_t>(H) * F) % 8 == 0, "ps_init_expert_slab: bad shape");
    float c_in, c_down;
    scales(H, F, &c_in, &c_down);
    const uint64_t n = 3ull * H * F, n_in = 2ull * H * F;
    init_slab_kernel<<<kNumSMs * 8, 256, 0, as_stream(stream)>>>(slab, n, n_in, slab_base(seed, layer, expert),
                                                                 c_in, c_down);
    PS_LAUNCH_CHECK("init_slab_kernel");
  });
}

ps_status ps_init_expert_slab_host(uint16_t* slab, int H, int F, uint64_t seed, int layer, int expert) {
  return guarded([&] {
    require(slab && H > 0 && F > 0, "ps_init_expert_slab_host: bad shape");
    float c_in, c_down;
    scales(H, F, &c_in, &c_down);
    const uint64_t n = 3ull * H * F, n_in = 2ull * H * F, base = slab_base(seed, layer, expert);
    const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    const uint64_t chunk = (n + nt - 1) / nt;
    for (unsigned t = 0; t < nt; ++t)
      pool.emplace_back([=] {
        const uint64_t end = std::min(n, (t + 1) * chunk);
        for (uint64_t i = t * chunk; i < end; ++i) slab[i] = host_bf16(hashed_value(base, i, i < n_in ? c_in : c_down));
      });
    for (auto& th : pool) th.join();
  });
}

}  // extern "C"
