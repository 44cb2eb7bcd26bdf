// A host model in C++ driving the B200 engine layer by layer through the C ABI — the call
// pattern INTEGRATION.md §3 documents for a model that runs its own attention between
// MoE layers (the reference's per-layer seam: plan_fn(inputs, l), simulator.cpp:136):
//
//   ps_engine_step_begin -> { attention(l) on my stream ; ps_engine_layer_forward(l) } -> ps_engine_step_end
//
// with the caller's own expert slabs (ps_engine_config.expert_weights). Checks the outputs
// are bit-identical to one ps_engine_decode_step on an identically configured engine.
// Built and run by tests/test_gpu_layer_api.py (needs a GPU); exits non-zero on failure.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ps_api.h"

#define OK(x)                                                                          \
  do {                                                                                 \
    ps_status s_ = (x);                                                                \
    if (s_ != PS_OK) {                                                                 \
      std::fprintf(stderr, "FAIL %s:%d %s -> %d: %s\n", __FILE__, __LINE__, #x, s_, ps_last_error()); \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)
#define CU(x)                                                                                      \
  do {                                                                                             \
    cudaError_t e_ = (x);                                                                          \
    if (e_ != cudaSuccess) {                                                                       \
      std::fprintf(stderr, "FAIL %s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                                \
    }                                                                                              \
  } while (0)

int main() {
  ps_model_spec full{}, spec{};
  OK(ps_spec_preset("mixtral", &full));
  OK(ps_desk_scale(&full, 4, 8, 256, &spec));
  const int H = spec.hidden_dim, F = 512, L = spec.num_layers, E = spec.experts_per_layer, K = spec.top_k, B = 8;
  spec.expert_bytes = 6ull * H * F;
  ps_trace_gen_config gen{{0.9, 0.5, 0.5}, {0.95, 0.6, 1.0}, {0.9, 0.5, 0.5}, 1.0};
  std::vector<double> gate64(static_cast<size_t>(L) * E * H), hid64(static_cast<size_t>(B) * L * H), zipf(L);
  std::vector<uint8_t> fol(static_cast<size_t>(B) * L);
  OK(ps_trace_inputs(&gen, &spec, B, 5, gate64.data(), hid64.data(), fol.data(), zipf.data()));
  std::vector<float> gate(gate64.begin(), gate64.end());
  // layer-major device inputs: hidden [L,B,H] f32, follow [L,B]
  std::vector<float> hid(static_cast<size_t>(L) * B * H);
  std::vector<uint8_t> fol_lb(static_cast<size_t>(L) * B);
  for (int t = 0; t < B; ++t)
    for (int l = 0; l < L; ++l) {
      for (int d = 0; d < H; ++d)
        hid[(static_cast<size_t>(l) * B + t) * H + d] = static_cast<float>(hid64[(static_cast<size_t>(t) * L + l) * H + d]);
      fol_lb[static_cast<size_t>(l) * B + t] = fol[static_cast<size_t>(t) * L + l];
    }
  // the model's own expert weights (host memory), here synthetic
  std::vector<std::vector<uint16_t>> slabs(static_cast<size_t>(L) * E, std::vector<uint16_t>(3ull * H * F));
  std::vector<const uint16_t*> ptrs;
  for (int l = 0; l < L; ++l)
    for (int e = 0; e < E; ++e) {
      OK(ps_init_expert_slab_host(slabs[static_cast<size_t>(l) * E + e].data(), H, F, 77, l, e));
      ptrs.push_back(slabs[static_cast<size_t>(l) * E + e].data());
    }
  std::vector<int32_t> resident;  // experts 0..3 of every layer in HBM (budget 50 %)
  for (int l = 0; l < L; ++l)
    for (int e = 0; e < E / 2; ++e) {
      resident.push_back(l);
      resident.push_back(e);
    }
  ps_engine_config cfg{};
  cfg.spec = spec;
  cfg.gen = gen;
  cfg.weight_seed = 0;
  cfg.budget_bytes = static_cast<uint64_t>(L) * (E / 2) * spec.expert_bytes;
  cfg.resident = resident.data();
  cfg.n_resident = static_cast<int32_t>(resident.size() / 2);
  cfg.max_batch = B;
  cfg.prefetch_slots = 8;
  cfg.policy = {PS_POLICY_ONDEMAND, 0};
  cfg.host_pinned = 1;
  cfg.expert_weights = ptrs.data();

  float *d_hid = nullptr, *y1 = nullptr, *y2 = nullptr, *x = nullptr;
  uint8_t* d_fol = nullptr;
  int32_t *ids1 = nullptr, *ids2 = nullptr;
  const size_t nh = static_cast<size_t>(L) * B * H;
  CU(cudaMalloc(&d_hid, nh * sizeof(float)));
  CU(cudaMalloc(&y1, nh * sizeof(float)));
  CU(cudaMalloc(&y2, nh * sizeof(float)));
  CU(cudaMalloc(&x, static_cast<size_t>(B) * H * sizeof(float)));
  CU(cudaMalloc(&d_fol, fol_lb.size()));
  CU(cudaMalloc(&ids1, static_cast<size_t>(L) * B * K * sizeof(int32_t)));
  CU(cudaMalloc(&ids2, static_cast<size_t>(L) * B * K * sizeof(int32_t)));
  CU(cudaMemcpy(d_hid, hid.data(), nh * sizeof(float), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_fol, fol_lb.data(), fol_lb.size(), cudaMemcpyHostToDevice));

  // whole step
  ps_engine e1 = nullptr, e2 = nullptr;
  OK(ps_engine_create(&cfg, &e1));
  OK(ps_engine_set_router(e1, gate.data()));
  OK(ps_engine_decode_step(e1, d_hid, d_fol, B, y1, ids1));

  // layer by layer, "attention" (a copy producing x_l) on the model's own stream
  OK(ps_engine_create(&cfg, &e2));
  OK(ps_engine_set_router(e2, gate.data()));
  cudaStream_t st;
  CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  OK(ps_engine_step_begin(e2, B));
  for (int l = 0; l < L; ++l) {
    const size_t off = static_cast<size_t>(l) * B * H;
    CU(cudaMemcpyAsync(x, d_hid + off, static_cast<size_t>(B) * H * sizeof(float), cudaMemcpyDeviceToDevice, st));
    OK(ps_engine_layer_forward(e2, l, x, d_fol + static_cast<size_t>(l) * B, y2 + off,
                               ids2 + static_cast<size_t>(l) * B * K, st));
  }
  OK(ps_engine_step_end(e2));
  CU(cudaStreamSynchronize(st));
  CU(cudaDeviceSynchronize());

  std::vector<float> h1(nh), h2(nh);
  std::vector<int32_t> i1(static_cast<size_t>(L) * B * K), i2(i1.size());
  CU(cudaMemcpy(h1.data(), y1, nh * sizeof(float), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(h2.data(), y2, nh * sizeof(float), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(i1.data(), ids1, i1.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(i2.data(), ids2, i2.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (std::memcmp(h1.data(), h2.data(), nh * sizeof(float)) != 0 ||
      std::memcmp(i1.data(), i2.data(), i1.size() * sizeof(int32_t)) != 0) {
    std::fprintf(stderr, "FAIL: per-layer outputs differ from the whole-step call\n");
    return 1;
  }
  double norm = 0;
  for (float v : h1) norm += static_cast<double>(v) * v;
  if (!(norm > 0)) {
    std::fprintf(stderr, "FAIL: zero output\n");
    return 1;
  }
  OK(ps_engine_destroy(e1));
  OK(ps_engine_destroy(e2));
  std::printf("layer loop ok (L=%d B=%d, |y|^2=%.6g)\n", L, B, norm);
  return 0;
}
