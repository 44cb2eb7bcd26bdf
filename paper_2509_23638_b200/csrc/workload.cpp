// Model shapes, top-k, routing map and the synthetic routing inputs.
//
// ModelSpec presets mirror workload.cpp:43-79 of the reference; ps_trace_inputs
// reproduces the RNG stream of generate_trace (workload.cpp:139-219) for everything
// that does NOT depend on routing (gate matrices, hidden trajectory, kappa draws), so
// the GPU router (K1) can recompute the trace's routing from identical inputs.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <vector>

#include "common.hpp"

namespace ps {
namespace {

constexpr uint64_t kMiB = 1ull << 20;

void validate_spec(const ps_model_spec& s) {
  if (s.num_layers < 1 || s.experts_per_layer < 1 || s.top_k < 1 || s.hidden_dim < 1)
    fail(PS_EINVAL, "ModelSpec: all counts must be >= 1");
  if (s.top_k > s.experts_per_layer) fail(PS_EINVAL, "ModelSpec: top_k exceeds experts_per_layer");
  if (!(0 <= s.group_begin_middle && s.group_begin_middle < s.group_begin_output &&
        s.group_begin_output <= s.num_layers))
    fail(PS_EINVAL, "ModelSpec: group bounds must be strictly increasing in [0, num_layers]");
}

// Group edges: first/last min(4, max(1, L/3)) layers (workload.cpp:50-53).
ps_model_spec make_spec(int layers, int experts, int k, uint64_t bytes, int hidden) {
  ps_model_spec s{};
  s.num_layers = layers;
  s.experts_per_layer = experts;
  s.top_k = k;
  s.expert_bytes = bytes;
  s.hidden_dim = hidden;
  int edge = std::min(4, std::max(1, layers / 3));
  s.group_begin_middle = edge;
  s.group_begin_output = layers - edge;
  validate_spec(s);
  return s;
}

int group_of(const ps_model_spec& s, int layer) {
  if (layer < 0 || layer >= s.num_layers) fail(PS_ERANGE, "ModelSpec::group_of: layer out of range");
  if (layer < s.group_begin_middle) return PS_GROUP_INPUT;
  if (layer < s.group_begin_output) return PS_GROUP_MIDDLE;
  return PS_GROUP_OUTPUT;
}

const ps_group_gen& gen_for(const ps_trace_gen_config& c, int g) {
  return g == PS_GROUP_INPUT ? c.input : g == PS_GROUP_OUTPUT ? c.output : c.middle;
}

void validate_gen(const ps_trace_gen_config& c) {
  for (const ps_group_gen* p : {&c.input, &c.middle, &c.output}) {
    if (p->rho < 0.0 || p->rho > 1.0) fail(PS_EINVAL, "TraceGenConfig: rho must be in [0,1]");
    if (p->kappa < 0.0 || p->kappa > 1.0) fail(PS_EINVAL, "TraceGenConfig: kappa must be in [0,1]");
    if (p->zipf_s < 0.0) fail(PS_EINVAL, "TraceGenConfig: zipf_s must be >= 0");
  }
  if (c.noise_scale < 0.0) fail(PS_EINVAL, "TraceGenConfig: noise_scale must be >= 0");
}

void unit_normalize(std::vector<double>& v) {
  double n = 0.0;
  for (double x : v) n += x * x;
  n = std::sqrt(n);
  if (n > 0.0)
    for (double& x : v) x /= n;
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" {

ps_status ps_spec_validate(const ps_model_spec* spec) {
  return guarded([&] { validate_spec(*spec); });
}

ps_status ps_spec_group_of(const ps_model_spec* spec, int layer, int* group) {
  return guarded([&] { *group = group_of(*spec, layer); });
}

ps_status ps_spec_preset(const char* name, ps_model_spec* out) {
  return guarded([&] {
    std::string n = name ? name : "";
    if (n == "mixtral") *out = make_spec(32, 8, 2, 336 * kMiB, 4096);
    else if (n == "qwen3") *out = make_spec(48, 128, 8, 9 * kMiB, 2048);
    else if (n == "deepseek" || n == "moonlight") *out = make_spec(26, 64, 6, kMiB * 33 / 2, 2048);
    else fail(PS_EINVAL, "unknown model preset: " + n);
  });
}

ps_status ps_desk_scale(const ps_model_spec* full, int num_layers, int experts, int hidden,
                        ps_model_spec* out) {
  return guarded([&] {
    *out = make_spec(num_layers, experts, std::min(full->top_k, experts), full->expert_bytes, hidden);
  });
}

ps_status ps_spec_ffn_dim(const ps_model_spec* spec, int* ffn_dim) {
  return guarded([&] {
    uint64_t per = 6ull * static_cast<uint64_t>(spec->hidden_dim);
    if (spec->hidden_dim < 1 || spec->expert_bytes % per != 0)
      fail(PS_EINVAL, "expert_bytes is not 3*H*F*2 for an integer F");
    *ffn_dim = static_cast<int>(spec->expert_bytes / per);
  });
}

// Ranking of workload.cpp:110-119 (stable sort by weight desc, ties lower index),
// as k selection rounds over the remaining entries.
int ps_topk_indices(const double* w, int n, int k, int32_t* out) {
  k = std::max(0, std::min(k, n));
  std::vector<unsigned char> used(static_cast<size_t>(std::max(n, 1)), 0);
  for (int r = 0; r < k; ++r) {
    int best = -1;
    for (int i = 0; i < n; ++i)
      if (!used[i] && (best < 0 || w[i] > w[best])) best = i;
    used[best] = 1;
    out[r] = best;
  }
  return k;
}

int ps_routing_map(const ps_model_spec* spec, int expert) {
  return (expert + 1) % spec->experts_per_layer;
}

// RNG order of generate_trace: L*E*H normals for the gate matrices,
// then per token H normals for a_0, then per layer: one uniform iff l >= 1 (the
// short-circuit at workload.cpp:183), and H normals iff l < L-1.
ps_status ps_trace_inputs(const ps_trace_gen_config* cfg, const ps_model_spec* spec, int batch,
                          uint64_t seed, double* gate, double* hidden, uint8_t* follow,
                          double* zipf_per_layer) {
  return guarded([&] {
    validate_gen(*cfg);
    validate_spec(*spec);
    require(batch >= 1, "generate_trace: batch_size must be >= 1");
    require(spec->hidden_dim >= 4, "generate_trace: hidden_dim must be >= 4");
    const int L = spec->num_layers, E = spec->experts_per_layer, D = spec->hidden_dim;

    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    std::uniform_real_distribution<double> unif(0.0, 1.0);

    const double wscale = 1.0 / std::sqrt(static_cast<double>(D));
    const size_t gate_n = static_cast<size_t>(L) * E * D;
    for (size_t i = 0; i < gate_n; ++i) {
      double g = gauss(rng) * wscale;
      if (gate) gate[i] = g;
    }
    if (zipf_per_layer)
      for (int l = 0; l < L; ++l) zipf_per_layer[l] = gen_for(*cfg, group_of(*spec, l)).zipf_s;

    std::vector<double> a(D), noise(D);
    for (int tok = 0; tok < batch; ++tok) {
      for (double& x : a) x = gauss(rng);
      unit_normalize(a);
      for (int l = 0; l < L; ++l) {
        const ps_group_gen& gp = gen_for(*cfg, group_of(*spec, l));
        const size_t step = static_cast<size_t>(tok) * L + l;
        bool f = l >= 1 && unif(rng) < gp.kappa;
        if (follow) follow[step] = f ? 1 : 0;
        if (hidden) std::memcpy(hidden + step * D, a.data(), sizeof(double) * D);
        if (l + 1 < L) {
          for (double& x : noise) x = gauss(rng);
          double proj = 0.0;
          for (int d = 0; d < D; ++d) proj += noise[d] * a[d];
          for (int d = 0; d < D; ++d) noise[d] -= proj * a[d];
          unit_normalize(noise);
          double nw = cfg->noise_scale * std::sqrt(std::max(0.0, 1.0 - gp.rho * gp.rho));
          for (int d = 0; d < D; ++d) a[d] = gp.rho * a[d] + nw * noise[d];
          unit_normalize(a);
        }
      }
    }
  });
}

// plan_residency over a hot table (predictor.cpp:405-433): (layer, expert) ranked by
// frequency desc, ties (layer, expert) asc; keep floor(budget / expert_bytes).
ps_status ps_plan_residency(const int64_t* freq, int L, int E, uint64_t budget_bytes,
                            uint64_t expert_bytes, int32_t* pairs_out, int* n_out) {
  return guarded([&] {
    require(expert_bytes != 0, "plan_residency: expert_bytes == 0");
    std::vector<int> idx(static_cast<size_t>(L) * E);
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = static_cast<int>(i);
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return freq[a] > freq[b]; });
    uint64_t count = std::min<uint64_t>(budget_bytes / expert_bytes, idx.size());
    for (uint64_t i = 0; i < count; ++i) {
      pairs_out[2 * i] = idx[i] / E;
      pairs_out[2 * i + 1] = idx[i] % E;
    }
    *n_out = static_cast<int>(count);
  });
}

}  // extern "C"
