// prescope_b200.hpp — header-only C++ mirror of the reference's operator API for the
// hot path (namespace prescope, /root/reference/proj/include/prescope/*.hpp), built on
// the C ABI of ps_api.h. Reference call sites for the scheduler / pipeline / routing /
// residency entry points compile against this header unchanged; failures re-throw the
// reference's exception types (tools/prescope_main.cpp:427-434):
//   PS_EINVAL -> std::invalid_argument, PS_ERANGE -> std::out_of_range, else std::runtime_error.
// Link with libprescope_b200.so.
#pragma once

#include <algorithm>
#include <cstdint>
#include <functional>
#include <map>
#include <set>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "ps_api.h"

namespace prescope {

inline void ps_throw_if(ps_status s) {
  if (s == PS_OK) return;
  const std::string msg = ps_last_error();
  if (s == PS_EINVAL) throw std::invalid_argument(msg);
  if (s == PS_ERANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}

// ---------------------------------------------------------------- workload.hpp:12-66
enum class LayerGroup { Input = 0, Middle = 1, Output = 2 };

struct ModelSpec {
  int num_layers = 0;
  int experts_per_layer = 0;
  int top_k = 0;
  std::uint64_t expert_bytes = 0;
  int hidden_dim = 0;
  int group_begin_middle = 0;
  int group_begin_output = 0;

  ps_model_spec c() const {
    return {num_layers, experts_per_layer, top_k, hidden_dim, expert_bytes, group_begin_middle, group_begin_output};
  }
  static ModelSpec from(const ps_model_spec& s) {
    return {s.num_layers, s.experts_per_layer, s.top_k, s.expert_bytes, s.hidden_dim, s.group_begin_middle,
            s.group_begin_output};
  }
  void validate() const {
    ps_model_spec s = c();
    ps_throw_if(ps_spec_validate(&s));
  }
  LayerGroup group_of(int layer) const {
    ps_model_spec s = c();
    int g = 0;
    ps_throw_if(ps_spec_group_of(&s, layer, &g));
    return static_cast<LayerGroup>(g);
  }
  bool operator==(const ModelSpec&) const = default;
};

inline ModelSpec spec_preset(const std::string& name) {
  ps_model_spec s{};
  ps_throw_if(ps_spec_preset(name.c_str(), &s));
  return ModelSpec::from(s);
}
inline ModelSpec mixtral_spec() { return spec_preset("mixtral"); }
inline ModelSpec qwen3_spec() { return spec_preset("qwen3"); }
inline ModelSpec deepseek_spec() { return spec_preset("deepseek"); }
inline ModelSpec moonlight_spec() { return spec_preset("moonlight"); }
inline ModelSpec desk_scale(const ModelSpec& full, int num_layers, int experts_per_layer, int hidden_dim) {
  ps_model_spec f = full.c(), s{};
  ps_throw_if(ps_desk_scale(&f, num_layers, experts_per_layer, hidden_dim, &s));
  return ModelSpec::from(s);
}

inline std::vector<int> topk_indices(const std::vector<double>& weights, int k) {
  std::vector<int32_t> out(std::max(0, std::min<int>(k, static_cast<int>(weights.size()))));
  int n = ps_topk_indices(weights.data(), static_cast<int>(weights.size()), k, out.data());
  return std::vector<int>(out.begin(), out.begin() + n);
}

// ---------------------------------------------------------------- trace files
// TraceStep / Trace (workload.hpp:47-66), TraceFormatError / TraceChecksumError
// (workload.hpp:106-111), write_trace / read_trace / fnv1a64 (workload.cpp:290-436),
// aggregate_layer_loads (workload.cpp:283-288).
struct TraceStep {
  int layer = 0;
  std::vector<double> hidden;
  std::vector<double> gate_weights;
  std::vector<int> active_experts;
  std::map<int, int> tokens_per_expert;
  bool operator==(const TraceStep&) const = default;
};

struct Trace {
  ModelSpec spec;
  int batch_size = 0;
  std::uint64_t seed = 0;
  std::vector<TraceStep> steps;  // ordered by (token, layer)
  bool operator==(const Trace&) const = default;
  const TraceStep& step(int token, int layer) const {
    const size_t i = static_cast<size_t>(token) * spec.num_layers + layer;
    if (token < 0 || layer < 0 || layer >= spec.num_layers || i >= steps.size())
      throw std::out_of_range("Trace::step: index out of range");
    return steps[i];
  }
};

struct TraceFormatError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct TraceChecksumError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void trace_throw_if(ps_status s) {
  if (s == PS_OK) return;
  const std::string msg = ps_last_error();
  if (s == PS_ERUNTIME && msg.rfind("TraceChecksumError", 0) == 0) throw TraceChecksumError(msg);
  if (s == PS_ERUNTIME && msg.rfind("TraceFormatError", 0) == 0) throw TraceFormatError(msg);
  ps_throw_if(s);
}
}  // namespace detail

inline std::uint64_t fnv1a64(const std::string& data) { return ps_fnv1a64(data.data(), data.size()); }

inline Trace read_trace(const std::string& path) {
  ps_trace h = nullptr;
  detail::trace_throw_if(ps_trace_read(path.c_str(), &h));
  ps_model_spec s{};
  int32_t b = 0;
  uint64_t seed = 0;
  ps_trace_shape(h, &s, &b, &seed, nullptr);
  const int L = s.num_layers, E = s.experts_per_layer, K = s.top_k, H = s.hidden_dim;
  const size_t n = static_cast<size_t>(b) * L;
  std::vector<double> hid(n * H), gw(n * E);
  std::vector<int32_t> act(n * K), tok(n * E);
  ps_trace_arrays(h, hid.data(), gw.data(), act.data(), tok.data());
  ps_trace_free(h);
  Trace t;
  t.spec = ModelSpec::from(s);
  t.batch_size = b;
  t.seed = seed;
  t.steps.resize(n);
  for (size_t i = 0; i < n; ++i) {
    TraceStep& st = t.steps[i];
    st.layer = static_cast<int>(i % L);
    st.hidden.assign(hid.begin() + i * H, hid.begin() + (i + 1) * H);
    st.gate_weights.assign(gw.begin() + i * E, gw.begin() + (i + 1) * E);
    st.active_experts.assign(act.begin() + i * K, act.begin() + (i + 1) * K);
    for (int e = 0; e < E; ++e)
      if (tok[i * E + e]) st.tokens_per_expert[e] = tok[i * E + e];
  }
  return t;
}

inline void write_trace(const Trace& t, const std::string& path) {
  const ModelSpec& s = t.spec;
  const int E = s.experts_per_layer, K = s.top_k, H = s.hidden_dim;
  const size_t n = t.steps.size();
  if (n != static_cast<size_t>(t.batch_size) * s.num_layers)
    throw std::invalid_argument("write_trace: steps != batch_size * num_layers");
  std::vector<double> hid(n * H), gw(n * E);
  std::vector<int32_t> act(n * K), tok(n * E, 0);
  for (size_t i = 0; i < n; ++i) {
    const TraceStep& st = t.steps[i];
    if (st.hidden.size() != static_cast<size_t>(H) || st.gate_weights.size() != static_cast<size_t>(E) ||
        st.active_experts.size() != static_cast<size_t>(K))
      throw std::invalid_argument("write_trace: step vector sizes do not match the spec");
    std::copy(st.hidden.begin(), st.hidden.end(), hid.begin() + i * H);
    std::copy(st.gate_weights.begin(), st.gate_weights.end(), gw.begin() + i * E);
    std::copy(st.active_experts.begin(), st.active_experts.end(), act.begin() + i * K);
    for (auto [e, m] : st.tokens_per_expert) tok[i * E + e] = m;
  }
  const ps_model_spec cs = s.c();
  detail::trace_throw_if(
      ps_trace_write(path.c_str(), &cs, t.batch_size, t.seed, hid.data(), gw.data(), act.data(), tok.data()));
}

inline std::map<int, int> aggregate_layer_loads(const Trace& trace, int layer) {
  std::map<int, int> loads;
  for (int tok = 0; tok < trace.batch_size; ++tok)
    for (auto [e, m] : trace.step(tok, layer).tokens_per_expert) loads[e] += m;
  return loads;
}
inline int routing_map(const ModelSpec& spec, int expert) {
  ps_model_spec s = spec.c();
  return ps_routing_map(&s, expert);
}

// -------------------------------------------------------------- cost_model.hpp:13-103
using Ticks = std::int64_t;
inline Ticks to_ticks(double x) { return ps_to_ticks(x); }

struct CostParams {
  Ticks t_io = 0, t_g = 0, t_attn = 0;
  double beta = 0.0;
  Ticks startup = 0, alpha = 0;
  ps_cost_params c() const { return {t_io, t_g, t_attn, beta, startup, alpha}; }
  void validate() const {
    ps_cost_params p = c();
    ps_throw_if(ps_cost_params_validate(&p));
  }
};

enum class ExpertLocation { Resident = 0, InFlight = 1, Host = 2 };

struct ExpertLoad {
  int expert = 0;
  int layer = 0;
  int tokens = 0;
  ExpertLocation location = ExpertLocation::Host;
};

struct HitStats {
  double r_hit = 1.0, r_miss = 0.0;
  int window = 32;
  void record(bool hit) {
    ps_hit_stats s{r_hit, r_miss, window};
    ps_throw_if(ps_hit_stats_record(&s, hit));
    r_hit = s.r_hit;
    r_miss = s.r_miss;
  }
};

inline Ticks cpu_cost(int tokens, const CostParams& params) {
  ps_cost_params p = params.c();
  int64_t out = 0;
  ps_throw_if(ps_cpu_cost(tokens, &p, &out));
  return out;
}

struct PrefetchCount {
  double f = 0.0;
  int f_int = 0;
};
inline PrefetchCount overlap_prefetch_count(Ticks t_gap, const CostParams& params) {
  ps_cost_params p = params.c();
  PrefetchCount pc;
  ps_throw_if(ps_overlap_prefetch_count(t_gap, &p, &pc.f, &pc.f_int));
  return pc;
}
inline double prefetch_gain(const HitStats& stats, double f, int f_int, const CostParams& params) {
  ps_hit_stats s{stats.r_hit, stats.r_miss, stats.window};
  ps_cost_params p = params.c();
  return ps_prefetch_gain(&s, f, f_int, &p);
}

// -------------------------------------------------------------- scheduler.hpp:13-105
struct LayerInputs {
  std::vector<ExpertLoad> e_cur, e_next, e_next2;
  CostParams params;
  HitStats stats;
};

struct DecisionTrace {
  std::vector<Ticks> sweep_gpu, sweep_cpu;
  Ticks t_g_at_split = 0, t_c_at_split = 0, t_gap = 0;
  double f = 0.0;
  int f_int = 0;
  double xi = 0.0;
  bool widened_window = false, all_gpu_fallback = false;
};

struct LayerPlan {
  std::vector<ExpertLoad> cpu_set, ondemand_seq, prefetch_seq;
  bool prefetch_from_widened = false;
  int split_index = 0;
  int issued_prefetches = 0;
  DecisionTrace trace;
};

struct SchedulerPolicy {
  enum class Kind { PreSched = 0, LayerGreedy = 1, OnDemandOnly = 2, FixedPrefetch = 3, Oracle = 4 };
  Kind kind = Kind::PreSched;
  int fixed_prefetch = 0;
  static SchedulerPolicy parse(const std::string& text) {
    ps_policy p{};
    ps_throw_if(ps_policy_parse(text.c_str(), &p));
    return {static_cast<Kind>(p.kind), p.fixed_prefetch};
  }
  std::string name() const {
    char buf[64];
    ps_throw_if(ps_policy_name(c(), buf, sizeof(buf)));
    return buf;
  }
  ps_policy c() const { return {static_cast<int32_t>(kind), fixed_prefetch}; }
};

namespace detail {
inline std::vector<ps_expert_load> to_c(const std::vector<ExpertLoad>& v) {
  std::vector<ps_expert_load> out;
  out.reserve(v.size());
  for (const ExpertLoad& e : v) out.push_back({e.expert, e.layer, e.tokens, static_cast<int32_t>(e.location)});
  return out;
}
inline std::vector<ExpertLoad> from_c(const ps_expert_load* p, int n) {
  std::vector<ExpertLoad> out;
  for (int i = 0; i < n; ++i) out.push_back({p[i].expert, p[i].layer, p[i].tokens, static_cast<ExpertLocation>(p[i].location)});
  return out;
}
inline LayerPlan run_plan(const LayerInputs& in, ps_policy pol) {
  auto cur = to_c(in.e_cur), nxt = to_c(in.e_next), nxt2 = to_c(in.e_next2);
  ps_layer_inputs ci{cur.data(), static_cast<int32_t>(cur.size()), nxt.data(), static_cast<int32_t>(nxt.size()),
                     nxt2.data(), static_cast<int32_t>(nxt2.size()), in.params.c(),
                     {in.stats.r_hit, in.stats.r_miss, in.stats.window}};
  const size_t cap = std::max({cur.size(), nxt.size(), nxt2.size(), size_t{1}});
  std::vector<ps_expert_load> cpu(cap), od(cap), pf(cap);
  std::vector<int64_t> sg(cur.size() + nxt.size() + 1), sc(sg.size());
  ps_layer_plan p{};
  p.cpu_set = cpu.data();
  p.ondemand_seq = od.data();
  p.prefetch_seq = pf.data();
  p.trace.sweep_gpu = sg.data();
  p.trace.sweep_cpu = sc.data();
  ps_throw_if(ps_presched_plan(&ci, pol, &p));
  LayerPlan out;
  out.cpu_set = from_c(cpu.data(), p.n_cpu);
  out.ondemand_seq = from_c(od.data(), p.n_ondemand);
  out.prefetch_seq = from_c(pf.data(), p.n_prefetch);
  out.prefetch_from_widened = p.prefetch_from_widened;
  out.split_index = p.split_index;
  out.issued_prefetches = p.issued_prefetches;
  out.trace.sweep_gpu.assign(sg.begin(), sg.begin() + p.trace.n_sweep);
  out.trace.sweep_cpu.assign(sc.begin(), sc.begin() + p.trace.n_sweep);
  out.trace.t_g_at_split = p.trace.t_g_at_split;
  out.trace.t_c_at_split = p.trace.t_c_at_split;
  out.trace.t_gap = p.trace.t_gap;
  out.trace.f = p.trace.f;
  out.trace.f_int = p.trace.f_int;
  out.trace.xi = p.trace.xi;
  out.trace.widened_window = p.trace.widened_window;
  out.trace.all_gpu_fallback = p.trace.all_gpu_fallback;
  return out;
}
}  // namespace detail

inline LayerPlan schedule_layer(const LayerInputs& in) { return detail::run_plan(in, {PS_POLICY_PRESCHED, 0}); }
inline LayerPlan greedy_layer_baseline(const LayerInputs& in) { return detail::run_plan(in, {PS_POLICY_GREEDY, 0}); }
inline LayerPlan ondemand_only_plan(const LayerInputs& in) { return detail::run_plan(in, {PS_POLICY_ONDEMAND, 0}); }
inline LayerPlan fixed_prefetch_plan(const LayerInputs& in, int c) { return detail::run_plan(in, {PS_POLICY_FIXED, c}); }
inline LayerPlan plan_layer(const LayerInputs& in, const SchedulerPolicy& p) { return detail::run_plan(in, p.c()); }

// -------------------------------------------------------------- simulator.hpp:14-128
enum class Resource { Gpu = 0, Cpu = 1, IoChannel = 2 };
enum class EventKind { Attention, GpuExpert, CpuExpert, Load, Prefetch, Idle };

struct TimelineEvent {
  Ticks t_start = 0, t_end = 0;
  Resource resource = Resource::Gpu;
  EventKind kind = EventKind::Attention;
  int layer = 0, expert = -1, tokens = 0;
  bool operator==(const TimelineEvent&) const = default;
};

struct Timeline {
  std::vector<TimelineEvent> events;
  std::vector<Ticks> layer_start, layer_end;
  Ticks makespan = 0;
  bool operator==(const Timeline&) const = default;
};

struct LayerLoads {
  std::map<int, int> truth, predicted;
};

struct PipelineInstance {
  std::vector<LayerLoads> layers;
  std::set<std::pair<int, int>> resident;
  std::vector<LayerGroup> groups;
  int num_layers() const { return static_cast<int>(layers.size()); }
};

struct SimOptions {
  int cpu_slots = 1;
  int prefetch_slots = 8;
  double initial_hit_rate = 1.0;
  int hit_window = 32;
};

struct SimResult {
  Timeline timeline;
  std::vector<LayerPlan> plans;  // split/issued/widened summary only
};

namespace detail {
struct DenseInstance {
  int L = 0, E = 1;
  std::vector<int32_t> truth, predicted, groups;
  std::vector<uint8_t> resident;
  ps_pipeline_instance c{};
  explicit DenseInstance(const PipelineInstance& inst) {
    L = inst.num_layers();
    for (const LayerLoads& l : inst.layers) {
      for (auto [e, m] : l.truth) E = std::max(E, e + 1);
      for (auto [e, m] : l.predicted) E = std::max(E, e + 1);
    }
    for (auto [l, e] : inst.resident) E = std::max(E, e + 1);
    truth.assign(static_cast<size_t>(L) * E, 0);
    predicted.assign(truth.size(), 0);
    resident.assign(truth.size(), 0);
    for (int l = 0; l < L; ++l) {
      for (auto [e, m] : inst.layers[l].truth) truth[static_cast<size_t>(l) * E + e] = m;
      for (auto [e, m] : inst.layers[l].predicted) predicted[static_cast<size_t>(l) * E + e] = m;
    }
    for (auto [l, e] : inst.resident)
      if (l >= 0 && l < L) resident[static_cast<size_t>(l) * E + e] = 1;
    for (LayerGroup g : inst.groups) groups.push_back(static_cast<int32_t>(g));
    c = {L, E, truth.data(), predicted.data(), resident.data(), groups.empty() ? nullptr : groups.data()};
  }
};
inline std::vector<TimelineEvent> events_from(const ps_timeline_event* ev, int n) {
  std::vector<TimelineEvent> out;
  for (int i = 0; i < n; ++i)
    out.push_back({ev[i].t_start, ev[i].t_end, static_cast<Resource>(ev[i].resource),
                   static_cast<EventKind>(ev[i].kind), ev[i].layer, ev[i].expert, ev[i].tokens});
  return out;
}
}  // namespace detail

inline SimResult simulate_policy(const PipelineInstance& instance, const SchedulerPolicy& policy,
                                 const CostParams& params, const SimOptions& options = {}) {
  detail::DenseInstance d(instance);
  std::vector<ps_timeline_event> ev(4 * (static_cast<size_t>(d.L) * d.E + d.L) + 16);
  std::vector<int64_t> ls(d.L), le(d.L);
  std::vector<int32_t> summary(4 * static_cast<size_t>(d.L));
  ps_timeline t{ev.data(), static_cast<int32_t>(ev.size()), 0, ls.data(), le.data(), 0, summary.data()};
  ps_cost_params p = params.c();
  ps_sim_options o{options.cpu_slots, options.prefetch_slots, options.initial_hit_rate, options.hit_window};
  ps_throw_if(ps_simulate_pipeline(&d.c, policy.c(), nullptr, nullptr, &p, &o, &t));
  SimResult r;
  r.timeline.events = detail::events_from(ev.data(), t.n_events);
  r.timeline.layer_start = ls;
  r.timeline.layer_end = le;
  r.timeline.makespan = t.makespan;
  for (int l = 0; l < d.L; ++l) {
    LayerPlan lp;
    lp.split_index = summary[4 * l];
    lp.issued_prefetches = summary[4 * l + 1];
    lp.prefetch_from_widened = summary[4 * l + 2];
    r.plans.push_back(lp);
  }
  return r;
}

inline std::vector<std::string> verify_timeline(const Timeline& timeline, const PipelineInstance& instance,
                                                const CostParams& params) {
  detail::DenseInstance d(instance);
  std::vector<ps_timeline_event> ev;
  for (const TimelineEvent& e : timeline.events)
    ev.push_back({e.t_start, e.t_end, static_cast<int32_t>(e.resource), static_cast<int32_t>(e.kind), e.layer,
                  e.expert, e.tokens});
  ps_cost_params p = params.c();
  int n = 0;
  std::string buf(1 << 16, '\0');
  ps_throw_if(ps_verify_timeline(ev.data(), static_cast<int>(ev.size()), &d.c, &p, &n, buf.data(),
                                 static_cast<int>(buf.size())));
  std::vector<std::string> out;
  size_t pos = 0;
  const std::string all = buf.c_str();
  while (pos < all.size()) {
    size_t nl = all.find('\n', pos);
    out.push_back(all.substr(pos, nl - pos));
    pos = nl == std::string::npos ? all.size() : nl + 1;
  }
  return out;
}

struct Metrics {
  std::vector<Ticks> per_layer_latency;
  std::vector<Ticks> cpu_gpu_gap;
  Ticks makespan = 0;
  Ticks decode_latency = 0;
  double throughput_tokens_per_s = 0.0;
  double io_busy_fraction = 0.0;
  double gpu_idle_fraction = 0.0;
};

inline Metrics compute_metrics(const Timeline& timeline, int output_tokens) {
  std::vector<ps_timeline_event> ev;
  for (const TimelineEvent& e : timeline.events)
    ev.push_back({e.t_start, e.t_end, static_cast<int32_t>(e.resource), static_cast<int32_t>(e.kind), e.layer,
                  e.expert, e.tokens});
  const int L = static_cast<int>(timeline.layer_start.size());
  Metrics m;
  m.per_layer_latency.resize(L);
  m.cpu_gpu_gap.resize(L);
  ps_metrics c{};
  ps_throw_if(ps_compute_metrics(ev.data(), static_cast<int>(ev.size()), timeline.layer_start.data(),
                                 timeline.layer_end.data(), L, timeline.makespan, output_tokens, &c,
                                 m.per_layer_latency.data(), m.cpu_gpu_gap.data()));
  m.makespan = c.makespan;
  m.decode_latency = c.decode_latency;
  m.throughput_tokens_per_s = c.throughput_tokens_per_s;
  m.io_busy_fraction = c.io_busy_fraction;
  m.gpu_idle_fraction = c.gpu_idle_fraction;
  return m;
}

// -------------------------------------------------------------- predictor.hpp:145-157
inline std::vector<std::pair<int, int>> plan_residency_from_freq(const std::vector<std::vector<long>>& freq,
                                                                 std::uint64_t budget_bytes,
                                                                 std::uint64_t expert_bytes) {
  const int L = static_cast<int>(freq.size()), E = L ? static_cast<int>(freq[0].size()) : 0;
  std::vector<int64_t> f;
  for (const auto& row : freq) f.insert(f.end(), row.begin(), row.end());
  std::vector<int32_t> pairs(2 * f.size() + 2);
  int n = 0;
  ps_throw_if(ps_plan_residency(f.data(), L, E, budget_bytes, expert_bytes, pairs.data(), &n));
  std::vector<std::pair<int, int>> out;
  for (int i = 0; i < n; ++i) out.emplace_back(pairs[2 * i], pairs[2 * i + 1]);
  return out;
}

}  // namespace prescope
