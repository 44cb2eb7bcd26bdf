// TEST INFRASTRUCTURE ONLY — not product code.
//
// extern "C" shim over the UNMODIFIED reference library (/root/reference/proj/src),
// compiled by oracle/Makefile into oracle/_ref/libprescope_ref.so. Only tests/,
// __graft_entry__.smoke() and bench.py's CPU-baseline leg may load it: it is the
// checker that pins oracle/oracle.c and the fixtures under tests/golden/, and the
// "reference" CPU arm of bench.py. Nothing in paper_2509_23638_b200/ links it.
//
// Every entry point returns 0 on success and maps the reference's exceptions the
// same way the reference CLI does (tools/prescope_main.cpp:427-434):
//   1 = std::invalid_argument, 2 = std::out_of_range, 3 = std::runtime_error/other.
#include <algorithm>
#include <cmath>
#include <random>
#include <chrono>
#include <thread>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <functional>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "json.hpp"
#include "prescope/experiment.hpp"
#include "prescope/golden.hpp"
#include "prescope/predictor.hpp"
#include "prescope/scheduler.hpp"
#include "prescope/simulator.hpp"
#include "prescope/workload.hpp"

using namespace prescope;

extern "C" {

struct ref_spec {
  int32_t num_layers, experts, top_k, hidden;
  uint64_t expert_bytes;
  int32_t group_begin_middle, group_begin_output;
};
struct ref_gen {
  double rho[3], kappa[3], zipf[3];  // input, middle, output
  double noise_scale;
};
struct ref_load {
  int32_t expert, layer, tokens;
};
struct ref_params {
  int64_t t_io, t_g, t_attn;
  double beta;
  int64_t startup, alpha;
};
struct ref_stats {
  double r_hit, r_miss;
  int32_t window;
};
struct ref_plan_info {
  int32_t split_index, issued_prefetches, prefetch_from_widened;
  int32_t n_cpu, n_od, n_pf, n_sweep;
  int64_t t_g_at_split, t_c_at_split, t_gap;
  double f;
  int32_t f_int;
  double xi;
  int32_t widened_window, all_gpu_fallback;
};
struct ref_event {
  int64_t t_start, t_end;
  int32_t resource, kind, layer, expert, tokens;
};
struct ref_sim_opts {
  int32_t cpu_slots, prefetch_slots;
  double initial_hit_rate;
  int32_t hit_window;
};
}

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

ModelSpec to_spec(const ref_spec& s) {
  ModelSpec m;
  m.num_layers = s.num_layers;
  m.experts_per_layer = s.experts;
  m.top_k = s.top_k;
  m.expert_bytes = s.expert_bytes;
  m.hidden_dim = s.hidden;
  m.group_begin_middle = s.group_begin_middle;
  m.group_begin_output = s.group_begin_output;
  return m;
}

TraceGenConfig to_gen(const ref_gen& g) {
  TraceGenConfig c;
  c.input = {g.rho[0], g.kappa[0], g.zipf[0]};
  c.middle = {g.rho[1], g.kappa[1], g.zipf[1]};
  c.output = {g.rho[2], g.kappa[2], g.zipf[2]};
  c.noise_scale = g.noise_scale;
  return c;
}

CostParams to_params(const ref_params& p) {
  CostParams c;
  c.t_io = p.t_io;
  c.t_g = p.t_g;
  c.t_attn = p.t_attn;
  c.beta = p.beta;
  c.startup = p.startup;
  c.alpha = p.alpha;
  return c;
}

std::vector<ExpertLoad> to_loads(const ref_load* l, int n) {
  std::vector<ExpertLoad> v;
  for (int i = 0; i < n; ++i) v.push_back({l[i].expert, l[i].layer, l[i].tokens, ExpertLocation::Host});
  return v;
}

void from_loads(const std::vector<ExpertLoad>& v, ref_load* out) {
  for (size_t i = 0; i < v.size(); ++i) out[i] = {v[i].expert, v[i].layer, v[i].tokens};
}

SchedulerPolicy to_policy(int kind, int fixed_c) {
  SchedulerPolicy p;
  p.kind = static_cast<SchedulerPolicy::Kind>(kind);
  p.fixed_prefetch = fixed_c;
  return p;
}

void fill_info(const LayerPlan& plan, ref_plan_info* info) {
  info->split_index = plan.split_index;
  info->issued_prefetches = plan.issued_prefetches;
  info->prefetch_from_widened = plan.prefetch_from_widened;
  info->n_cpu = static_cast<int32_t>(plan.cpu_set.size());
  info->n_od = static_cast<int32_t>(plan.ondemand_seq.size());
  info->n_pf = static_cast<int32_t>(plan.prefetch_seq.size());
  info->n_sweep = static_cast<int32_t>(plan.trace.sweep_gpu.size());
  info->t_g_at_split = plan.trace.t_g_at_split;
  info->t_c_at_split = plan.trace.t_c_at_split;
  info->t_gap = plan.trace.t_gap;
  info->f = plan.trace.f;
  info->f_int = plan.trace.f_int;
  info->xi = plan.trace.xi;
  info->widened_window = plan.trace.widened_window;
  info->all_gpu_fallback = plan.trace.all_gpu_fallback;
}

PipelineInstance make_instance(int L, const int32_t* truth, int n_truth, const int32_t* pred,
                               int n_pred, const int32_t* resident, int n_res,
                               const int32_t* groups) {
  PipelineInstance inst;
  inst.layers.resize(L);
  for (int i = 0; i < n_truth; ++i) inst.layers.at(truth[3 * i]).truth[truth[3 * i + 1]] = truth[3 * i + 2];
  for (int i = 0; i < n_pred; ++i) inst.layers.at(pred[3 * i]).predicted[pred[3 * i + 1]] = pred[3 * i + 2];
  for (int i = 0; i < n_res; ++i) inst.resident.insert({resident[2 * i], resident[2 * i + 1]});
  if (groups)
    for (int l = 0; l < L; ++l) inst.groups.push_back(static_cast<LayerGroup>(groups[l]));
  return inst;
}

nlohmann::json timeline_json(const Timeline& t) {
  nlohmann::json ev = nlohmann::json::array();
  for (const TimelineEvent& e : t.events)
    ev.push_back({e.t_start, e.t_end, static_cast<int>(e.resource), static_cast<int>(e.kind),
                  e.layer, e.expert, e.tokens});
  return {{"events", ev},
          {"layer_start", t.layer_start},
          {"layer_end", t.layer_end},
          {"makespan", t.makespan}};
}

nlohmann::json instance_json(const PipelineInstance& inst) {
  nlohmann::json layers = nlohmann::json::array();
  for (const LayerLoads& l : inst.layers) {
    nlohmann::json truth = nlohmann::json::array(), pred = nlohmann::json::array();
    for (auto [e, m] : l.truth) truth.push_back({e, m});
    for (auto [e, m] : l.predicted) pred.push_back({e, m});
    layers.push_back({{"truth", truth}, {"predicted", pred}});
  }
  nlohmann::json res = nlohmann::json::array();
  for (auto [l, e] : inst.resident) res.push_back({l, e});
  nlohmann::json groups = nlohmann::json::array();
  for (LayerGroup g : inst.groups) groups.push_back(static_cast<int>(g));
  return {{"layers", layers}, {"resident", res}, {"groups", groups}};
}

nlohmann::json params_json(const CostParams& p) {
  return {{"t_io", p.t_io}, {"t_g", p.t_g}, {"t_attn", p.t_attn},
          {"beta", p.beta}, {"startup", p.startup}, {"alpha", p.alpha}};
}

nlohmann::json plan_json(const LayerPlan& plan) {
  auto loads = [](const std::vector<ExpertLoad>& v) {
    nlohmann::json a = nlohmann::json::array();
    for (const ExpertLoad& e : v) a.push_back({e.expert, e.layer, e.tokens});
    return a;
  };
  return {{"split_index", plan.split_index},
          {"issued_prefetches", plan.issued_prefetches},
          {"prefetch_from_widened", plan.prefetch_from_widened},
          {"cpu_set", loads(plan.cpu_set)},
          {"ondemand_seq", loads(plan.ondemand_seq)},
          {"prefetch_seq", loads(plan.prefetch_seq)},
          {"t_g_at_split", plan.trace.t_g_at_split},
          {"t_c_at_split", plan.trace.t_c_at_split},
          {"t_gap", plan.trace.t_gap},
          {"f", plan.trace.f},
          {"f_int", plan.trace.f_int},
          {"xi", plan.trace.xi},
          {"widened_window", plan.trace.widened_window},
          {"all_gpu_fallback", plan.trace.all_gpu_fallback},
          {"sweep_gpu", plan.trace.sweep_gpu},
          {"sweep_cpu", plan.trace.sweep_cpu}};
}

struct LLaPorHandle {
  LLaPor model;
  uint64_t checksum = 0;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_spec_preset(const char* name, ref_spec* out) {
  return guarded([&] {
    ModelSpec m = spec_preset(name);
    *out = {m.num_layers, m.experts_per_layer, m.top_k, m.hidden_dim, m.expert_bytes,
            m.group_begin_middle, m.group_begin_output};
  });
}

int ref_desk_scale(const char* name, int layers, int experts, int hidden, ref_spec* out) {
  return guarded([&] {
    ModelSpec m = desk_scale(spec_preset(name), layers, experts, hidden);
    *out = {m.num_layers, m.experts_per_layer, m.top_k, m.hidden_dim, m.expert_bytes,
            m.group_begin_middle, m.group_begin_output};
  });
}

// generate_trace (workload.cpp:139-219) flattened: hidden [B*L*H], gate_weights
// [B*L*E], active [B*L*k]; each indexed (token*L + layer).
int ref_generate_trace(const ref_gen* gen, const ref_spec* spec, int batch, uint64_t seed,
                       double* hidden, double* gate_weights, int32_t* active) {
  return guarded([&] {
    Trace t = generate_trace(to_gen(*gen), to_spec(*spec), batch, seed);
    const int H = spec->hidden, E = spec->experts, K = spec->top_k;
    for (size_t i = 0; i < t.steps.size(); ++i) {
      const TraceStep& s = t.steps[i];
      if (hidden) std::memcpy(hidden + i * H, s.hidden.data(), sizeof(double) * H);
      if (gate_weights) std::memcpy(gate_weights + i * E, s.gate_weights.data(), sizeof(double) * E);
      if (active)
        for (int j = 0; j < K; ++j) active[i * K + j] = s.active_experts[j];
    }
  });
}

int ref_write_trace(const ref_gen* gen, const ref_spec* spec, int batch, uint64_t seed,
                    const char* path) {
  return guarded([&] { write_trace(generate_trace(to_gen(*gen), to_spec(*spec), batch, seed), path); });
}

// read_trace (workload.cpp:409-436) of a file written by anyone: batch, seed, checksum
// and the flattened routing (active [B*L*k]) as the reference parses them.
int ref_read_trace(const char* path, int* batch, uint64_t* seed, int32_t* active, int cap) {
  return guarded([&] {
    Trace t = read_trace(path);
    *batch = t.batch_size;
    *seed = t.seed;
    int n = 0;
    for (const TraceStep& s : t.steps)
      for (int e : s.active_experts)
        if (n < cap) active[n++] = e;
  });
}

int ref_topk(const double* w, int n, int k, int32_t* out, int* n_out) {
  return guarded([&] {
    std::vector<int> r = topk_indices(std::vector<double>(w, w + n), k);
    for (size_t i = 0; i < r.size(); ++i) out[i] = r[i];
    *n_out = static_cast<int>(r.size());
  });
}

// Hot table + residency from one trace (predictor.cpp:405-433); pairs out [2*n].
int ref_residency(const ref_gen* gen, const ref_spec* spec, int batch, uint64_t seed,
                  uint64_t budget_bytes, int32_t* pairs, int* n_out) {
  return guarded([&] {
    Trace t = generate_trace(to_gen(*gen), to_spec(*spec), batch, seed);
    HotExpertTable table = build_hot_table({t});
    auto res = plan_residency(table, budget_bytes, spec->expert_bytes);
    for (size_t i = 0; i < res.size(); ++i) {
      pairs[2 * i] = res[i].first;
      pairs[2 * i + 1] = res[i].second;
    }
    *n_out = static_cast<int>(res.size());
  });
}

// plan_layer (scheduler.cpp:402-413) on explicit LayerInputs. Output buffers sized
// by the caller: cpu/od <= n_cur, pf <= max(n_next, n_next2), sweeps <= n_cur+n_next.
int ref_plan_layer(int policy_kind, int fixed_c, const ref_load* cur, int n_cur,
                   const ref_load* nxt, int n_next, const ref_load* nxt2, int n_next2,
                   const ref_params* params, const ref_stats* stats, ref_plan_info* info,
                   ref_load* cpu, ref_load* od, ref_load* pf, int64_t* sweep_gpu,
                   int64_t* sweep_cpu) {
  return guarded([&] {
    LayerInputs in;
    in.e_cur = to_loads(cur, n_cur);
    in.e_next = to_loads(nxt, n_next);
    in.e_next2 = to_loads(nxt2, n_next2);
    in.params = to_params(*params);
    in.stats.r_hit = stats->r_hit;
    in.stats.r_miss = stats->r_miss;
    in.stats.window = stats->window;
    LayerPlan plan = plan_layer(in, to_policy(policy_kind, fixed_c));
    fill_info(plan, info);
    from_loads(plan.cpu_set, cpu);
    from_loads(plan.ondemand_seq, od);
    from_loads(plan.prefetch_seq, pf);
    for (size_t i = 0; i < plan.trace.sweep_gpu.size(); ++i) {
      if (sweep_gpu) sweep_gpu[i] = plan.trace.sweep_gpu[i];
      if (sweep_cpu) sweep_cpu[i] = plan.trace.sweep_cpu[i];
    }
  });
}

// simulate_policy (simulator.cpp:244-252). truth/pred are (layer, expert, tokens)
// triples, resident (layer, expert) pairs, groups per layer (nullable).
// plan_summary per layer: split_index, issued_prefetches, prefetch_from_widened, alpha.
int ref_simulate(int L, const int32_t* truth, int n_truth, const int32_t* pred, int n_pred,
                 const int32_t* resident, int n_res, const int32_t* groups, int policy_kind,
                 int fixed_c, const ref_params* params, const ref_sim_opts* opts,
                 ref_event* events, int max_events, int* n_events, int64_t* layer_start,
                 int64_t* layer_end, int64_t* makespan, int32_t* plan_summary) {
  return guarded([&] {
    PipelineInstance inst = make_instance(L, truth, n_truth, pred, n_pred, resident, n_res, groups);
    SimOptions so;
    so.cpu_slots = opts->cpu_slots;
    so.prefetch_slots = opts->prefetch_slots;
    so.initial_hit_rate = opts->initial_hit_rate;
    so.hit_window = opts->hit_window;
    SimResult r = simulate_policy(inst, to_policy(policy_kind, fixed_c), to_params(*params), so);
    if (static_cast<int>(r.timeline.events.size()) > max_events)
      throw std::runtime_error("ref_simulate: event buffer too small");
    for (size_t i = 0; i < r.timeline.events.size(); ++i) {
      const TimelineEvent& e = r.timeline.events[i];
      events[i] = {e.t_start, e.t_end, static_cast<int32_t>(e.resource),
                   static_cast<int32_t>(e.kind), e.layer, e.expert, e.tokens};
    }
    *n_events = static_cast<int>(r.timeline.events.size());
    for (int l = 0; l < L; ++l) {
      layer_start[l] = r.timeline.layer_start[l];
      layer_end[l] = r.timeline.layer_end[l];
    }
    *makespan = r.timeline.makespan;
    if (plan_summary)
      for (size_t l = 0; l < r.plans.size(); ++l) {
        plan_summary[4 * l + 0] = r.plans[l].split_index;
        plan_summary[4 * l + 1] = r.plans[l].issued_prefetches;
        plan_summary[4 * l + 2] = r.plans[l].prefetch_from_widened;
        plan_summary[4 * l + 3] = static_cast<int32_t>(r.plans[l].ondemand_seq.size());
      }
  });
}

// verify_timeline (simulator.cpp:323-394) over a caller-supplied event list; returns
// the number of violations in *n_viol.
int ref_verify_timeline(int L, const int32_t* truth, int n_truth, const int32_t* resident,
                        int n_res, const ref_params* params, const ref_event* events,
                        int n_events, int* n_viol) {
  return guarded([&] {
    PipelineInstance inst = make_instance(L, truth, n_truth, nullptr, 0, resident, n_res, nullptr);
    Timeline t;
    for (int i = 0; i < n_events; ++i) {
      const ref_event& e = events[i];
      t.events.push_back({e.t_start, e.t_end, static_cast<Resource>(e.resource),
                          static_cast<EventKind>(e.kind), e.layer, e.expert, e.tokens});
    }
    *n_viol = static_cast<int>(verify_timeline(t, inst, to_params(*params)).size());
  });
}

// export_timeline (simulator.cpp:428-436) of a caller-supplied event list.
int ref_export_timeline(const ref_event* events, int n_events, int64_t makespan, char* buf, int cap, int* needed) {
  return guarded([&] {
    Timeline t;
    t.makespan = makespan;
    for (int i = 0; i < n_events; ++i) {
      const ref_event& e = events[i];
      t.events.push_back({e.t_start, e.t_end, static_cast<Resource>(e.resource), static_cast<EventKind>(e.kind),
                          e.layer, e.expert, e.tokens});
    }
    const std::string s = export_timeline(t);
    *needed = static_cast<int>(s.size()) + 1;
    if (buf && cap > 0) {
      const size_t n = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
      std::memcpy(buf, s.data(), n);
      buf[n] = 0;
    }
  });
}

// Dumps the six golden scenarios (golden.cpp:61-234) with their hand-derived
// timelines, plus the reference PreSched plans/timeline on each instance.
int ref_dump_golden(const char* path) {
  return guarded([&] {
    nlohmann::json all = nlohmann::json::array();
    for (const std::string& id : golden_ids()) {
      const GoldenScenario& s = golden_scenario(id);
      SimResult got = simulate_policy(s.instance, s.policy, s.params, s.options);
      SimResult pre = simulate_policy(s.instance, SchedulerPolicy::parse("presched"), s.params, s.options);
      nlohmann::json plans = nlohmann::json::array(), pre_plans = nlohmann::json::array();
      for (const LayerPlan& p : got.plans) plans.push_back(plan_json(p));
      for (const LayerPlan& p : pre.plans) pre_plans.push_back(plan_json(p));
      all.push_back({{"id", s.id},
                     {"description", s.description},
                     {"policy", s.policy.name()},
                     {"params", params_json(s.params)},
                     {"options", {{"cpu_slots", s.options.cpu_slots},
                                  {"prefetch_slots", s.options.prefetch_slots},
                                  {"initial_hit_rate", s.options.initial_hit_rate},
                                  {"hit_window", s.options.hit_window}}},
                     {"instance", instance_json(s.instance)},
                     {"expected", timeline_json(s.expected)},
                     {"replayed", timeline_json(got.timeline)},
                     {"plans", plans},
                     {"presched_timeline", timeline_json(pre.timeline)},
                     {"presched_plans", pre_plans},
                     {"pass", replay_golden(id).pass}});
    }
    std::ofstream out(path);
    if (!out) throw std::runtime_error("ref_dump_golden: cannot open output");
    out << all.dump(1) << '\n';
  });
}

// LLaPor: train on `n_seeds` traces (make_llapor + train, predictor.cpp:467, 613)
// and write the LLPC v1 checkpoint (predictor.cpp:833).
int ref_train_llapor(const ref_gen* gen, const ref_spec* spec, int batch, const uint64_t* seeds,
                     int n_seeds, int epochs, int warmup, uint64_t train_seed, const char* path) {
  return guarded([&] {
    std::vector<Trace> traces;
    for (int i = 0; i < n_seeds; ++i)
      traces.push_back(generate_trace(to_gen(*gen), to_spec(*spec), batch, seeds[i]));
    TrainConfig cfg;
    cfg.epochs = epochs;
    cfg.warmup_epochs = warmup;
    cfg.seed = train_seed;
    LLaPor model = make_llapor(to_spec(*spec), cfg);
    train(model, traces);
    save_checkpoint(model, 0, path);
  });
}

void* ref_llapor_load(const char* path) {
  LLaPorHandle* h = nullptr;
  int rc = guarded([&] {
    auto p = std::make_unique<LLaPorHandle>();
    p->model = load_checkpoint(path, &p->checksum);
    h = p.release();
  });
  return rc == 0 ? h : nullptr;
}

void ref_llapor_free(void* h) { delete static_cast<LLaPorHandle*>(h); }

// pca_apply + forward + predict_topk for net `layer` on one token's layer-1
// features (experiment.cpp:85-98). reduced_out [P_eff], logits_out [E], topk_out [k].
int ref_llapor_predict(void* handle, int layer, const double* hidden_prev,
                       const int32_t* active_prev, int k_prev, const double* gate_prev, int k,
                       double* reduced_out, double* logits_out, int32_t* topk_out) {
  return guarded([&] {
    const LLaPor& m = static_cast<LLaPorHandle*>(handle)->model;
    const LLaPorNet& net = m.nets.at(layer);
    const int H = m.spec.hidden_dim, E = net.experts_per_layer;
    PredictorFeatures feat;
    feat.hidden_reduced = pca_apply(net.pca, std::vector<double>(hidden_prev, hidden_prev + H));
    feat.active_onehot.assign(E, 0.0);
    for (int j = 0; j < k_prev; ++j) feat.active_onehot.at(active_prev[j]) = 1.0;
    feat.gate_weights_prev.assign(gate_prev, gate_prev + E);
    ForwardResult r = forward(net, feat);
    std::vector<int> top = predict_topk(net, feat, k);
    if (reduced_out)
      std::memcpy(reduced_out, feat.hidden_reduced.data(), sizeof(double) * feat.hidden_reduced.size());
    if (logits_out) std::memcpy(logits_out, r.logits.data(), sizeof(double) * E);
    if (topk_out)
      for (size_t i = 0; i < top.size(); ++i) topk_out[i] = top[i];
  });
}

// predict_loads with the LLaPor predictor (experiment.cpp:104-112): loads_out [L*E].
int ref_llapor_predict_loads(void* handle, const ref_gen* gen, int batch, uint64_t seed, int k,
                             int32_t* loads_out) {
  return guarded([&] {
    const LLaPor& m = static_cast<LLaPorHandle*>(handle)->model;
    Trace t = generate_trace(to_gen(*gen), m.spec, batch, seed);
    PredictorChoice c;
    c.kind = PredictorChoice::Kind::LLaPorCkpt;
    c.checkpoint = "in-memory";
    PredictFn fn = make_predict_fn(c, &m, nullptr, k, 0);
    auto loads = predict_loads(t, fn);
    const int E = m.spec.experts_per_layer;
    std::fill(loads_out, loads_out + static_cast<size_t>(m.spec.num_layers) * E, 0);
    for (int l = 0; l < m.spec.num_layers; ++l)
      for (auto [e, c2] : loads[l]) loads_out[l * E + e] = c2;
  });
}

// CPU-baseline leg: the reference's own per-decode-step scheduling work on one trace —
// build_hot_table + plan_residency, predict_loads with the "perfect" PredictFn (the
// LLaPor inference leg is timed separately by ref_time_legs / ref_llapor_predict_batch),
// build_instance, simulate_policy(presched) — timed here in C++ so no ctypes overhead
// is counted.
// Returns mean seconds per call over `reps` in *sec_out.
int ref_time_schedule_pass(const ref_gen* gen, const ref_spec* spec, int batch, uint64_t seed,
                           uint64_t budget_bytes, const ref_params* params, int reps,
                           double* sec_out, int64_t* makespan_out) {
  return guarded([&] {
    Trace t = generate_trace(to_gen(*gen), to_spec(*spec), batch, seed);
    HotExpertTable table = build_hot_table({t});
    std::set<std::pair<int, int>> resident;
    for (auto key : plan_residency(table, budget_bytes, spec->expert_bytes)) resident.insert(key);
    PredictFn perfect = make_predict_fn(PredictorChoice::parse("perfect"), nullptr, nullptr,
                                        spec->top_k, 0);
    auto loads = predict_loads(t, perfect);
    PipelineInstance inst = build_instance(t, loads, resident);
    auto t0 = std::chrono::steady_clock::now();
    int64_t ms = 0;
    for (int r = 0; r < reps; ++r)
      ms = simulate_policy(inst, SchedulerPolicy::parse("presched"), to_params(*params)).timeline.makespan;
    *sec_out = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / reps;
    *makespan_out = ms;
  });
}

// LLaPor inference over a batch (bench.py --impl reference: the reference's
// pca_apply + forward + predict_topk, predictor.cpp:116-124, 166-247, 669-672, per
// token, tokens split over `threads` host threads; the model is read-only). hidden
// [B*H], active [B*k_prev], gate [B*E] of layer-1 features -> topk_out [B*k].
int ref_llapor_predict_batch(void* handle, int layer, int B, const double* hidden, const int32_t* active,
                             int k_prev, const double* gate, int k, int32_t* topk_out, int threads) {
  return guarded([&] {
    const LLaPor& m = static_cast<LLaPorHandle*>(handle)->model;
    const LLaPorNet& net = m.nets.at(layer);
    const int H = m.spec.hidden_dim, E = net.experts_per_layer;
    const int T = std::max(1, std::min(threads, B));
    std::vector<std::string> errs(T);
    auto work = [&](int w) {
      try {
        for (int t = B * w / T; t < B * (w + 1) / T; ++t) {
          PredictorFeatures feat;
          feat.hidden_reduced = pca_apply(net.pca, std::vector<double>(hidden + static_cast<size_t>(t) * H,
                                                                       hidden + static_cast<size_t>(t + 1) * H));
          feat.active_onehot.assign(E, 0.0);
          for (int j = 0; j < k_prev; ++j) feat.active_onehot.at(active[t * k_prev + j]) = 1.0;
          feat.gate_weights_prev.assign(gate + static_cast<size_t>(t) * E, gate + static_cast<size_t>(t + 1) * E);
          std::vector<int> top = predict_topk(net, feat, k);
          for (int j = 0; j < k; ++j) topk_out[t * k + j] = top.at(j);
        }
      } catch (const std::exception& ex) {
        errs[w] = ex.what();
      }
    };
    std::vector<std::thread> th;
    for (int w = 1; w < T; ++w) th.emplace_back(work, w);
    work(0);
    for (auto& x : th) x.join();
    for (auto& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
  });
}

// Per-leg 1-core timing of the reference's hot-path functions (SURVEY.md §8d CPU
// baseline) on one reference trace of `batch` tokens. Each leg repeats until
// `min_seconds` elapsed; us_out[i] = mean microseconds per call, calls_out[i] = calls.
//   0 topk_indices          (workload.cpp:110-119) on one (token, layer)'s gate weights
//   1 aggregate_layer_loads (workload.cpp:283-288) for one layer of the batch
//   2 pca_apply+forward+predict_topk, input-group net (predictor.cpp:116-124, 344-352, 669-672)
//   3 the same, middle-group net (the wider PCA)
//   4 build_hot_table + plan_residency (predictor.cpp:405-433)
//   5 schedule_layer (scheduler.cpp:54-213) on one layer's LayerInputs (E_cur, E_next, E_next2)
//   6 simulate_policy(presched) over all layers (simulator.cpp:61-242), per step
//   7 generate_trace (RNG + router, workload.cpp:139-219), per token
// Legs 2-3 need an LLaPor handle (nullable: reported as 0).
int ref_time_legs(const ref_gen* gen, const ref_spec* spec, int batch, uint64_t seed, void* llapor,
                  uint64_t budget_bytes, const ref_params* params, double min_seconds, double* us_out,
                  int64_t* calls_out) {
  return guarded([&] {
    using clk = std::chrono::steady_clock;
    const ModelSpec sp = to_spec(*spec);
    Trace t = generate_trace(to_gen(*gen), sp, batch, seed);
    const int L = sp.num_layers, K = sp.top_k, E = sp.experts_per_layer;
    volatile int64_t sink = 0;
    auto timed = [&](int leg, const std::function<void(int64_t)>& body) {
      int64_t n = 0;
      const auto t0 = clk::now();
      double el = 0;
      do {
        body(n++);
        el = std::chrono::duration<double>(clk::now() - t0).count();
      } while (el < min_seconds);
      us_out[leg] = el * 1e6 / static_cast<double>(n);
      calls_out[leg] = n;
    };
    const size_t S = t.steps.size();
    timed(0, [&](int64_t i) { sink = sink + topk_indices(t.steps[i % S].gate_weights, K).size(); });
    timed(1, [&](int64_t i) { sink = sink + aggregate_layer_loads(t, static_cast<int>(i % L)).size(); });
    for (int leg = 2; leg <= 3; ++leg) {
      us_out[leg] = 0;
      calls_out[leg] = 0;
      if (!llapor) continue;
      const LLaPor& m = static_cast<LLaPorHandle*>(llapor)->model;
      const int l = leg == 2 ? 1 : sp.group_begin_middle;  // input group / middle group target
      if (l < 1 || l >= static_cast<int>(m.nets.size()) || m.nets[l].blocks.empty()) continue;
      const LLaPorNet& net = m.nets[l];
      timed(leg, [&](int64_t i) {
        const TraceStep& st = t.steps[static_cast<size_t>(i % batch) * L + (l - 1)];
        PredictorFeatures feat;
        feat.hidden_reduced = pca_apply(net.pca, st.hidden);
        feat.active_onehot.assign(E, 0.0);
        for (int e : st.active_experts) feat.active_onehot.at(e) = 1.0;
        feat.gate_weights_prev = st.gate_weights;
        sink = sink + predict_topk(net, feat, K).size();
      });
    }
    std::set<std::pair<int, int>> resident;
    timed(4, [&](int64_t) {
      HotExpertTable table = build_hot_table({t});
      auto res = plan_residency(table, budget_bytes, spec->expert_bytes);
      sink = sink + res.size();
      if (resident.empty())
        for (auto key : res) resident.insert(key);
    });
    PredictFn perfect = make_predict_fn(PredictorChoice::parse("perfect"), nullptr, nullptr, K, 0);
    PipelineInstance inst = build_instance(t, predict_loads(t, perfect), resident);
    auto sorted = [&](const std::map<int, int>& m, int layer) {
      std::vector<ExpertLoad> v;
      for (auto [e, c] : m)
        if (!resident.count({layer, e})) v.push_back({e, layer, c, ExpertLocation::Host});
      std::sort(v.begin(), v.end(), [](const ExpertLoad& a, const ExpertLoad& b) {
        return a.tokens != b.tokens ? a.tokens < b.tokens : a.expert < b.expert;
      });
      return v;
    };
    std::vector<LayerInputs> ins(L);
    for (int l = 0; l < L; ++l) {
      ins[l].e_cur = sorted(inst.layers[l].truth, l);
      if (l + 1 < L) ins[l].e_next = sorted(inst.layers[l + 1].predicted, l + 1);
      if (l + 2 < L) ins[l].e_next2 = sorted(inst.layers[l + 2].predicted, l + 2);
      ins[l].params = to_params(*params);
    }
    timed(5, [&](int64_t i) { sink = sink + schedule_layer(ins[i % L]).split_index; });
    timed(6, [&](int64_t) {
      sink = sink + simulate_policy(inst, SchedulerPolicy::parse("presched"), to_params(*params)).timeline.makespan;
    });
    timed(7, [&](int64_t i) { sink = sink + generate_trace(to_gen(*gen), sp, 1, seed + 1 + i).steps.size(); });
    (void)sink;
  });
}

// Router inputs of generate_trace (workload.cpp:139-219) without the routing, for the
// f64 router restatement (oracle.c or_route_batch) in bench.py's reference arm: the
// gate matrices G [L*E*D] (the first L*E*D draws of the seeded engine), the
// kappa-follow flags [batch*L] and zipf_s per layer [L]. The engine's draw sequence does
// not depend on the routing (one uniform per layer >= 1, drawn before the follow test;
// D normals per token and per layer transition), so it is replayed here with the same
// libstdc++ distributions; tests/test_oracle.py checks that or_route_batch on these
// inputs reproduces generate_trace's gate weights bit for bit.
int ref_router_inputs(const ref_gen* gen, const ref_spec* spec, int batch, uint64_t seed, double* gate,
                      uint8_t* follow, double* zipf) {
  return guarded([&] {
    const TraceGenConfig cfg = to_gen(*gen);
    const ModelSpec sp = to_spec(*spec);
    cfg.validate();
    sp.validate();
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    std::uniform_real_distribution<double> unif(0.0, 1.0);
    const int L = sp.num_layers, E = sp.experts_per_layer, D = sp.hidden_dim;
    const double wscale = 1.0 / std::sqrt(static_cast<double>(D));
    for (size_t i = 0; i < static_cast<size_t>(L) * E * D; ++i) gate[i] = gauss(rng) * wscale;
    for (int l = 0; l < L; ++l) zipf[l] = cfg.for_group(sp.group_of(l)).zipf_s;
    for (int tok = 0; tok < batch; ++tok) {
      for (int d = 0; d < D; ++d) (void)gauss(rng);
      for (int l = 0; l < L; ++l) {
        const GroupGenParams& gp = cfg.for_group(sp.group_of(l));
        follow[static_cast<size_t>(tok) * L + l] = l > 0 && unif(rng) < gp.kappa;
        if (l + 1 < L)
          for (int d = 0; d < D; ++d) (void)gauss(rng);
      }
    }
  });
}

// compute_metrics (simulator.cpp:396-426) on a caller-supplied Timeline. out_scalars:
// makespan, decode_latency, throughput, io_busy_fraction, gpu_idle_fraction.
int ref_compute_metrics(const ref_event* events, int n_events, const int64_t* layer_start,
                        const int64_t* layer_end, int L, int64_t makespan, int output_tokens,
                        double* out_scalars, int64_t* per_layer, int64_t* gap) {
  return guarded([&] {
    Timeline t;
    for (int i = 0; i < n_events; ++i)
      t.events.push_back({events[i].t_start, events[i].t_end, static_cast<Resource>(events[i].resource),
                          static_cast<EventKind>(events[i].kind), events[i].layer, events[i].expert,
                          events[i].tokens});
    t.layer_start.assign(layer_start, layer_start + L);
    t.layer_end.assign(layer_end, layer_end + L);
    t.makespan = makespan;
    Metrics m = compute_metrics(t, output_tokens);
    out_scalars[0] = static_cast<double>(m.makespan);
    out_scalars[1] = static_cast<double>(m.decode_latency);
    out_scalars[2] = m.throughput_tokens_per_s;
    out_scalars[3] = m.io_busy_fraction;
    out_scalars[4] = m.gpu_idle_fraction;
    for (int l = 0; l < L; ++l) {
      per_layer[l] = m.per_layer_latency[l];
      gap[l] = m.cpu_gpu_gap[l];
    }
  });
}

// fine_tune (predictor.cpp:654-663) of a loaded model's net `layer` on explicit samples
// built the way build_samples does (predictor.cpp:596-613), then save_checkpoint.
int ref_llapor_fine_tune(void* handle, int layer, int n, const double* hidden_prev, const int32_t* active_prev,
                         int k_prev, const double* gate_prev, const int32_t* active, int k, int steps, double lr) {
  return guarded([&] {
    LLaPor& m = static_cast<LLaPorHandle*>(handle)->model;
    LLaPorNet& net = m.nets.at(layer);
    const int H = m.spec.hidden_dim, E = net.experts_per_layer;
    std::vector<Sample> samples;
    for (int t = 0; t < n; ++t) {
      Sample s;
      s.features.hidden_reduced = pca_apply(net.pca, std::vector<double>(hidden_prev + static_cast<size_t>(t) * H,
                                                                         hidden_prev + static_cast<size_t>(t + 1) * H));
      s.features.active_onehot.assign(E, 0.0);
      for (int j = 0; j < k_prev; ++j) s.features.active_onehot.at(active_prev[t * k_prev + j]) = 1.0;
      s.features.gate_weights_prev.assign(gate_prev + static_cast<size_t>(t) * E,
                                          gate_prev + static_cast<size_t>(t + 1) * E);
      s.labels.assign(E, 0.0);
      for (int j = 0; j < k; ++j) s.labels.at(active[t * k + j]) = 1.0;
      samples.push_back(std::move(s));
    }
    fine_tune(net, samples, steps, lr, m.cfg);
  });
}

int ref_llapor_save(void* handle, const char* path) {
  return guarded([&] {
    const LLaPorHandle* h = static_cast<LLaPorHandle*>(handle);
    save_checkpoint(h->model, h->checksum, path);
  });
}

}  // extern "C"
