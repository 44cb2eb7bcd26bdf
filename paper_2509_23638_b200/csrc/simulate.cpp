// AsyncIO model-clock pipeline: the integer-tick executor semantics the real loader
// (engine.cpp) reproduces on the GPU, used for parity mode and for checking measured
// timelines. Rules R1-R8 of SURVEY.md §8a (simulator.cpp:61-242), verify_timeline
// (simulator.cpp:323-394) and compute_metrics (simulator.cpp:396-426).
//
// Dense (layer, expert) tables replace the reference's std::map/std::set state; the
// event insertion order is kept identical so the final stable sort by (resource,
// t_start, t_end) yields the same timeline (golden replays in tests/test_host_parity.py).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "common.hpp"

namespace ps {
void plan_layer(const ps_layer_inputs& in, ps_policy pol, ps_layer_plan& out);

namespace {

struct Pending {
  int64_t start, end;
  int target_layer, expert, tokens;
  bool critical;
  int issue_group;
};

struct Ev {
  int64_t t_start, t_end;
  int resource, kind, layer, expert, tokens;
};

int group_at(const ps_pipeline_instance& inst, int l) {
  return inst.groups ? inst.groups[l] : PS_GROUP_MIDDLE;
}

void hit_record(ps_hit_stats& s, bool hit) {
  double w = 1.0 / s.window;
  s.r_hit = (1.0 - w) * s.r_hit + (hit ? w : 0.0);
  s.r_miss = 1.0 - s.r_hit;
}

// Host experts of one layer with m >= 1, not excluded, ordered (tokens, expert)
// (simulator.cpp:45-57).
void host_loads(const int32_t* counts, int E, int layer, const std::vector<char>& exclude,
                std::vector<ps_expert_load>& out) {
  out.clear();
  for (int e = 0; e < E; ++e)
    if (counts[e] >= 1 && !exclude[e]) out.push_back({e, layer, counts[e], PS_LOC_HOST});
  std::sort(out.begin(), out.end(), [](const ps_expert_load& a, const ps_expert_load& b) {
    if (a.tokens != b.tokens) return a.tokens < b.tokens;
    return a.expert < b.expert;
  });
}

}  // namespace

void simulate(const ps_pipeline_instance& inst, ps_policy policy, ps_plan_fn plan_fn, void* user,
              const ps_cost_params& params, const ps_sim_options& opt, ps_timeline& out) {
  if (params.t_io < 0 || params.t_g < 0 || params.t_attn < 0 || params.beta < 0 ||
      params.startup < 0 || params.alpha < 0)
    fail(PS_EINVAL, "CostParams: all parameters must be >= 0");
  if (!(params.t_g < params.t_io)) fail(PS_EINVAL, "CostParams: requires t_g < t_io");
  const int L = inst.num_layers, E = inst.experts;
  require(L >= 0 && E >= 1 && inst.truth && inst.predicted, "PipelineInstance: bad shape");
  auto truth = [&](int l) { return inst.truth + static_cast<size_t>(l) * E; };
  auto pred = [&](int l) { return inst.predicted + static_cast<size_t>(l) * E; };
  auto resident = [&](int l, int e) {
    return inst.resident && inst.resident[static_cast<size_t>(l) * E + e] != 0;
  };

  std::vector<Ev> events;
  int64_t io_free = 0, io_free_base = 0;
  std::vector<Pending> pending;
  std::vector<int64_t> ready(static_cast<size_t>(L) * E, -1);  // prefetched -> ready tick
  std::vector<int> slot_use(static_cast<size_t>(L) + 3, 0);   // per target layer
  ps_hit_stats stats[3];
  for (auto& h : stats) h = {opt.initial_hit_rate, 1.0 - opt.initial_hit_rate, opt.hit_window};

  std::vector<ps_expert_load> e_cur, e_next, e_next2;
  std::vector<char> excl(E);
  std::vector<ps_expert_load> cpu_buf(E), od_buf(E), pf_buf(E);
  std::vector<int64_t> sweep_g(2 * E), sweep_c(2 * E);

  int64_t prev_end = 0;
  for (int l = 0; l < L; ++l) {
    const int64_t attn_start = prev_end, t0 = attn_start + params.t_attn;
    events.push_back({attn_start, t0, PS_RES_GPU, PS_EV_ATTENTION, l, -1, 0});
    out.layer_start[l] = attn_start;

    // R2: started prefetches commit (non-interruptible), the rest are cancelled.
    for (const Pending& p : pending) {
      if (p.start < t0) {
        events.push_back({p.start, p.end, PS_RES_IO, PS_EV_PREFETCH, p.target_layer, p.expert, p.tokens});
        if (p.target_layer < L) ready[static_cast<size_t>(p.target_layer) * E + p.expert] = p.end;
        io_free_base = std::max(io_free_base, p.end);
        if (p.critical) {
          bool hit = p.target_layer < L && truth(p.target_layer)[p.expert] > 0;
          hit_record(stats[p.issue_group], hit);
        }
      } else {
        slot_use[p.target_layer]--;
      }
    }
    pending.clear();
    io_free = io_free_base;
    // R3: slots of target layers <= l are released.
    for (int t = 0; t <= l && t < static_cast<int>(slot_use.size()); ++t) slot_use[t] = 0;

    // R4: exclude resident / prefetched; alpha = backlog beyond t0.
    auto build = [&](int layer, const int32_t* counts, std::vector<ps_expert_load>& dst) {
      for (int e = 0; e < E; ++e)
        excl[e] = resident(layer, e) || ready[static_cast<size_t>(layer) * E + e] >= 0;
      host_loads(counts, E, layer, excl, dst);
    };
    build(l, truth(l), e_cur);
    e_next.clear();
    e_next2.clear();
    if (l + 1 < L) build(l + 1, pred(l + 1), e_next);
    if (l + 2 < L) build(l + 2, pred(l + 2), e_next2);

    ps_layer_inputs in{};
    in.e_cur = e_cur.data();
    in.n_cur = static_cast<int32_t>(e_cur.size());
    in.e_next = e_next.data();
    in.n_next = static_cast<int32_t>(e_next.size());
    in.e_next2 = e_next2.data();
    in.n_next2 = static_cast<int32_t>(e_next2.size());
    in.params = params;
    in.params.alpha = std::max<int64_t>(0, io_free - t0);
    in.stats = stats[group_at(inst, l)];

    ps_layer_plan plan{};
    plan.cpu_set = cpu_buf.data();
    plan.ondemand_seq = od_buf.data();
    plan.prefetch_seq = pf_buf.data();
    plan.trace.sweep_gpu = sweep_g.data();
    plan.trace.sweep_cpu = sweep_c.data();
    if (plan_fn) {
      ps_status st = plan_fn(user, &in, l, &plan);
      if (st != PS_OK) fail(st, "plan_fn failed at layer " + std::to_string(l));
    } else {
      plan_layer(in, policy, plan);
    }
    if (out.plan_summary) {
      out.plan_summary[4 * l + 0] = plan.split_index;
      out.plan_summary[4 * l + 1] = plan.issued_prefetches;
      out.plan_summary[4 * l + 2] = plan.prefetch_from_widened;
      out.plan_summary[4 * l + 3] = plan.n_ondemand;
    }

    // R5: CPU experts from t0 on the earliest-free slot.
    std::vector<int64_t> cpu_free(std::max(1, opt.cpu_slots), t0);
    for (int i = 0; i < plan.n_cpu; ++i) {
      const ps_expert_load& e = plan.cpu_set[i];
      auto slot = std::min_element(cpu_free.begin(), cpu_free.end());
      const int64_t dur = static_cast<int64_t>(std::floor(params.beta * e.tokens + 0.5)) + params.startup;
      events.push_back({*slot, *slot + dur, PS_RES_CPU, PS_EV_CPU_EXPERT, l, e.expert, e.tokens});
      *slot += dur;
    }

    // R6: resident / prefetched experts compute when ready (ready, expert) order.
    struct Avail {
      int64_t ready;
      int expert, tokens;
    };
    std::vector<Avail> avail;
    for (int e = 0; e < E; ++e) {
      const int m = truth(l)[e];
      if (m == 0) continue;
      if (resident(l, e)) avail.push_back({t0, e, m});
      else if (int64_t r = ready[static_cast<size_t>(l) * E + e]; r >= 0) avail.push_back({std::max(t0, r), e, m});
    }
    std::sort(avail.begin(), avail.end(), [](const Avail& a, const Avail& b) {
      if (a.ready != b.ready) return a.ready < b.ready;
      return a.expert < b.expert;
    });
    int64_t gpu_free = t0;
    size_t ai = 0;
    auto run_avail_until = [&](int64_t bound) {
      while (ai < avail.size() && avail[ai].ready <= bound) {
        const int64_t s = std::max(gpu_free, avail[ai].ready);
        events.push_back({s, s + params.t_g, PS_RES_GPU, PS_EV_GPU_EXPERT, l, avail[ai].expert, avail[ai].tokens});
        gpu_free = s + params.t_g;
        ++ai;
      }
    };

    // R7: on-demand loads through two alternating buffer slots.
    std::vector<int64_t> compute_end(plan.n_ondemand, 0);
    for (int j = 0; j < plan.n_ondemand; ++j) {
      const ps_expert_load& e = plan.ondemand_seq[j];
      const int64_t slot_free = j >= 2 ? compute_end[j - 2] : 0;
      const int64_t start = std::max({io_free, t0, slot_free});
      const int64_t end = start + params.t_io;
      io_free = end;
      events.push_back({start, end, PS_RES_IO, PS_EV_LOAD, l, e.expert, e.tokens});
      run_avail_until(end);
      const int64_t cs = std::max(gpu_free, end), ce = cs + params.t_g;
      events.push_back({cs, ce, PS_RES_GPU, PS_EV_GPU_EXPERT, l, e.expert, e.tokens});
      gpu_free = ce;
      compute_end[j] = ce;
    }
    run_avail_until(std::numeric_limits<int64_t>::max());

    int64_t layer_end = std::max(t0, gpu_free);
    for (int64_t c : cpu_free) layer_end = std::max(layer_end, c);
    out.layer_end[l] = layer_end;

    // R8: prefetches queue behind the loads; resolved at the next layer.
    io_free_base = io_free;
    if (plan.n_prefetch > 0) {
      const int target = plan.prefetch_from_widened ? l + 2 : l + 1;
      if (target >= static_cast<int>(slot_use.size())) slot_use.resize(target + 1, 0);
      int& used = slot_use[target];
      if (used + plan.n_prefetch > opt.prefetch_slots)
        fail(PS_ERUNTIME, "simulate_pipeline: prefetch buffer overflow for layer " + std::to_string(target));
      for (int j = 0; j < plan.n_prefetch; ++j) {
        const ps_expert_load& e = plan.prefetch_seq[j];
        Pending p;
        p.start = std::max(io_free, t0);
        p.end = p.start + params.t_io;
        p.target_layer = target;
        p.expert = e.expert;
        p.tokens = e.tokens;
        p.critical = j + 1 == plan.n_prefetch;
        p.issue_group = group_at(inst, l);
        io_free = p.end;
        pending.push_back(p);
        ++used;
      }
    }
    prev_end = layer_end;
  }

  std::stable_sort(events.begin(), events.end(), [](const Ev& a, const Ev& b) {
    if (a.resource != b.resource) return a.resource < b.resource;
    if (a.t_start != b.t_start) return a.t_start < b.t_start;
    return a.t_end < b.t_end;
  });
  if (static_cast<int>(events.size()) > out.cap_events)
    fail(PS_ERANGE, "simulate_pipeline: event buffer too small (" + std::to_string(events.size()) + ")");
  out.makespan = 0;
  for (size_t i = 0; i < events.size(); ++i) {
    const Ev& e = events[i];
    out.events[i] = {e.t_start, e.t_end, e.resource, e.kind, e.layer, e.expert, e.tokens};
    out.makespan = std::max(out.makespan, e.t_end);
  }
  out.n_events = static_cast<int32_t>(events.size());
}

// measured = true: a timeline recorded on the GPU (engine.cpp) — transfer durations
// are measured, so the "atomic t_io interval" rule is replaced by "a transfer is one
// interval" (it cannot be split: one cudaMemcpyAsync per expert), all other
// invariants are the reference's.
std::vector<std::string> verify(const ps_timeline_event* ev, int n, const ps_pipeline_instance& inst,
                                const ps_cost_params& params, bool measured = false) {
  std::vector<std::string> v;
  const int L = inst.num_layers, E = inst.experts;
  auto truth = [&](int l, int e) { return inst.truth[static_cast<size_t>(l) * E + e]; };
  auto in_range = [&](int l, int e) { return l >= 0 && l < L && e >= 0 && e < E; };

  std::vector<const ps_timeline_event*> io;
  for (int i = 0; i < n; ++i)
    if (ev[i].resource == PS_RES_IO) io.push_back(&ev[i]);
  std::stable_sort(io.begin(), io.end(), [](auto* a, auto* b) { return a->t_start < b->t_start; });
  for (size_t i = 1; i < io.size(); ++i)
    if (io[i]->t_start < io[i - 1]->t_end)
      v.push_back("serial-io: overlapping transfers at t=" + std::to_string(io[i]->t_start));
  for (auto* e : io)
    if (measured ? e->t_end < e->t_start : e->t_end - e->t_start != params.t_io)
      v.push_back("non-interruptible: transfer of expert " + std::to_string(e->expert) +
                  " is not an atomic t_io interval");

  // Conservation: each activated (layer, expert) computed exactly once.
  std::vector<int> computed(static_cast<size_t>(L) * E, 0);
  std::vector<std::pair<int, int>> ghosts;  // computed but not activated, one entry per key
  for (int i = 0; i < n; ++i) {
    const auto& e = ev[i];
    if (e.kind != PS_EV_GPU_EXPERT && e.kind != PS_EV_CPU_EXPERT) continue;
    if (!in_range(e.layer, e.expert) || truth(e.layer, e.expert) == 0) {
      std::pair<int, int> key{e.layer, e.expert};
      if (std::find(ghosts.begin(), ghosts.end(), key) == ghosts.end()) ghosts.push_back(key);
      continue;
    }
    computed[static_cast<size_t>(e.layer) * E + e.expert]++;
  }
  for (int l = 0; l < L; ++l)
    for (int e = 0; e < E; ++e)
      if (truth(l, e) > 0 && computed[static_cast<size_t>(l) * E + e] != 1)
        v.push_back("conservation: (" + std::to_string(l) + "," + std::to_string(e) + ") computed " +
                    std::to_string(computed[static_cast<size_t>(l) * E + e]) + " times");
  std::sort(ghosts.begin(), ghosts.end());
  for (auto [l, e] : ghosts)
    v.push_back("conservation: non-activated (" + std::to_string(l) + "," + std::to_string(e) + ") computed");

  // Causality: non-resident GPU compute needs a completed transfer first.
  for (int i = 0; i < n; ++i) {
    const auto& e = ev[i];
    if (e.kind != PS_EV_GPU_EXPERT) continue;
    if (inst.resident && in_range(e.layer, e.expert) &&
        inst.resident[static_cast<size_t>(e.layer) * E + e.expert])
      continue;
    bool ok = false;
    for (auto* t : io)
      if (t->layer == e.layer && t->expert == e.expert && t->t_end <= e.t_start) ok = true;
    if (!ok)
      v.push_back("causality: gpu compute of (" + std::to_string(e.layer) + "," +
                  std::to_string(e.expert) + ") without completed transfer");
  }

  // Dual on-demand buffer: load j+2 must not start before compute of load j ends.
  for (int l = 0; l < L; ++l) {
    std::vector<const ps_timeline_event*> loads;
    for (auto* t : io)
      if (t->kind == PS_EV_LOAD && t->layer == l) loads.push_back(t);
    for (size_t j = 2; j < loads.size(); ++j) {
      int64_t prev_end = 0;
      for (int i = 0; i < n; ++i)
        if (ev[i].kind == PS_EV_GPU_EXPERT && ev[i].layer == l && ev[i].expert == loads[j - 2]->expert)
          prev_end = ev[i].t_end;
      if (loads[j]->t_start < prev_end)
        v.push_back("buffer: load of expert " + std::to_string(loads[j]->expert) +
                    " overwrites a slot before its compute finished");
    }
  }
  for (int i = 0; i < n; ++i)
    if (ev[i].t_start > ev[i].t_end) v.push_back("event with t_start > t_end");
  return v;
}

}  // namespace ps

using namespace ps;

extern "C" {

ps_status ps_simulate_pipeline(const ps_pipeline_instance* inst, ps_policy policy, ps_plan_fn plan_fn,
                               void* user, const ps_cost_params* params, const ps_sim_options* opts,
                               ps_timeline* out) {
  return guarded([&] {
    ps_sim_options o = opts ? *opts : ps_sim_options{1, 8, 1.0, 32};
    if (!plan_fn && policy.kind == PS_POLICY_ORACLE)
      fail(PS_EINVAL, "oracle policy requires the pipeline enumerator");
    simulate(*inst, policy, plan_fn, user, *params, o, *out);
  });
}

ps_status ps_verify_timeline(const ps_timeline_event* events, int n_events, const ps_pipeline_instance* inst,
                             const ps_cost_params* params, int* n_violations, char* msg_buf, int msg_cap) {
  return ps_verify_timeline_ex(events, n_events, inst, params, 0, n_violations, msg_buf, msg_cap);
}

ps_status ps_verify_timeline_ex(const ps_timeline_event* events, int n_events, const ps_pipeline_instance* inst,
                                const ps_cost_params* params, int measured, int* n_violations, char* msg_buf,
                                int msg_cap) {
  return guarded([&] {
    std::vector<std::string> v = verify(events, n_events, *inst, *params, measured != 0);
    *n_violations = static_cast<int>(v.size());
    if (msg_buf && msg_cap > 0) {
      std::string all;
      for (const auto& s : v) all += s + "\n";
      size_t len = std::min<size_t>(all.size(), static_cast<size_t>(msg_cap - 1));
      std::memcpy(msg_buf, all.data(), len);
      msg_buf[len] = 0;
    }
  });
}

ps_status ps_export_timeline(const ps_timeline_event* events, int n, int64_t makespan, char* buf, int cap,
                             int* needed) {
  return guarded([&] {
    require(n >= 0 && (n == 0 || events) && needed, "ps_export_timeline: bad arguments");
    static const char* kRes[] = {"gpu", "cpu", "io"};
    static const char* kKind[] = {"attention", "gpu_expert", "cpu_expert", "load", "prefetch", "idle"};
    std::string out = "# tick_unit=us makespan=" + std::to_string(makespan) + "\n";
    for (int i = 0; i < n; ++i) {
      const ps_timeline_event& e = events[i];
      const char* r = e.resource >= 0 && e.resource < 3 ? kRes[e.resource] : "?";
      const char* k = e.kind >= 0 && e.kind < 6 ? kKind[e.kind] : "?";
      out += std::to_string(e.t_start) + ' ' + std::to_string(e.t_end) + ' ' + r + ' ' + k + ' ' +
             std::to_string(e.layer) + ' ' + std::to_string(e.expert) + ' ' + std::to_string(e.tokens) + '\n';
    }
    *needed = static_cast<int>(out.size()) + 1;
    if (buf && cap > 0) {
      const size_t m = std::min<size_t>(out.size(), static_cast<size_t>(cap - 1));
      std::memcpy(buf, out.data(), m);
      buf[m] = 0;
    }
  });
}

ps_status ps_compute_metrics(const ps_timeline_event* events, int n, const int64_t* layer_start,
                             const int64_t* layer_end, int L, int64_t makespan, int output_tokens, ps_metrics* m,
                             int64_t* per_layer_latency, int64_t* cpu_gpu_gap) {
  return guarded([&] {
    require(n >= 0 && L >= 0 && m && (n == 0 || events) && (L == 0 || (layer_start && layer_end)),
            "compute_metrics: null argument");
    // The reference indexes per-layer arrays with event.layer (simulator.cpp:410-414);
    // an event outside [0, L) is an index error here instead of undefined behaviour.
    for (int i = 0; i < n; ++i)
      if (events[i].layer < 0 || events[i].layer >= L)
        fail(PS_ERANGE, "compute_metrics: event layer " + std::to_string(events[i].layer) + " out of range");
    *m = ps_metrics{};
    m->makespan = m->decode_latency = makespan;
    if (makespan > 0) m->throughput_tokens_per_s = output_tokens * 1e6 / static_cast<double>(makespan);
    std::vector<int64_t> cpu_fin(L, -1), gpu_fin(L, -1), attn_end(L, 0);
    int64_t io_busy = 0, gpu_busy = 0;
    for (int i = 0; i < n; ++i) {
      const auto& e = events[i];
      if (e.resource == PS_RES_IO) io_busy += e.t_end - e.t_start;
      if (e.resource == PS_RES_GPU) gpu_busy += e.t_end - e.t_start;
      if (e.kind == PS_EV_ATTENTION) attn_end[e.layer] = e.t_end;
      if (e.kind == PS_EV_CPU_EXPERT) cpu_fin[e.layer] = std::max(cpu_fin[e.layer], e.t_end);
      if (e.kind == PS_EV_GPU_EXPERT) gpu_fin[e.layer] = std::max(gpu_fin[e.layer], e.t_end);
    }
    for (int l = 0; l < L; ++l) {
      if (per_layer_latency) per_layer_latency[l] = layer_end[l] - layer_start[l];
      int64_t fc = cpu_fin[l] >= 0 ? cpu_fin[l] : attn_end[l];
      int64_t fg = gpu_fin[l] >= 0 ? gpu_fin[l] : attn_end[l];
      if (cpu_gpu_gap) cpu_gpu_gap[l] = fc > fg ? fc - fg : fg - fc;
    }
    if (makespan > 0) {
      m->io_busy_fraction = static_cast<double>(io_busy) / makespan;
      m->gpu_idle_fraction = 1.0 - static_cast<double>(gpu_busy) / makespan;
    }
  });
}

}  // extern "C"
