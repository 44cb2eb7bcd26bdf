// Cost model (Eq.3-7) and PreSched plan — host, pure, reentrant.
//
// Same decisions as the reference's schedule_layer / greedy / on-demand / fixed
// policies (scheduler.cpp:54-282, cost_model.cpp:11-106) but restructured around
// prefix sums: the reference re-sums the CPU prefix for every merged element
// (O((n+n')^2), 551 us at n=n'=256); here each list is scanned once after one stable
// sort, O((n+n') log(n+n')). All tick arithmetic is int64 and every double is formed
// with the reference's operand order (compiled with -ffp-contract=off), so plans,
// sweeps, f and xi are bit-identical (tests/test_host_parity.py: test_presched_product_vs_reference_random_large, test_cost_model_kats).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <set>
#include <string>
#include <vector>

#include "common.hpp"

namespace ps {
namespace {

inline int64_t ticks(double x) { return static_cast<int64_t>(std::floor(x + 0.5)); }

inline int64_t cpu_cost_of(int tokens, const ps_cost_params& p) {
  return ticks(p.beta * tokens) + p.startup;
}

void validate_params(const ps_cost_params& p) {
  if (p.t_io < 0 || p.t_g < 0 || p.t_attn < 0 || p.beta < 0 || p.startup < 0 || p.alpha < 0)
    fail(PS_EINVAL, "CostParams: all parameters must be >= 0");
  if (!(p.t_g < p.t_io)) fail(PS_EINVAL, "CostParams: requires t_g < t_io");
}

void validate_stats(const ps_hit_stats& s) {
  if (s.r_hit < 0 || s.r_hit > 1 || s.r_miss < 0 || s.r_miss > 1)
    fail(PS_EINVAL, "HitStats: rates must be in [0,1]");
  if (std::abs(s.r_hit + s.r_miss - 1.0) > 1e-9)
    fail(PS_EINVAL, "HitStats: r_hit + r_miss must equal 1");
  if (s.window < 1) fail(PS_EINVAL, "HitStats: window must be >= 1");
}

void validate_inputs(const ps_layer_inputs& in) {
  validate_params(in.params);
  validate_stats(in.stats);
  const ps_expert_load* lists[3] = {in.e_cur, in.e_next, in.e_next2};
  const int ns[3] = {in.n_cur, in.n_next, in.n_next2};
  for (int li = 0; li < 3; ++li) {
    if (ns[li] < 0 || (ns[li] > 0 && !lists[li])) fail(PS_EINVAL, "LayerInputs: bad list");
    for (int i = 0; i < ns[li]; ++i) {
      if (lists[li][i].location != PS_LOC_HOST)
        fail(PS_EINVAL, "LayerInputs: lists must contain Host experts only");
      if (lists[li][i].tokens < 1)
        fail(PS_EINVAL, "LayerInputs: schedulable experts need tokens >= 1");
      if (i > 0 && lists[li][i - 1].tokens > lists[li][i].tokens)
        fail(PS_EINVAL, "LayerInputs: lists must be sorted ascending by tokens");
    }
  }
}

// Prefix sums of the per-expert CPU cost over a list: P[i] = sum_{j<i} cpu(list[j]).
std::vector<int64_t> cpu_prefix(const ps_expert_load* l, int n, const ps_cost_params& p) {
  std::vector<int64_t> P(static_cast<size_t>(n) + 1, 0);
  for (int i = 0; i < n; ++i) P[i + 1] = P[i] + cpu_cost_of(l[i].tokens, p);
  return P;
}

struct Merged {
  int tokens, expert;
  bool current;
  int index_in_list;
};

// Cross-layer merge order of scheduler.cpp:54-69: (tokens asc, current first,
// expert asc), stable.
std::vector<Merged> merge_lists(const ps_expert_load* cur, int n, const ps_expert_load* nxt, int m) {
  std::vector<Merged> v;
  v.reserve(static_cast<size_t>(n) + m);
  for (int i = 0; i < n; ++i) v.push_back({cur[i].tokens, cur[i].expert, true, i});
  for (int i = 0; i < m; ++i) v.push_back({nxt[i].tokens, nxt[i].expert, false, i});
  std::stable_sort(v.begin(), v.end(), [](const Merged& a, const Merged& b) {
    if (a.tokens != b.tokens) return a.tokens < b.tokens;
    if (a.current != b.current) return a.current;
    return a.expert < b.expert;
  });
  return v;
}

// GPU-queue membership (Eq.4 sweep): merged element k joins iff
// alpha + (N-k) t_io + t_g < sum_{j<=k} cpu + t_attn. Returns the member flags.
std::vector<char> gpu_queue(const std::vector<Merged>& merged, const ps_cost_params& p,
                            int64_t* sweep_gpu, int64_t* sweep_cpu) {
  const int N = static_cast<int>(merged.size());
  std::vector<char> member(N, 0);
  int64_t prefix = 0;
  for (int k = 0; k < N; ++k) {
    prefix += cpu_cost_of(merged[k].tokens, p);
    const int64_t g = p.alpha + static_cast<int64_t>(N - k) * p.t_io + p.t_g;
    const int64_t c = prefix + p.t_attn;
    if (sweep_gpu) sweep_gpu[k] = g;
    if (sweep_cpu) sweep_cpu[k] = c;
    member[k] = g < c;
  }
  return member;
}

// Completion estimate of suffix split s (scheduler.cpp:99-106).
inline int64_t split_cost(int s, int n, const std::vector<int64_t>& P, const ps_cost_params& p) {
  if (s == n) return P[n];
  const int64_t tg = p.alpha + static_cast<int64_t>(n - s) * p.t_io + p.t_g;
  return std::max(P[s], tg);
}

void set_sets(const ps_layer_inputs& in, int split, ps_layer_plan& out) {
  out.split_index = split;
  out.n_cpu = split;
  out.n_ondemand = in.n_cur - split;
  if (out.cpu_set) std::copy(in.e_cur, in.e_cur + split, out.cpu_set);
  if (out.ondemand_seq) std::copy(in.e_cur + split, in.e_cur + in.n_cur, out.ondemand_seq);
}

void set_prefetch(const ps_expert_load* list, int len, int c, ps_layer_plan& out) {
  out.issued_prefetches = c;
  out.n_prefetch = c;
  if (out.prefetch_seq)
    for (int i = 0; i < c; ++i) out.prefetch_seq[i] = list[len - 1 - i];  // hottest first
}

void current_costs(int ip, int n, const std::vector<int64_t>& P, const ps_cost_params& p,
                   ps_decision_trace& t) {
  t.t_g_at_split = p.alpha + static_cast<int64_t>(n - ip) * p.t_io + p.t_g;
  t.t_c_at_split = P[ip];
}

void presched(const ps_layer_inputs& in, ps_layer_plan& out) {
  const ps_cost_params& p = in.params;
  const int n = in.n_cur;
  const std::vector<int64_t> P = cpu_prefix(in.e_cur, n, p);
  ps_decision_trace& tr = out.trace;

  std::vector<Merged> merged = merge_lists(in.e_cur, n, in.e_next, in.n_next);
  std::vector<char> member = gpu_queue(merged, p, tr.sweep_gpu, tr.sweep_cpu);
  tr.n_sweep = static_cast<int32_t>(merged.size());

  // On-demand split: first current-layer GPU_Q member (token order) with T_G < T_C.
  int split = n;
  bool queue_has_next = false;
  for (size_t k = 0; k < merged.size(); ++k) {
    if (!member[k]) continue;
    if (!merged[k].current) {
      queue_has_next = true;
      continue;
    }
    if (split != n) continue;
    const int ip = merged[k].index_in_list;
    const int64_t g = p.alpha + static_cast<int64_t>(n - ip) * p.t_io + p.t_g;
    if (g < P[ip]) split = ip;
  }
  current_costs(split, n, P, p, tr);

  // All-GPU fallback (scheduler.cpp:197-205).
  if (n > 0 && split_cost(0, n, P, p) < split_cost(split, n, P, p)) {
    split = 0;
    tr.all_gpu_fallback = 1;
    current_costs(0, n, P, p, tr);
  }
  set_sets(in, split, out);

  // Gap-window prefetch with one widening step (scheduler.cpp:147-186).
  const ps_expert_load* target = in.e_next;
  int target_len = in.n_next;
  bool widened = false;
  if (!queue_has_next) {
    widened = true;
    tr.widened_window = 1;
    bool has2 = false;
    if (in.n_next2 > 0) {
      std::vector<Merged> m2 = merge_lists(in.e_cur, n, in.e_next2, in.n_next2);
      std::vector<char> mem2 = gpu_queue(m2, p, nullptr, nullptr);
      for (size_t k = 0; k < m2.size() && !has2; ++k) has2 = mem2[k] && !m2[k].current;
    }
    if (!has2) {
      set_prefetch(nullptr, 0, 0, out);
      out.prefetch_from_widened = 0;
      return;
    }
    target = in.e_next2;
    target_len = in.n_next2;
  }
  const int64_t loads = static_cast<int64_t>(n) - split;
  const int64_t t_gap = P[split] - p.alpha - loads * p.t_io;
  const double f = static_cast<double>(t_gap + p.t_attn) / p.t_io;
  const int f_int = static_cast<int>(ticks(std::max(f, 0.0)));
  const double t_e = static_cast<double>(p.t_io);
  const double xi = in.stats.r_hit * (f - f_int + 1.0) * t_e - in.stats.r_miss * (f_int - f) * t_e;
  int c = xi > 0 ? f_int : std::max(f_int - 1, 0);
  c = std::min(c, target_len);
  tr.t_gap = t_gap;
  tr.f = f;
  tr.f_int = f_int;
  tr.xi = xi;
  set_prefetch(target, target_len, c, out);
  out.prefetch_from_widened = widened && c > 0;
}

// Layer-local greedy (Eq.2) with ceil-fill prefetch (scheduler.cpp:215-250).
void greedy(const ps_layer_inputs& in, ps_layer_plan& out) {
  const ps_cost_params& p = in.params;
  const int n = in.n_cur;
  const std::vector<int64_t> P = cpu_prefix(in.e_cur, n, p);
  int best = n;
  int64_t best_cost = split_cost(n, n, P, p);
  for (int s = n - 1; s >= 0; --s) {
    const int64_t cost = split_cost(s, n, P, p);
    if (cost < best_cost) {  // ties keep the larger s
      best_cost = cost;
      best = s;
    }
  }
  set_sets(in, best, out);
  current_costs(best, n, P, p, out.trace);
  const int64_t t_free = p.alpha + static_cast<int64_t>(n - best) * p.t_io;
  const int64_t window_end = best_cost + p.t_attn;
  int cnt = 0;
  if (t_free < window_end)
    cnt = std::min<int>(static_cast<int>((window_end - t_free + p.t_io - 1) / p.t_io), in.n_next);
  set_prefetch(in.e_next, in.n_next, cnt, out);
  out.trace.t_gap = out.trace.t_c_at_split - t_free;
  out.trace.f_int = cnt;
}

void reset_plan(ps_layer_plan& out) {
  out.n_cpu = out.n_ondemand = out.n_prefetch = 0;
  out.prefetch_from_widened = out.split_index = out.issued_prefetches = 0;
  int64_t* sg = out.trace.sweep_gpu;
  int64_t* sc = out.trace.sweep_cpu;
  std::memset(&out.trace, 0, sizeof(out.trace));
  out.trace.sweep_gpu = sg;
  out.trace.sweep_cpu = sc;
}

}  // namespace

void plan_layer(const ps_layer_inputs& in, ps_policy pol, ps_layer_plan& out) {
  reset_plan(out);
  switch (pol.kind) {
    case PS_POLICY_PRESCHED:
      validate_inputs(in);
      presched(in, out);
      return;
    case PS_POLICY_GREEDY:
      validate_inputs(in);
      greedy(in, out);
      return;
    case PS_POLICY_ONDEMAND: {
      validate_inputs(in);
      set_sets(in, 0, out);
      current_costs(0, in.n_cur, cpu_prefix(in.e_cur, in.n_cur, in.params), in.params, out.trace);
      return;
    }
    case PS_POLICY_FIXED: {
      validate_inputs(in);
      greedy(in, out);
      int cnt = std::min<int>(pol.fixed_prefetch, in.n_next);
      set_prefetch(in.e_next, in.n_next, cnt, out);
      out.trace.f_int = cnt;
      return;
    }
    case PS_POLICY_ORACLE:
      fail(PS_EINVAL, "oracle policy requires the pipeline enumerator");
  }
  fail(PS_EINVAL, "unknown policy kind");
}

}  // namespace ps

using namespace ps;

extern "C" {

int64_t ps_to_ticks(double x) { return ticks(x); }

ps_status ps_cost_params_validate(const ps_cost_params* p) {
  return guarded([&] { validate_params(*p); });
}

ps_status ps_hit_stats_record(ps_hit_stats* s, int hit) {
  return guarded([&] {
    double w = 1.0 / s->window;
    s->r_hit = (1.0 - w) * s->r_hit + (hit ? w : 0.0);
    s->r_miss = 1.0 - s->r_hit;
  });
}

ps_status ps_cpu_cost(int tokens, const ps_cost_params* p, int64_t* out) {
  return guarded([&] {
    require(tokens >= 0, "cpu_cost: negative token count");
    *out = cpu_cost_of(tokens, *p);
  });
}

ps_status ps_overlap_prefetch_count(int64_t t_gap, const ps_cost_params* p, double* f, int* f_int) {
  return guarded([&] {
    require(p->t_io > 0, "overlap_prefetch_count: t_io must be > 0");
    *f = static_cast<double>(t_gap + p->t_attn) / p->t_io;
    *f_int = static_cast<int>(ticks(std::max(*f, 0.0)));
  });
}

double ps_prefetch_gain(const ps_hit_stats* s, double f, int f_int, const ps_cost_params* p) {
  double t_e = static_cast<double>(p->t_io);
  return s->r_hit * (f - f_int + 1.0) * t_e - s->r_miss * (f_int - f) * t_e;
}

ps_status ps_fit_cost_params(const int32_t* tokens, const int64_t* tk, int n, double* beta,
                             double* startup, double* r2) {
  return guarded([&] {
    std::set<int> distinct(tokens, tokens + n);
    require(distinct.size() >= 2, "fit_cost_params: need >= 2 distinct token counts");
    const double N = n;
    double sx = 0, sy = 0, sxx = 0, sxy = 0;
    for (int i = 0; i < n; ++i) {
      sx += tokens[i];
      sy += static_cast<double>(tk[i]);
      sxx += static_cast<double>(tokens[i]) * tokens[i];
      sxy += static_cast<double>(tokens[i]) * tk[i];
    }
    double denom = N * sxx - sx * sx;
    *beta = (N * sxy - sx * sy) / denom;
    *startup = (sy - *beta * sx) / N;
    double ybar = sy / N, ss_res = 0, ss_tot = 0;
    for (int i = 0; i < n; ++i) {
      double pred = *beta * tokens[i] + *startup;
      ss_res += (tk[i] - pred) * (tk[i] - pred);
      ss_tot += (tk[i] - ybar) * (tk[i] - ybar);
    }
    *r2 = ss_tot > 0 ? 1.0 - ss_res / ss_tot : 1.0;
  });
}

ps_status ps_policy_parse(const char* text, ps_policy* out) {
  return guarded([&] {
    std::string t = text ? text : "";
    ps_policy p{PS_POLICY_PRESCHED, 0};
    if (t == "presched") p.kind = PS_POLICY_PRESCHED;
    else if (t == "greedy") p.kind = PS_POLICY_GREEDY;
    else if (t == "ondemand") p.kind = PS_POLICY_ONDEMAND;
    else if (t == "oracle") p.kind = PS_POLICY_ORACLE;
    else if (t.rfind("fixed:", 0) == 0) {
      p.kind = PS_POLICY_FIXED;
      p.fixed_prefetch = std::stoi(t.substr(6));
      require(p.fixed_prefetch >= 0, "fixed:<c> needs c >= 0");
    } else {
      fail(PS_EINVAL, "unknown policy: " + t);
    }
    *out = p;
  });
}

ps_status ps_policy_name(ps_policy p, char* buf, int cap) {
  return guarded([&] {
    std::string n;
    switch (p.kind) {
      case PS_POLICY_PRESCHED: n = "presched"; break;
      case PS_POLICY_GREEDY: n = "greedy"; break;
      case PS_POLICY_ONDEMAND: n = "ondemand"; break;
      case PS_POLICY_FIXED: n = "fixed:" + std::to_string(p.fixed_prefetch); break;
      case PS_POLICY_ORACLE: n = "oracle"; break;
      default: n = "?";
    }
    require(cap > static_cast<int>(n.size()), "policy name buffer too small");
    std::memcpy(buf, n.c_str(), n.size() + 1);
  });
}

ps_status ps_layer_inputs_validate(const ps_layer_inputs* in) {
  return guarded([&] { validate_inputs(*in); });
}

ps_status ps_presched_plan(const ps_layer_inputs* in, ps_policy policy, ps_layer_plan* out) {
  return guarded([&] { plan_layer(*in, policy, *out); });
}

}  // extern "C"
