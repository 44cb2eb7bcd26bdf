// Reference-style call sites compiled against include/prescope_b200.hpp (the drop-in
// C++ mirror over the C ABI). Cases restate test_scheduler.cpp / test_golden.cpp /
// test_workload.cpp checks; exits non-zero on the first failure.
#include <cstdio>
#include <cstdlib>

#include "prescope_b200.hpp"

using namespace prescope;

#define CHECK(c)                                                      \
  do {                                                                \
    if (!(c)) {                                                       \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
      std::exit(1);                                                   \
    }                                                                 \
  } while (0)

template <typename Ex, typename F>
bool throws(F&& f) {
  try {
    f();
  } catch (const Ex&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main() {
  // workload: presets, desk scale, top-k ties (test_workload.cpp:26-61, 187-192)
  ModelSpec m = mixtral_spec();
  CHECK(m.num_layers == 32 && m.experts_per_layer == 8 && m.top_k == 2 && m.hidden_dim == 4096);
  CHECK(m.group_begin_middle == 4 && m.group_begin_output == 28);
  CHECK(m.group_of(27) == LayerGroup::Middle && m.group_of(28) == LayerGroup::Output);
  CHECK(throws<std::out_of_range>([&] { m.group_of(32); }));
  CHECK(throws<std::invalid_argument>([] { spec_preset("gpt"); }));
  ModelSpec s = desk_scale(deepseek_spec(), 8, 8, 32);
  CHECK(s.top_k == 6 && s.group_begin_middle == 2 && s.group_begin_output == 6);
  CHECK((topk_indices({0.1, 0.4, 0.4, 0.05, 0.05}, 3) == std::vector<int>{1, 2, 0}));
  CHECK(routing_map(desk_scale(mixtral_spec(), 4, 8, 16), 7) == 0);

  // scheduler (test_scheduler.cpp:60-72, 129-140, 186-228, 270-287)
  CHECK(SchedulerPolicy::parse("fixed:3").fixed_prefetch == 3);
  CHECK(SchedulerPolicy::parse("greedy").name() == "greedy");
  CHECK(throws<std::invalid_argument>([] { SchedulerPolicy::parse("fifo"); }));
  LayerInputs in;
  in.params = {10, 2, 3, 1.0, 1, 0};
  in.e_cur = {{0, 0, 5, ExpertLocation::Host}, {1, 0, 2, ExpertLocation::Host}};
  CHECK(throws<std::invalid_argument>([&] { schedule_layer(in); }));
  in.params = {2, 1, 3, 1.0, 1, 0};
  in.e_cur = {{0, 0, 3, ExpertLocation::Host}, {1, 0, 50, ExpertLocation::Host}};
  LayerPlan plan = schedule_layer(in);
  CHECK(plan.split_index == 1 && plan.ondemand_seq.size() == 1u && plan.ondemand_seq[0].expert == 1);
  in = LayerInputs{};
  in.params = {5, 2, 3, 1.0, 1, 0};
  in.e_cur = {{0, 0, 5, ExpertLocation::Host}};
  in.e_next2 = {{1, 2, 2, ExpertLocation::Host}, {2, 2, 50, ExpertLocation::Host}};
  plan = schedule_layer(in);
  CHECK(plan.trace.widened_window && plan.prefetch_from_widened && plan.trace.f_int == 2);
  CHECK(plan.issued_prefetches == 2 && plan.prefetch_seq[0].expert == 2 && plan.prefetch_seq[1].expert == 1);
  in.e_next2.clear();
  in.e_cur = {{0, 0, 100, ExpertLocation::Host}};
  plan = schedule_layer(in);
  CHECK(plan.split_index == 0 && plan.trace.all_gpu_fallback && plan.cpu_set.empty());
  in = LayerInputs{};
  in.params = {4, 2, 0, 1.0, 0, 0};
  in.e_cur = {{0, 0, 3, ExpertLocation::Host}, {1, 0, 7, ExpertLocation::Host}, {2, 0, 8, ExpertLocation::Host}};
  CHECK(greedy_layer_baseline(in).split_index == 2);
  CHECK(ondemand_only_plan(in).split_index == 0);
  CHECK(throws<std::invalid_argument>([&] { plan_layer(in, SchedulerPolicy::parse("oracle")); }));

  // cost model (test_cost_model.cpp:15-24, 147-173)
  CHECK(to_ticks(0.5) == 1 && to_ticks(-0.5) == 0 && to_ticks(-0.51) == -1);
  CostParams p{14, 2, 3, 3.0, 2, 0};
  PrefetchCount pc = overlap_prefetch_count(17, p);
  CHECK(pc.f_int == 1);
  CHECK(prefetch_gain(HitStats{}, pc.f, pc.f_int, p) == 20.0);
  CHECK(cpu_cost(4, p) == 14);

  // golden case 4 (golden.cpp:61-234; test_golden.cpp:36-48): PreSched makespan 53
  PipelineInstance inst;
  inst.layers.resize(2);
  inst.layers[0].truth = {{0, 4}, {1, 5}, {2, 9}};
  inst.layers[1].truth = {{3, 6}, {4, 8}};
  inst.layers[1].predicted = inst.layers[1].truth;
  SimResult r = simulate_policy(inst, SchedulerPolicy::parse("presched"), p);
  CHECK(r.timeline.makespan == 53);
  CHECK(verify_timeline(r.timeline, inst, p).empty());
  CHECK(simulate_policy(inst, SchedulerPolicy::parse("ondemand"), p).timeline.makespan == 80);
  Metrics met = compute_metrics(r.timeline, 1);  // simulator.cpp:396-426
  CHECK(met.makespan == 53 && met.decode_latency == 53 && met.per_layer_latency.size() == 2);
  CHECK(met.io_busy_fraction > 0.0 && met.gpu_idle_fraction < 1.0);
  Timeline bad = r.timeline;
  bad.events.push_back({100, 102, Resource::Gpu, EventKind::GpuExpert, 0, 7, 1});
  CHECK(!verify_timeline(bad, inst, p).empty());
  // trace files (test_workload.cpp round-trip + checksum): a reference-written file reads
  // into prescope::Trace, re-writes byte-identically, and a corrupted copy throws
  // TraceChecksumError (PRESCOPE_GOLDEN_TRACE points at tests/golden/ref_trace_desk.tsv).
  if (const char* gold = std::getenv("PRESCOPE_GOLDEN_TRACE")) {
    Trace t = read_trace(gold);
    CHECK(t.batch_size == 3 && t.seed == 17 && t.spec.num_layers == 4 && t.steps.size() == 12);
    CHECK(t.step(2, 3).layer == 3 && t.step(0, 0).active_experts.size() == 2);
    CHECK(topk_indices(t.step(1, 2).gate_weights, 2) == t.step(1, 2).active_experts);
    int total = 0;
    for (auto [e, m] : aggregate_layer_loads(t, 1)) total += m;
    CHECK(total == 3 * 2);
    const std::string out = std::string(gold) + ".shim_rt.tsv";
    write_trace(t, out);
    CHECK(read_trace(out) == t);
    {
      std::FILE* f = std::fopen(out.c_str(), "r+b");
      CHECK(f != nullptr);
      std::fseek(f, -5, SEEK_END);
      std::fputc('9', f);
      std::fclose(f);
    }
    CHECK(throws<TraceChecksumError>([&] { read_trace(out); }));
    CHECK(throws<std::out_of_range>([&] { t.step(3, 0); }));
    std::remove(out.c_str());
  }

  std::printf("shim ok\n");
  return 0;
}
