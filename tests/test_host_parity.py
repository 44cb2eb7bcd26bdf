"""Host-side product code vs the reference: RNG replay of the routing inputs,
PreSched plans (bit-exact, incl. f and xi), the AsyncIO model-clock pipeline (golden
timelines tick-exact) and verify_timeline. All through the C ABI (libprescope_b200)."""
import json
import random

import numpy as np
import pytest

import oracle as orc
import paper_2509_23638_b200 as ps
from conftest import GOLDEN

needs_ref = pytest.mark.skipif(not orc.ref_available(), reason="oracle/_ref not built")


def test_spec_presets():
    m = ps.spec_preset("mixtral")
    assert (m.num_layers, m.experts_per_layer, m.top_k, m.hidden_dim) == (32, 8, 2, 4096)
    assert (m.group_begin_middle, m.group_begin_output) == (4, 28)
    assert ps.ffn_dim(m) == 14336
    assert ps.ffn_dim(ps.spec_preset("qwen3")) == 768
    assert ps.ffn_dim(ps.spec_preset("deepseek")) == 1408
    d = ps.desk_scale("deepseek", 8, 8, 32)
    assert (d.top_k, d.group_begin_middle, d.group_begin_output) == (6, 2, 6)
    with pytest.raises(ps.capi.PsError) as e:
        ps.spec_preset("gpt")
    assert e.value.status == ps.capi.PS_EINVAL


def test_trace_inputs_bit_exact_vs_golden():
    d = np.load(GOLDEN / "desk_trace_c0.npz")
    spec = ps.desk_scale("mixtral", 4, 8, 16)
    cfg = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    _, hidden, follow, _ = ps.trace_inputs(cfg, spec, 32, 0)
    assert np.array_equal(hidden, d["hidden"])
    assert follow[:, 0].sum() == 0  # layer 0 never follows


@needs_ref
@pytest.mark.parametrize("preset,L,E,H,B,seed", [("mixtral", 6, 8, 16, 12, 17), ("qwen3", 5, 128, 64, 4, 3),
                                                 ("deepseek", 4, 64, 32, 6, 9)])
def test_trace_inputs_vs_reference(preset, L, E, H, B, seed):
    spec = ps.desk_scale(preset, L, E, H)
    knobs = (0.9, 0.3, 0.5)
    cfg = ps.TraceGenConfig(knobs, (0.95, 0.6, 1.0), knobs)
    _, hidden, _, _ = ps.trace_inputs(cfg, spec, B, seed)
    h2, _, _ = orc.ref_trace(orc.ref_gen(knobs, (0.95, 0.6, 1.0), knobs), orc.ref_spec_from(spec), B, seed)
    assert np.array_equal(hidden, h2)


def _plan_dict(p):
    return {k: (getattr(p, k)) for k in p.__dataclass_fields__}


def test_presched_product_vs_golden_cases():
    data = json.loads((GOLDEN / "presched_cases.json").read_text())
    for c in data["cases"]:
        for pol, ref in c["plans"].items():
            got = _plan_dict(ps.plan_layer([tuple(x) for x in c["e_cur"]], [tuple(x) for x in c["e_next"]],
                                           [tuple(x) for x in c["e_next2"]], tuple(c["params"]), tuple(c["stats"]),
                                           pol))
            for key, val in ref.items():
                if key in ("cpu_set", "ondemand_seq", "prefetch_seq"):
                    val = [tuple(x) for x in val]
                if key in ("sweep_gpu", "sweep_cpu") and pol != "presched":
                    continue
                assert got[key] == val, (pol, key)
    for b in data["invalid"]:
        with pytest.raises(ps.capi.PsError) as e:
            ps.plan_layer([tuple(x) for x in b["e_cur"]], [], [], tuple(b["params"]))
        assert e.value.status == b["rc"] == ps.capi.PS_EINVAL


@needs_ref
def test_presched_product_vs_reference_random_large():
    """>= 10^4 random LayerInputs incl. long lists (n = n' up to 256, the O(n^2) regime)."""
    rng = random.Random(99)
    n = 0
    for it in range(2500):
        hi = 256 if it % 50 == 0 else 12

        def lst(layer, lo):
            m = rng.randint(lo, hi)
            return sorted([(e, layer, rng.randint(1, 40)) for e in range(m)], key=lambda x: (x[2], x[0]))
        t_io = rng.randint(5, 300)
        params = (t_io, rng.randint(1, min(t_io - 1, 40)), rng.randint(0, 100), rng.choice([0.5, 1.0, 2.7, 1e9]),
                  rng.randint(0, 5), rng.randint(0, 200))
        h = rng.random()
        cur, nxt, nxt2 = lst(0, 1), lst(1, 0), lst(2, 0)
        for pol in ("presched", "greedy", "ondemand", "fixed:3"):
            rc, ref = orc.ref_plan_layer(cur, nxt, nxt2, params, (h, 1 - h, 32), pol)
            got = _plan_dict(ps.plan_layer(cur, nxt, nxt2, params, (h, 1 - h, 32), pol))
            for key, val in ref.items():
                if key in ("sweep_gpu", "sweep_cpu") and pol != "presched":
                    continue
                assert got[key] == val, (pol, key, cur, nxt, params)
            n += 1
    assert n >= 10000


def test_policy_parse_roundtrip():
    import ctypes as C
    lib = ps.load()
    for name in ("presched", "greedy", "ondemand", "oracle", "fixed:2"):
        buf = C.create_string_buffer(32)
        ps.check(lib.ps_policy_name(ps.parse_policy(name), buf, 32))
        assert buf.value.decode() == name
    for bad in ("fifo", "fixed:-1"):
        with pytest.raises(ps.capi.PsError):
            ps.parse_policy(bad)
    with pytest.raises(ps.capi.PsError):
        ps.plan_layer([(0, 0, 1)], [], [], (10, 2, 3, 1.0, 1, 0), policy="oracle")


def _golden_instance(s):
    inst = s["instance"]
    L = len(inst["layers"])
    E = 1 + max(e for ly in inst["layers"] for e, _ in ly["truth"] + ly["predicted"])
    truth, pred = np.zeros((L, E), np.int32), np.zeros((L, E), np.int32)
    for l, ly in enumerate(inst["layers"]):
        for e, m in ly["truth"]:
            truth[l, e] = m
        for e, m in ly["predicted"]:
            pred[l, e] = m
    p = s["params"]
    return truth, pred, (p["t_io"], p["t_g"], p["t_attn"], p["beta"], p["startup"], p["alpha"])


def test_golden_scenarios_replay_tick_exactly():
    scen = json.loads((GOLDEN / "golden_scenarios.json").read_text())
    assert len(scen) == 6
    spans = {}
    for s in scen:
        truth, pred, params = _golden_instance(s)
        r = ps.simulate(truth, pred, params, s["policy"])
        exp = s["expected"]
        assert [list(e) for e in r["events"]] == exp["events"], s["id"]
        assert r["layer_start"] == exp["layer_start"] and r["layer_end"] == exp["layer_end"]
        spans[s["id"]] = r["makespan"]
        pre = ps.simulate(truth, pred, params, "presched")
        assert [list(e) for e in pre["events"]] == s["presched_timeline"]["events"]
        assert ps.verify_timeline(pre["events"], truth, params) == []
    # test_golden.cpp:36-48
    assert spans == {"prefetch-case1-ondemand": 80, "prefetch-case2-mispredicted": 61,
                     "prefetch-case3-layerwise": 56, "prefetch-case4-crosslayer": 53,
                     "greedy-case1-gpu-bound": 47, "greedy-case2-cpu-bound": 61}


def test_gpu_bound_overhang():
    # test_golden.cpp:50-65
    s = {x["id"]: x for x in json.loads((GOLDEN / "golden_scenarios.json").read_text())}["greedy-case1-gpu-bound"]
    truth, pred, params = _golden_instance(s)
    ev = ps.simulate(truth, pred, params, "greedy")["events"]
    attn1 = [e for e in ev if e[3] == 0 and e[4] == 1][0]
    pf = [e for e in ev if e[3] == 4 and e[4] == 1][0]
    load1 = [e for e in ev if e[3] == 3 and e[4] == 1][0]
    assert attn1[1] == 22 and pf[1] == 31 and load1[0] == 31


def test_random_pipelines_vs_golden_reference_timelines():
    cases = json.loads((GOLDEN / "sim_cases.json").read_text())
    for c in cases:
        truth, pred, res = np.array(c["truth"]), np.array(c["predicted"]), np.array(c["resident"])
        for pol, ref in c["runs"].items():
            r = ps.simulate(truth, pred, tuple(c["params"]), pol, resident=res, groups=c["groups"],
                            options=(1, 64, 1.0, 32))
            assert [list(e) for e in r["events"]] == ref["events"], pol
            assert r["makespan"] == ref["makespan"]
            assert [list(p) for p in r["plans"]] == ref["plans"]
            assert len(ps.verify_timeline(r["events"], truth, tuple(c["params"]), res)) == ref["violations"] == 0


def test_verify_timeline_injected_faults():
    # test_simulator.cpp:130-193 style: overlap, double compute, missing transfer, ghost
    truth = np.array([[4, 5]], np.int32)
    params = (10, 2, 3, 1.0, 1, 0)
    good = ps.simulate(truth, truth, params, "ondemand")["events"]
    assert ps.verify_timeline(good, truth, params) == []
    ev = [list(e) for e in good]
    loads = [e for e in ev if e[3] == 3]
    overlap = [list(e) for e in ev]
    for e in overlap:
        if e == loads[1]:
            e[0] -= 5
            e[1] -= 5
    assert any("serial-io" in m for m in ps.verify_timeline([tuple(e) for e in overlap], truth, params))
    ghost = ev + [[100, 102, 0, 1, 0, 7, 1]]
    assert any("non-activated" in m for m in ps.verify_timeline([tuple(e) for e in ghost], truth, params,))
    missing = [e for e in ev if not (e[3] == 3 and e[5] == 0)]
    assert any("causality" in m for m in ps.verify_timeline([tuple(e) for e in missing], truth, params))
    double = ev + [e for e in ev if e[3] == 1][:1]
    assert any("computed 2 times" in m for m in ps.verify_timeline([tuple(e) for e in double], truth, params))


def test_plan_fn_plugin_seam():
    """PlanFn (simulator.hpp:66): a C callback can replace the policy; here it reuses
    the library's own planner and must reproduce the policy timeline."""
    import ctypes as C
    lib = ps.load()
    pol = ps.parse_policy("presched")

    def cb(user, inputs, layer, plan):
        return lib.ps_presched_plan(inputs, pol, plan)
    s = json.loads((GOLDEN / "golden_scenarios.json").read_text())[3]
    truth, pred, params = _golden_instance(s)
    assert ps.simulate(truth, pred, params, plan_fn=cb)["events"] == \
        ps.simulate(truth, pred, params, "presched")["events"]


def test_residency_product_vs_oracle():
    rng = np.random.default_rng(3)
    for _ in range(50):
        L, E = int(rng.integers(1, 40)), int(rng.integers(1, 130))
        freq = rng.integers(0, 5, (L, E)).astype(np.int64)
        budget = int(rng.integers(0, L * E + 2)) * 1000 + int(rng.integers(0, 999))
        got = ps.plan_residency(freq, budget, 1000)
        out = np.empty((L * E, 2), np.int32)
        n = orc.oracle_lib().or_plan_residency(freq.ctypes.data, L, E, budget, 1000, out.ctypes.data)
        assert got == [tuple(map(int, r)) for r in out[:n]]


def test_cost_model_kats():
    import ctypes as C
    lib = ps.load()
    # test_cost_model.cpp:15-24: half-up, negatives
    assert [lib.ps_to_ticks(x) for x in (0.5, 1.49, -0.5, -0.51, 2.5)] == [1, 1, 0, -1, 3]
    p = ps.capi.CostParams(14, 2, 3, 3.0, 2, 0)
    f, fi = C.c_double(), C.c_int()
    ps.check(lib.ps_overlap_prefetch_count(17, C.byref(p), C.byref(f), C.byref(fi)))
    assert f.value == pytest.approx(20 / 14) and fi.value == 1
    s = ps.capi.HitStats(1.0, 0.0, 32)
    assert lib.ps_prefetch_gain(C.byref(s), f.value, fi.value, C.byref(p)) == pytest.approx(20.0)
    ps.check(lib.ps_hit_stats_record(C.byref(s), 0))
    assert s.r_hit == pytest.approx(31 / 32) and s.r_miss == pytest.approx(1 / 32)
    tok = np.arange(1, 51, dtype=np.int32)
    tk = (3 * tok + 5).astype(np.int64)
    b, c, r2 = C.c_double(), C.c_double(), C.c_double()
    ps.check(lib.ps_fit_cost_params(tok.ctypes.data, tk.ctypes.data, 50, C.byref(b), C.byref(c), C.byref(r2)))
    assert b.value == pytest.approx(3.0) and c.value == pytest.approx(5.0) and r2.value == pytest.approx(1.0)


def test_export_timeline_text_matches_reference():
    """export_timeline (simulator.cpp:428-436): same text as the reference for every
    golden timeline (and the GPU engine's measured timelines use the same call)."""
    import ctypes as C
    import oracle as orc
    lib = ps.load()
    scen = json.loads((GOLDEN / "golden_scenarios.json").read_text())
    for s in scen:
        ev = s["presched_timeline"]["events"]
        mk = s["presched_timeline"].get("makespan", max(e[1] for e in ev))
        arr = (ps.capi.TimelineEvent * len(ev))(*[ps.capi.TimelineEvent(*e) for e in ev])
        need = C.c_int()
        ps.check(lib.ps_export_timeline(arr, len(ev), mk, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        ps.check(lib.ps_export_timeline(arr, len(ev), mk, buf, need.value, C.byref(need)))
        text = buf.value.decode()
        assert text.startswith(f"# tick_unit=us makespan={mk}\n") and text.count("\n") == len(ev) + 1
        if orc.ref_available():
            rarr = (orc.RefEvent * len(ev))(*[orc.RefEvent(*e) for e in ev])
            rneed = C.c_int()
            orc.ref_check(orc.ref_lib().ref_export_timeline(rarr, len(ev), mk, None, 0, C.byref(rneed)))
            rbuf = C.create_string_buffer(rneed.value)
            orc.ref_check(orc.ref_lib().ref_export_timeline(rarr, len(ev), mk, rbuf, rneed.value, C.byref(rneed)))
            assert rbuf.value.decode() == text


def _metrics_pair(events, ls, le, makespan, tokens):
    m, pl, gap = ps.compute_metrics(events, ls, le, makespan, tokens)
    mine = np.array([m.makespan, m.decode_latency, m.throughput_tokens_per_s, m.io_busy_fraction,
                     m.gpu_idle_fraction])
    return (mine, pl, gap), orc.ref_compute_metrics(events, ls, le, makespan, tokens)


@pytest.mark.skipif(not orc.ref_available(), reason="oracle/_ref not built")
def test_compute_metrics_matches_reference():
    """ps_compute_metrics == the reference's compute_metrics (simulator.cpp:396-426),
    bitwise, on every golden timeline, on the random pipelines under all four policies,
    and on a Timeline whose makespan field is NOT max(t_end) (the reference reads the
    field; so does ps_compute_metrics)."""
    timelines = []
    for s in json.loads((GOLDEN / "golden_scenarios.json").read_text()):
        truth, pred, params = _golden_instance(s)
        for pol in (s["policy"], "presched"):
            timelines.append(ps.simulate(truth, pred, params, pol))
    for c in json.loads((GOLDEN / "sim_cases.json").read_text())[:100]:
        truth, pred, res = np.array(c["truth"]), np.array(c["predicted"]), np.array(c["resident"])
        for pol in c["runs"]:
            timelines.append(ps.simulate(truth, pred, tuple(c["params"]), pol, resident=res, groups=c["groups"],
                                         options=(1, 64, 1.0, 32)))
    for i, r in enumerate(timelines):
        for makespan in (r["makespan"], r["makespan"] + 17):
            (a, pl, gap), (b, pl2, gap2) = _metrics_pair(r["events"], r["layer_start"], r["layer_end"], makespan,
                                                        1 + i % 7)
            assert np.array_equal(a, b) and np.array_equal(pl, pl2) and np.array_equal(gap, gap2), i
    # an event of a layer outside the timeline is an index error (the reference would read out of bounds)
    r = timelines[0]
    bad = list(r["events"]) + [(0, 1, 0, 1, len(r["layer_start"]), 0, 1)]
    with pytest.raises(ps.capi.PsError) as err:
        ps.compute_metrics(bad, r["layer_start"], r["layer_end"], r["makespan"], 1)
    assert err.value.status == ps.capi.PS_ERANGE
