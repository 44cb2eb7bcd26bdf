"""Decode engine (K5 + the per-layer driver) end to end through the C ABI vs the CPU
oracle: routing ids vs the f64 router, per-layer MoE outputs vs the SwiGLU oracle on
the same synthetic bf16 weights, and loader accounting (every non-resident routed
expert crosses PCIe exactly once per layer it is used in)."""
import numpy as np
import pytest

import oracle as orc
import paper_2509_23638_b200 as ps
from paper_2509_23638_b200 import engine as eng
from conftest import GOLDEN as GOLD

pytestmark = pytest.mark.gpu

BF16_RTOL = 2e-2


def _small_spec(L=4, E=8, H=256, F=512, preset="mixtral"):
    spec = ps.desk_scale(preset, L, E, H)
    spec.expert_bytes = 6 * H * F
    return spec


def _run(spec, B, budget, policy="presched", seed=3, steps=2, predictor=None, n_shared=0, **kw):
    cfg = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    gate, hidden, follow, zipf = ps.trace_inputs(cfg, spec, B, seed)
    F = ps.ffn_dim(spec)
    with eng.Engine(spec, cfg, budget_fraction=budget, max_batch=B, weight_seed=9, gate=gate,
                    trace_hidden=hidden, trace_follow=follow, policy=policy, predictor=predictor,
                    n_shared=n_shared, **kw) as e:
        for _ in range(steps):
            y, ids = e.step_host(hidden, follow)
        st = e.stats()
        if kw.get("host_threads"):
            assert e.verify_last_step() == []
        resident = set(e.resident)
    _, ref_w, ref_ids = orc.or_route_trace(gate, hidden, follow, zipf, spec.top_k)
    agree = (np.sort(ids, -1) == np.sort(ref_ids.transpose(1, 0, 2), -1)).all(-1).mean()
    y_ref = orc.or_engine_reference(spec, F, 9, hidden, ids, ref_w.transpose(1, 0, 2), n_shared=n_shared)
    return y, y_ref, ids, st, resident, agree


@pytest.mark.parametrize("budget", [0.0, 0.5, 1.0])
def test_engine_decode_matches_oracle(torch_cuda, budget):
    spec = _small_spec()
    y, y_ref, ids, st, resident, agree = _run(spec, 8, budget)
    assert agree >= 0.99
    rel = np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref)
    assert rel < BF16_RTOL, rel
    # loader accounting: each (layer, routed, non-resident) expert is loaded once per step
    needed = sum(1 for l in range(spec.num_layers) for e in set(ids[l].ravel().tolist()) if (l, e) not in resident)
    assert st["ondemand_loads"] <= needed * st["steps"]
    assert st["ondemand_loads"] + st["prefetches_committed"] >= needed * st["steps"]
    if budget == 1.0:
        assert st["ondemand_loads"] == 0 and st["h2d_bytes"] == 0
    if budget == 0.0:
        assert st["resident_hits"] == 0


@pytest.mark.parametrize("policy", ["ondemand", "greedy", "fixed:2"])
def test_engine_policies_same_outputs(torch_cuda, policy):
    spec = _small_spec()
    y, y_ref, *_ = _run(spec, 8, 0.25, policy=policy)
    assert np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref) < BF16_RTOL


def test_engine_qwen3_like_shape_with_llapor(torch_cuda):
    import ctypes as C
    lib = ps.load()
    spec = _small_spec(L=6, E=128, H=256, F=128, preset="qwen3")
    m = C.c_void_p()
    ps.check(lib.ps_llapor_random(C.byref(spec), 32, 64, 32, 48, 1, C.byref(m)))
    try:
        y, y_ref, ids, st, _, agree = _run(spec, 32, 0.5, predictor=m)
    finally:
        lib.ps_llapor_free(m)
    assert agree >= 0.98
    assert np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref) < BF16_RTOL
    assert st["kernel_launches"] > 0


@pytest.mark.parametrize("budget", [1.0, 0.5])
def test_engine_prefill_chunk_uses_tcgen05_and_matches_oracle(torch_cuda, budget):
    """B > 64 switches the engine to prefill mode: gathered x_perm, exact-count
    launches, tcgen05 grouped GEMM for experts with >= 128 rows."""
    spec = _small_spec(L=3, E=8, H=256, F=512)
    y, y_ref, ids, st, _, agree = _run(spec, 512, budget, steps=1)
    assert st["tc_launches"] > 0
    assert agree >= 0.99
    assert np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref) < BF16_RTOL


@pytest.mark.parametrize("budget,policy", [(0.5, "presched"), (0.25, "fixed:2"), (0.0, "ondemand")])
def test_measured_timeline_satisfies_reference_invariants(torch_cuda, budget, policy):
    """The GPU run's own timeline (CUDA events) passes verify_timeline: serial I/O,
    one interval per transfer, every routed (layer, expert) computed exactly once,
    causality (compute after its copy), dual on-demand buffer."""
    spec = _small_spec(L=4, E=8, H=256, F=512)
    cfg = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    gate, hidden, follow, _ = ps.trace_inputs(cfg, spec, 8, 5)
    with eng.Engine(spec, cfg, budget_fraction=budget, max_batch=8, weight_seed=1, gate=gate, trace_hidden=hidden,
                    trace_follow=follow, policy=policy) as e:
        e.step_host(hidden, follow)
        events, truth, res, ls, le = e.last_timeline()
        assert e.verify_last_step() == []
        kinds = {ev[3] for ev in events}
        assert 0 in kinds and 1 in kinds  # attention-phase and expert events
        if budget < 1.0:
            assert 3 in kinds  # on-demand loads
        assert all(a <= b for a, b in zip(ls, le)) and all(le[i] <= ls[i + 1] for i in range(len(ls) - 1))
        if orc.ref_available():  # compute_metrics of the measured timeline == the reference's
            mk = max(ev[1] for ev in events)
            m, pl, gap = ps.compute_metrics(events, ls, le, mk, 8)
            sc, pl2, gap2 = orc.ref_compute_metrics(events, ls, le, mk, 8)
            assert np.array_equal([m.makespan, m.decode_latency, m.throughput_tokens_per_s, m.io_busy_fraction,
                                   m.gpu_idle_fraction], sc)
            assert np.array_equal(pl, pl2) and np.array_equal(gap, gap2)
        cost = e.calibrate()
        assert cost["t_io"] > cost["t_g"] >= 0 and cost["t_attn"] > 0


def test_engine_batch_one(torch_cuda):
    spec = _small_spec()
    y, y_ref, *_ = _run(spec, 1, 0.5)
    assert np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref) < BF16_RTOL


@pytest.mark.parametrize("B,budget", [(8, 0.5), (16, 0.0), (512, 0.5)])
def test_engine_shared_experts_deepseek_shape(torch_cuda, B, budget):
    """BASELINE config 3 (DeepSeek-V2-Lite: 64 routed top-6 + 2 shared experts): the
    shared experts run with the resident group on every token (gate weight 1), both on
    the decode GEMV path and, for a 512-token chunk, on the tcgen05 prefill path."""
    spec = _small_spec(L=3, E=64, H=256, F=256, preset="deepseek")
    y, y_ref, ids, st, resident, agree = _run(spec, B, budget, n_shared=2, steps=1)
    assert agree >= 0.98
    assert np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref) < BF16_RTOL
    if B >= 128:
        assert st["tc_launches"] > 0
    # shared experts are outside the routed budget: never loaded over PCIe
    needed = sum(1 for l in range(spec.num_layers) for e in set(ids[l].ravel().tolist()) if (l, e) not in resident)
    assert st["ondemand_loads"] + st["prefetches_committed"] >= needed
    assert st["ondemand_loads"] <= needed


@pytest.mark.parametrize("B,budget,n_shared", [(8, 0.25, 0), (16, 0.0, 0), (8, 0.2, 2)])
def test_engine_host_lane_runs_cpu_set_and_matches_oracle(torch_cuda, B, budget, n_shared):
    """Host expert lane (R5): with PCIe priced far above the host's cpu_cost, PreSched
    puts the coldest experts in cpu_set; the lane computes them from pinned host DRAM
    while the remaining loads run; outputs still match the oracle, every routed
    non-resident expert is either computed on the host or crosses PCIe, and the measured
    timeline (CPU_EXPERT events included) passes verify_timeline."""
    spec = _small_spec() if not n_shared else _small_spec(L=3, E=64, H=256, F=256, preset="deepseek")
    cost = (1000, 5, 10, 1.0, 1, 0)  # t_io, t_g, t_attn, beta, startup, alpha (us)
    y, y_ref, ids, st, resident, agree = _run(spec, B, budget, host_threads=4, cost=cost, n_shared=n_shared)
    assert agree >= 0.98
    assert np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref) < BF16_RTOL
    assert st["cpu_experts"] > 0 and st["cpu_ms_total"] > 0
    needed = sum(1 for l in range(spec.num_layers) for e in set(ids[l].ravel().tolist()) if (l, e) not in resident)
    assert st["cpu_experts"] + st["ondemand_loads"] + st["prefetches_committed"] >= needed * st["steps"]
    assert st["cpu_experts"] + st["ondemand_loads"] <= needed * st["steps"]


def test_engine_set_cost_and_calibrate_semantics(torch_cuda):
    """ps_engine_set_cost validates like CostParams::validate (t_g < t_io, ...); beta = 1e9
    keeps cpu_set empty (GPU-only executor) on a host-lane engine; calibrate refits from
    the samples since the last stats reset."""
    spec = _small_spec()
    cfg = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    gate, hidden, follow, _ = ps.trace_inputs(cfg, spec, 8, 3)
    with eng.Engine(spec, cfg, budget_fraction=0.25, max_batch=8, weight_seed=9, gate=gate, trace_hidden=hidden,
                    trace_follow=follow, host_threads=2, cost=(1000, 5, 10, 1.0, 1, 0)) as e:
        with pytest.raises(ps.capi.PsError):
            e.set_cost(10, 20, 1, 1.0, 0)  # t_g >= t_io
        e.set_cost(1000, 5, 10, 1e9, 0)
        e.step_host(hidden, follow)
        assert e.stats()["cpu_experts"] == 0 and e.stats()["ondemand_loads"] > 0
        e.set_cost(1000, 5, 10, 1.0, 1)
        e.reset_stats()
        e.step_host(hidden, follow)
        assert e.stats()["cpu_experts"] > 0
        c = e.calibrate()
        # beta is kept unless fit_cost_params found a physical fit of the lane samples
        # (timing-dependent), in which case the fitted beta is positive
        fitted = e.stats()["calibration_fit"]
        assert (c["beta"] == 1.0 or (fitted and c["beta"] > 0)) and c["startup"] >= 0 and c["t_io"] > c["t_g"]


@pytest.mark.parametrize("budget,host_threads", [(0.5, 0), (0.25, 2)])
def test_engine_replays_reference_trace_file(torch_cuda, budget, host_threads):
    """a trace written by the reference (write_trace) is read with
    ps_trace_read and its gating truth replayed through the real executor
    (ps_engine_decode_step_routed): outputs match the oracle MoE layer on the trace's own
    routing, and every (layer, expert) the trace activates is computed (loaded, host lane
    or resident) exactly as the trace's aggregate_layer_loads says."""
    t = ps.read_trace(GOLD / "ref_trace_h256.tsv")
    spec = t.spec
    H, F = spec.hidden_dim, 512
    spec.expert_bytes = 6 * H * F
    cfg = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    gate, _, _, _ = ps.trace_inputs(cfg, spec, 1, t.seed)
    kw = dict(host_threads=host_threads, cost=(1000, 5, 10, 1.0, 1, 0)) if host_threads else {}
    with eng.Engine(spec, cfg, budget_fraction=budget, max_batch=t.batch_size, weight_seed=4, gate=gate,
                    trace_hidden=t.hidden, trace_follow=np.zeros(t.hidden.shape[:2], np.uint8), **kw) as e:
        y = e.step_routed(t.hidden, t.active, t.gate_weights)
        st = e.stats()
        assert e.verify_last_step() == []
        events, truth, res, _, _ = e.last_timeline()
        L, E = spec.num_layers, spec.experts_per_layer
        want = t.tokens.sum(0)  # [L,E] aggregate_layer_loads of the trace
        assert np.array_equal(np.asarray(truth).reshape(L, E), want)
    ids = np.ascontiguousarray(t.active.transpose(1, 0, 2))
    y_ref = orc.or_engine_reference(spec, F, 4, t.hidden, ids, t.gate_weights.transpose(1, 0, 2))
    assert np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref) < BF16_RTOL
    if host_threads:
        assert st["cpu_experts"] > 0


@pytest.mark.parametrize("compress", [False, True])
def test_engine_prefill_chunk_with_host_lane(torch_cuda, compress):
    """A prefill-sized chunk (B > 64: gathered rows, exact-count tcgen05 launches) with the
    host lane taking PreSched's cpu_set (m_e in the tens of tokens per expert) and z-slab
    loads for the rest: outputs match the oracle."""
    spec = _small_spec(L=3, E=8, H=256, F=512)
    cost = (1000, 5, 10, 0.5, 1, 0)
    y, y_ref, ids, st, resident, agree = _run(spec, 256, 0.25, steps=1, host_threads=3, cost=cost,
                                              compress_host=compress)
    assert agree >= 0.99
    assert np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref) < BF16_RTOL
    assert st["cpu_experts"] > 0


def test_engine_predictor_menu_matches_reference_predict_loads(torch_cuda):
    """The reference's PredictFn menu (experiment.cpp:60-99) on the executor: the loads
    PreSched sees for layer l+1 equal predict_loads of that predictor — PERFECT = the true
    histogram of l+1, GATE = gate_reuse_predict = layer l's own histogram, STATS = the hot
    table's top-k of l+1 for every token — and the MoE outputs do not depend on it."""
    spec = _small_spec()
    cfg = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    B = 8
    gate, hidden, follow, zipf = ps.trace_inputs(cfg, spec, B, 3)
    L, E, k = spec.num_layers, spec.experts_per_layer, spec.top_k
    freq = eng.hot_table(spec, gate, hidden, follow, zipf)
    rank = np.argsort(-freq, axis=1, kind="stable").astype(np.int32)  # ties -> lower expert
    outs = {}
    for kind in ("perfect", "gate", "stats", "none"):
        with eng.Engine(spec, cfg, budget_fraction=0.0, max_batch=B, weight_seed=9, gate=gate, trace_hidden=hidden,
                        trace_follow=follow, predictor_kind=kind, stats_ranking=rank) as e:
            y, ids = e.step_host(hidden, follow)
            pred = e.last_predictions()
            _, truth, _, _, _ = e.last_timeline()
        truth = np.asarray(truth).reshape(L, E)
        outs[kind] = y
        for l in range(1, L):
            if kind == "perfect":
                np.testing.assert_array_equal(pred[l], truth[l])
            elif kind == "gate":
                np.testing.assert_array_equal(pred[l], truth[l - 1])
            elif kind == "stats":
                want = np.zeros(E, np.int32)
                want[rank[l, :k]] = B
                np.testing.assert_array_equal(pred[l], want)
            else:
                assert not pred[l].any()
    for kind in ("gate", "stats", "none"):
        np.testing.assert_array_equal(outs[kind], outs["perfect"])


@pytest.mark.parametrize("lookahead", [0, 1, 2, 3])
def test_engine_host_lane_lookahead_and_late_steal(torch_cuda, lookahead):
    """Executor extensions (perf mode, off in the reference configuration): the lookahead
    top-up of the serial channel (1: l+1, 2: l+1 and l+2, 3: l+2 only) and steal_late
    (the lane computes committed prefetches whose copies would land after it). Outputs
    still match the oracle, every routed expert is computed exactly once (verify_timeline
    conservation), and the top-up queued copies."""
    spec = _small_spec(L=5, F=2048)
    cost = (1000, 5, 10, 0.5, 1, 0)
    y, y_ref, ids, st, resident, agree = _run(spec, 8, 0.25, host_threads=4, cost=cost, lookahead=lookahead,
                                              steal_late=True, steps=3, predictor_kind="gate")
    assert agree >= 0.98
    assert np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref) < BF16_RTOL
    assert (st["lookahead_prefetches"] > 0) == (lookahead > 0)
    assert st["stolen_prefetches"] <= st["prefetches_committed"]


@pytest.mark.parametrize("preset,E,n_shared", [("mixtral", 8, 0), ("qwen3", 128, 0), ("deepseek", 64, 2)])
def test_engine_scheduling_point_graph_equals_eager(torch_cuda, monkeypatch, preset, E, n_shared):
    """The decode scheduling point replayed from CUDA graphs (default) gives bitwise the
    outputs and routing of the eager launches (PS_SCHED_GRAPH=0), over several steps
    (graph reuse) and with LLaPor predictions."""
    import ctypes as C
    lib = ps.load()
    spec = _small_spec(L=4, E=E, H=256, F=256, preset=preset)
    cfg = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    B = 8
    gate, hidden, follow, _ = ps.trace_inputs(cfg, spec, 3 * B, 5)
    pred = C.c_void_p()
    ps.check(lib.ps_llapor_random(C.byref(spec), 16, 32, 16, 24, 3, C.byref(pred)))
    outs = []
    try:
        for graph in ("1", "0"):
            monkeypatch.setenv("PS_SCHED_GRAPH", graph)
            with eng.Engine(spec, cfg, budget_fraction=0.5, max_batch=B, weight_seed=9, gate=gate,
                            trace_hidden=hidden[:B], trace_follow=follow[:B], predictor=pred,
                            n_shared=n_shared) as e:
                res = []
                for s in range(3):
                    y, ids = e.step_host(hidden[s * B:(s + 1) * B], follow[s * B:(s + 1) * B])
                    res.append((y.copy(), ids.copy()))
                outs.append(res)
    finally:
        lib.ps_llapor_free(pred)
    for (ya, ia), (yb, ib) in zip(*outs):
        assert np.array_equal(ia, ib)
        assert np.array_equal(ya, yb)
