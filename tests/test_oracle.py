"""Pins the CPU oracle (oracle/oracle.c) to the reference: golden vectors, KATs and the
UNMODIFIED reference compiled in oracle/_ref. The oracle is only trusted after this."""
import ctypes as C
import json

import numpy as np
import pytest

import oracle as orc
import paper_2509_23638_b200 as ps
from conftest import GOLDEN

needs_ref = pytest.mark.skipif(not orc.ref_available(), reason="oracle/_ref not built")


def test_topk_kat():
    # test_workload.cpp:187-192
    w = [0.1, 0.4, 0.4, 0.05, 0.05]
    assert orc.or_topk(w, 3) == [1, 2, 0]
    assert orc.or_topk(w, 10) == [1, 2, 0, 3, 4]


def test_router_restatement_matches_reference_trace_bit_exact():
    """or_route on the product's RNG replay (gate, hidden, follow) reproduces the
    reference trace's f64 gate weights and top-k exactly (desk config[0])."""
    d = np.load(GOLDEN / "desk_trace_c0.npz")
    spec = ps.desk_scale("mixtral", 4, 8, 16)
    cfg = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    gate, hidden, follow, zipf = ps.trace_inputs(cfg, spec, 32, 0)
    assert np.array_equal(hidden, d["hidden"])
    _, w, ids = orc.or_route_trace(gate, hidden, follow, zipf, spec.top_k)
    assert np.array_equal(w, d["gate_weights"])
    assert np.array_equal(ids, d["active"])


def test_trace_fingerprints_first_steps():
    """SURVEY.md §8c fingerprints: first (token 0) top-k at layers 0 and 1."""
    for fp in json.loads((GOLDEN / "trace_fingerprints.json").read_text()):
        name, L, E, H = fp["spec"]
        spec = ps.desk_scale(name, L, E, H)
        knobs = tuple(fp["knobs"])
        cfg = ps.TraceGenConfig(knobs, knobs, knobs)
        gate, hidden, follow, zipf = ps.trace_inputs(cfg, spec, fp["batch"], fp["seed"])
        _, _, ids = orc.or_route_trace(gate, hidden[:1], follow[:1], zipf, spec.top_k)
        assert ids[0, 0].tolist() == fp["top0"] and ids[0, 1].tolist() == fp["top1"]


def _plan_eq(a, b):
    return all(a[k] == b[k] for k in a)


def test_presched_restatement_matches_golden_cases():
    data = json.loads((GOLDEN / "presched_cases.json").read_text())
    for c in data["cases"]:
        for pol, ref in c["plans"].items():
            rc, got = orc.or_plan_layer([tuple(x) for x in c["e_cur"]], [tuple(x) for x in c["e_next"]],
                                        [tuple(x) for x in c["e_next2"]], tuple(c["params"]), tuple(c["stats"]),
                                        pol)
            assert rc == 0
            ref = dict(ref)
            for key in ("cpu_set", "ondemand_seq", "prefetch_seq"):
                ref[key] = [tuple(x) for x in ref[key]]
            assert _plan_eq(ref, got), (pol, c)
    for b in data["invalid"]:
        rc, _ = orc.or_plan_layer([tuple(x) for x in b["e_cur"]], [], [], tuple(b["params"]))
        assert rc == b["rc"] == 1


def test_presched_kats_from_reference_tests():
    # test_scheduler.cpp:129-140: split = 1
    assert orc.or_plan_layer([(0, 0, 3), (1, 0, 50)], [], [], (2, 1, 3, 1.0, 1, 0))[1]["split_index"] == 1
    # test_scheduler.cpp:186-212: widened window, f = 1.8, |f| = 2, seq [e2, e1]
    rc, p = orc.or_plan_layer([(0, 0, 5)], [], [(1, 2, 2), (2, 2, 50)], (5, 2, 3, 1.0, 1, 0))
    assert p["split_index"] == 1 and p["widened_window"] and p["prefetch_from_widened"]
    assert p["f"] == pytest.approx(1.8) and p["f_int"] == 2
    assert [e[0] for e in p["prefetch_seq"]] == [2, 1]
    # test_scheduler.cpp:214-228: fallback to split 0
    rc, p = orc.or_plan_layer([(0, 0, 100)], [], [], (5, 2, 3, 1.0, 1, 0))
    assert p["split_index"] == 0 and p["all_gpu_fallback"]
    rc, p = orc.or_plan_layer([(0, 0, 2)], [], [], (5, 2, 3, 1.0, 1, 0))
    assert not p["all_gpu_fallback"] and p["split_index"] == 1
    # test_scheduler.cpp:270-287: greedy tie-break prefers fewer GPU loads
    assert orc.or_plan_layer([(0, 0, 3), (1, 0, 5), (2, 0, 6)], [], [], (4, 2, 0, 1.0, 0, 0),
                             policy="greedy")[1]["split_index"] == 2
    assert orc.or_plan_layer([(0, 0, 3), (1, 0, 7), (2, 0, 8)], [], [], (4, 2, 0, 1.0, 0, 0),
                             policy="greedy")[1]["split_index"] == 2


def test_presched_golden_decision_traces():
    """SURVEY.md §8c decision-trace KATs: layer-0 plans of the golden instances."""
    scen = {s["id"]: s for s in json.loads((GOLDEN / "golden_scenarios.json").read_text())}
    p0 = scen["prefetch-case4-crosslayer"]["presched_plans"][0]
    assert p0["split_index"] == 2 and p0["t_gap"] == 17 and p0["f_int"] == 1 and p0["xi"] == 20.0
    p0 = scen["greedy-case2-cpu-bound"]["presched_plans"][0]
    assert p0["split_index"] == 1 and p0["t_gap"] == 16 and p0["xi"] == 19.0
    assert scen["greedy-case2-cpu-bound"]["presched_timeline"]["makespan"] == 55


@needs_ref
def test_presched_restatement_vs_reference_random():
    rng = np.random.default_rng(5)
    for it in range(2000):
        def lst(layer, lo, hi):
            n = int(rng.integers(lo, hi + 1))
            v = sorted([(e, layer, int(rng.integers(1, 21))) for e in range(n)], key=lambda x: (x[2], x[0]))
            return v
        t_io = int(rng.integers(5, 31))
        params = (t_io, int(rng.integers(1, min(t_io - 1, 8) + 1)), int(rng.integers(0, 11)),
                  float(rng.uniform(0.5, 4.0)), int(rng.integers(0, 6)), int(rng.integers(0, 21)))
        h = float(rng.random())
        cur, nxt, nxt2 = lst(0, 1, 8), lst(1, 0, 8), lst(2, 0, 8)
        for pol in ("presched", "greedy", "ondemand", "fixed:1"):
            assert orc.or_plan_layer(cur, nxt, nxt2, params, (h, 1 - h, 32), pol) == \
                orc.ref_plan_layer(cur, nxt, nxt2, params, (h, 1 - h, 32), pol)


def test_residency_kat():
    # acceptance.cpp:345-365 / test_predictor.cpp:225-242: 1 GiB at 336 MiB -> 3 residents, monotone
    freq = np.arange(32 * 8, dtype=np.int64).reshape(32, 8)[::-1].copy()
    import ctypes as C
    out = np.empty((256, 2), np.int32)
    n = orc.oracle_lib().or_plan_residency(freq.ctypes.data, 32, 8, 1 << 30, 336 << 20, out.ctypes.data)
    assert n == 3
    prev = 0
    for mib in range(0, 8193, 128):
        m = orc.oracle_lib().or_plan_residency(freq.ctypes.data, 32, 8, mib << 20, 336 << 20, out.ctypes.data)
        assert m >= prev
        prev = m


@needs_ref
def test_residency_vs_reference():
    import ctypes as C
    spec = ps.desk_scale("mixtral", 4, 8, 16)
    cfg = ps.TraceGenConfig((0.9, 0.0, 0.0), (0.9, 0.0, 1.0), (0.9, 0.0, 0.0))
    gate, hidden, follow, zipf = ps.trace_inputs(cfg, spec, 16, 21)
    _, _, ids = orc.or_route_trace(gate, hidden, follow, zipf, spec.top_k)
    freq = np.zeros((4, 8), np.int64)
    for l in range(4):
        for e in ids[:, l].ravel():
            freq[l, e] += 1
    for budget in (0, 1 << 30, 5 << 30, 64 << 30):
        out = np.empty((32, 2), np.int32)
        n = orc.oracle_lib().or_plan_residency(freq.ctypes.data, 4, 8, budget, spec.expert_bytes, out.ctypes.data)
        ref = np.empty((32, 2), np.int32)
        nr = C.c_int()
        orc.ref_check(orc.ref_lib().ref_residency(C.byref(orc.ref_gen((0.9, 0.0, 0.0), (0.9, 0.0, 1.0),
                                                                      (0.9, 0.0, 0.0))),
                                                  C.byref(orc.ref_spec_from(spec)), 16, 21, budget,
                                                  ref.ctypes.data, C.byref(nr)))
        assert n == nr.value and np.array_equal(out[:n], ref[:n])


def test_llapor_restatement_matches_reference_fixture():
    spec_d, nets = orc.llapor_net_from_ckpt(GOLDEN / "llapor_desk.llpc")
    exp = np.load(GOLDEN / "llapor_desk_expected.npz")
    for i, (t, l) in enumerate(exp["rows"]):
        net = nets[int(l)]
        red, lg, top = orc.or_llapor_forward(net, exp["hidden"][t, l - 1], exp["active"][t, l - 1],
                                             exp["gate_weights"][t, l - 1], spec_d["k"])
        np.testing.assert_allclose(lg, exp["logits"][i], rtol=1e-12, atol=1e-12)
        assert list(top) == list(exp["topk"][i])


def test_permute_restatement_order():
    ids = np.array([[3, 1], [1, 0], [3, 2], [0, 1]], np.int32)
    off, src, inv = orc.or_permute(ids, 4)
    assert off.tolist() == [0, 2, 5, 6, 8]
    # expert 0: tokens 1,3 ; expert 1: tokens 0,1,3 ; expert 2: token 2 ; expert 3: tokens 0,2
    assert [s // 2 for s in src] == [1, 3, 0, 1, 3, 2, 0, 2]
    assert all(src[inv[i]] == i for i in range(8))


def test_expert_ffn_oracle_linear_in_down_weights():
    """SwiGLU oracle property: scaling x by 0 gives 0; a tiny FFN checked in numpy."""
    H, F = 16, 32
    slab = orc.or_init_slab(H, F, 1, 0, 0)
    x = orc.f32_to_bf16(np.linspace(-1, 1, H).astype(np.float32))[None]
    import ctypes as C
    y = np.empty((1, H), np.float32)
    orc.oracle_lib().or_expert_ffn(slab.ctypes.data, H, F, 1, x.ctypes.data, y.ctypes.data, 0)
    w = orc.bf16_to_f32(slab).astype(np.float64)
    wg, wu, wd = w[:F * H].reshape(F, H), w[F * H:2 * F * H].reshape(F, H), w[2 * F * H:].reshape(H, F)
    xf = orc.bf16_to_f32(x[0]).astype(np.float64)
    g, u = wg @ xf, wu @ xf
    ref = wd @ (g / (1 + np.exp(-g)) * u)
    np.testing.assert_allclose(y[0], ref, rtol=1e-5, atol=1e-7)


@needs_ref
def test_near_tie_list_regenerates_from_reference():
    """tests/golden/near_ties.json (the list test_route_topk_parity accepts top-k
    mismatches from) is what make_near_ties.py derives from oracle/_ref today."""
    import sys
    sys.path.insert(0, str(GOLDEN))
    import make_near_ties
    fresh = make_near_ties.generate()
    committed = json.loads((GOLDEN / "near_ties.json").read_text())
    assert fresh == json.loads(json.dumps(committed))


@needs_ref
@pytest.mark.parametrize("preset,E,H,p_in,p_mid", [("mixtral", 8, 4096, 256, 512), ("qwen3", 128, 2048, 128, 256)])
def test_llapor_oracle_full_shape_equals_reference(tmp_path, preset, E, H, p_in, p_mid):
    """The f64 LLaPor restatement at paper dims (multi-chunk PCA, E=128 outputs) equals
    the reference's load_checkpoint + pca_apply + forward + predict_topk bit for bit."""
    from oracle.llpc import random_nets, write_llpc
    spec = ps.desk_scale(preset, 3, E, H)
    k = spec.top_k
    path = tmp_path / "n.llpc"
    write_llpc(path, spec, random_nets(spec, p_in, p_mid, 32, 48, seed=1))
    _, onets = orc.llapor_net_from_ckpt(path)
    h = orc.ref_lib().ref_llapor_load(str(path).encode())
    assert h
    rng = np.random.default_rng(2)
    try:
        for l in (1, 2):
            for _ in range(4):
                x = rng.standard_normal(H)
                act = rng.choice(E, k, replace=False).astype(np.int32)
                gw = np.exp(rng.standard_normal(E))
                gw /= gw.sum()
                P = p_mid if l == 1 else p_in
                red, lg, top = np.empty(P), np.empty(E), np.empty(k, np.int32)
                orc.ref_check(orc.ref_lib().ref_llapor_predict(h, l, x.ctypes.data, act.ctypes.data, k, gw.ctypes.data,
                                                               k, red.ctypes.data, lg.ctypes.data, top.ctypes.data))
                r2, lg2, top2 = orc.or_llapor_forward(onets[l], x, act, gw, k)
                assert np.array_equal(red, r2) and np.array_equal(lg, lg2) and np.array_equal(top, top2)
    finally:
        orc.ref_lib().ref_llapor_free(h)


@needs_ref
@pytest.mark.parametrize("preset,L,E,H,B,seed", [("mixtral", 4, 8, 16, 32, 0), ("qwen3", 3, 128, 2048, 8, 5),
                                                 ("mixtral", None, None, None, 4, 1000)])
def test_reference_router_inputs_reproduce_generate_trace(preset, L, E, H, B, seed):
    """bench.py's reference arm routes with or_route_batch on ref_router_inputs (the
    reference engine's draws replayed in the shim) and the reference trace's hidden
    states: bit-exact gate weights / top-k of generate_trace itself."""
    spec = orc.ref_spec_preset(preset)
    if L is not None:
        orc.ref_check(orc.ref_lib().ref_desk_scale(preset.encode(), L, E, H, C.byref(spec)))
    rg = orc.ref_gen(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    hidden, gw, act = orc.ref_trace(rg, spec, B, seed)
    gate, follow, zipf = orc.ref_router_inputs(rg, spec, B, seed)
    w, ids = orc.or_route_batch(gate, hidden, follow, zipf, spec.top_k, threads=4)
    assert np.array_equal(w, gw) and np.array_equal(ids, act)


def test_cpu_port_moe_layer_matches_oracle():
    """The CPU-baseline port (cpu_port.c: each expert streamed once, f32 AVX-512
    accumulation) computes the oracle's MoE layer within fp32 rounding."""
    rng = np.random.default_rng(0)
    for H, F, E, k, B in ((256, 512, 8, 2, 16), (64, 96, 4, 2, 5), (512, 1408, 64, 6, 40)):
        ids = np.stack([rng.choice(E, k, replace=False) for _ in range(B)]).astype(np.int32)
        g = np.exp(rng.standard_normal((B, E)))
        g = (g / g.sum(1, keepdims=True)).astype(np.float32)
        x = orc.f32_to_bf16((rng.standard_normal((B, H)) / np.sqrt(H)).astype(np.float32))
        slabs = orc.bl_init_slabs([(0, e) for e in range(E)], H, F, 3, 4)
        assert all(np.array_equal(slabs[e], orc.or_init_slab(H, F, 3, 0, e)) for e in (0, E - 1))
        y = orc.bl_moe_layer(slabs, H, F, x, ids, g, 4)
        y2 = orc.or_moe_layer(slabs, H, F, x, ids, g, True, 4)
        assert np.linalg.norm(y - y2) / np.linalg.norm(y2) < 1e-4
