"""TEST INFRASTRUCTURE ONLY — the CPU checker for the B200 hot path.

  * oracle.c (liboracle.so): plain-C restatement of the reference algorithms, each
    function citing /root/reference/proj file:line.
  * _ref/libprescope_ref.so: the UNMODIFIED reference sources + ref_shim.cpp, built by
    oracle/Makefile; pins the restatement and generates tests/golden/.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may import this
package. The product (paper_2509_23638_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import pathlib

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libprescope_ref.so"


class OrLoad(C.Structure):
    _fields_ = [("expert", C.c_int32), ("layer", C.c_int32), ("tokens", C.c_int32)]


class OrParams(C.Structure):
    _fields_ = [("t_io", C.c_int64), ("t_g", C.c_int64), ("t_attn", C.c_int64), ("beta", C.c_double),
                ("startup", C.c_int64), ("alpha", C.c_int64)]


class OrStats(C.Structure):
    _fields_ = [("r_hit", C.c_double), ("r_miss", C.c_double), ("window", C.c_int32)]


class OrPlanInfo(C.Structure):
    _fields_ = [("split_index", C.c_int32), ("issued_prefetches", C.c_int32), ("prefetch_from_widened", C.c_int32),
                ("n_cpu", C.c_int32), ("n_od", C.c_int32), ("n_pf", C.c_int32), ("n_sweep", C.c_int32),
                ("t_g_at_split", C.c_int64), ("t_c_at_split", C.c_int64), ("t_gap", C.c_int64),
                ("f", C.c_double), ("f_int", C.c_int32), ("xi", C.c_double),
                ("widened_window", C.c_int32), ("all_gpu_fallback", C.c_int32)]


MAXB = 8


class OrNet(C.Structure):
    _fields_ = [("H", C.c_int), ("P", C.c_int), ("E", C.c_int), ("width", C.c_int),
                ("pca_mean", C.c_void_p), ("pca_comp", C.c_void_p), ("n_blocks", C.c_int),
                ("dims", C.c_int * (MAXB + 1)), ("w", C.c_void_p * MAXB), ("b", C.c_void_p * MAXB),
                ("n_res", C.c_int), ("rw", C.c_void_p * MAXB), ("rb", C.c_void_p * MAXB),
                ("gate_w", C.c_void_p), ("gate_b", C.c_double), ("out_w", C.c_void_p), ("out_b", C.c_void_p)]


# Reference shim structs (oracle/ref_shim.cpp)
class RefSpec(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("experts", C.c_int32), ("top_k", C.c_int32), ("hidden", C.c_int32),
                ("expert_bytes", C.c_uint64), ("group_begin_middle", C.c_int32), ("group_begin_output", C.c_int32)]


class RefGen(C.Structure):
    _fields_ = [("rho", C.c_double * 3), ("kappa", C.c_double * 3), ("zipf", C.c_double * 3),
                ("noise_scale", C.c_double)]


RefParams = OrParams
RefStats = OrStats
RefPlanInfo = OrPlanInfo
RefLoad = OrLoad


class RefEvent(C.Structure):
    _fields_ = [("t_start", C.c_int64), ("t_end", C.c_int64), ("resource", C.c_int32), ("kind", C.c_int32),
                ("layer", C.c_int32), ("expert", C.c_int32), ("tokens", C.c_int32)]


class RefSimOpts(C.Structure):
    _fields_ = [("cpu_slots", C.c_int32), ("prefetch_slots", C.c_int32), ("initial_hit_rate", C.c_double),
                ("hit_window", C.c_int32)]


_oracle = None
_ref = None


def oracle_lib() -> C.CDLL:
    global _oracle
    if _oracle is None:
        if not ORACLE_SO.exists():
            raise RuntimeError(f"{ORACLE_SO} missing: run `make -C oracle`")
        _oracle = C.CDLL(str(ORACLE_SO))
        _oracle.or_topk.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p]
        _oracle.or_route.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                                     C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        _oracle.or_plan_layer.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p,
                                          C.c_int, C.POINTER(OrParams), C.POINTER(OrStats),
                                          C.POINTER(OrPlanInfo), C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p]
        _oracle.or_plan_residency.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_void_p]
        _oracle.or_llapor_forward.argtypes = [C.POINTER(OrNet), C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                              C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        _oracle.or_permute.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        _oracle.or_moe_layer.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int]
        _oracle.or_expert_ffn.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int]
        _oracle.or_init_slab.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int]
        _oracle.or_route_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                           C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int]
        _oracle.bl_moe_layer.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        _oracle.bl_init_slabs.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                          C.c_uint64, C.c_int]
    return _oracle


def ref_available() -> bool:
    return REF_SO.exists()


def ref_lib() -> C.CDLL:
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            raise RuntimeError(f"{REF_SO} missing: run `make -C oracle ref` where /root/reference exists")
        _ref = C.CDLL(str(REF_SO))
        _ref.ref_last_error.restype = C.c_char_p
        _ref.ref_llapor_load.restype = C.c_void_p
        _ref.ref_llapor_load.argtypes = [C.c_char_p]
        _ref.ref_llapor_free.argtypes = [C.c_void_p]
        _ref.ref_llapor_predict.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                            C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        _ref.ref_llapor_predict_loads.argtypes = [C.c_void_p, C.POINTER(RefGen), C.c_int, C.c_uint64, C.c_int,
                                                  C.c_void_p]
        _ref.ref_generate_trace.argtypes = [C.POINTER(RefGen), C.POINTER(RefSpec), C.c_int, C.c_uint64,
                                            C.c_void_p, C.c_void_p, C.c_void_p]
        _ref.ref_write_trace.argtypes = [C.POINTER(RefGen), C.POINTER(RefSpec), C.c_int, C.c_uint64, C.c_char_p]
        _ref.ref_export_timeline.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_char_p, C.c_int,
                                             C.POINTER(C.c_int)]
        _ref.ref_read_trace.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_uint64), C.c_void_p, C.c_int]
        _ref.ref_residency.argtypes = [C.POINTER(RefGen), C.POINTER(RefSpec), C.c_int, C.c_uint64, C.c_uint64,
                                       C.c_void_p, C.POINTER(C.c_int)]
        _ref.ref_plan_layer.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p,
                                        C.c_int, C.POINTER(RefParams), C.POINTER(RefStats),
                                        C.POINTER(RefPlanInfo), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p]
        _ref.ref_simulate.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                                      C.c_void_p, C.c_int, C.c_int, C.POINTER(RefParams), C.POINTER(RefSimOpts),
                                      C.c_void_p, C.c_int, C.POINTER(C.c_int), C.c_void_p, C.c_void_p,
                                      C.POINTER(C.c_int64), C.c_void_p]
        _ref.ref_verify_timeline.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                                             C.POINTER(RefParams), C.c_void_p, C.c_int, C.POINTER(C.c_int)]
        _ref.ref_dump_golden.argtypes = [C.c_char_p]
        _ref.ref_train_llapor.argtypes = [C.POINTER(RefGen), C.POINTER(RefSpec), C.c_int, C.c_void_p, C.c_int,
                                          C.c_int, C.c_int, C.c_uint64, C.c_char_p]
        _ref.ref_spec_preset.argtypes = [C.c_char_p, C.POINTER(RefSpec)]
        _ref.ref_desk_scale.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(RefSpec)]
        _ref.ref_topk.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_int)]
        _ref.ref_compute_metrics.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int64,
                                             C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        _ref.ref_llapor_fine_tune.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                              C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_double]
        _ref.ref_llapor_save.argtypes = [C.c_void_p, C.c_char_p]
        _ref.ref_router_inputs.argtypes = [C.POINTER(RefGen), C.POINTER(RefSpec), C.c_int, C.c_uint64, C.c_void_p,
                                           C.c_void_p, C.c_void_p]
        _ref.ref_llapor_predict_batch.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                                  C.c_void_p, C.c_int, C.c_void_p, C.c_int]
        _ref.ref_time_legs.argtypes = [C.POINTER(RefGen), C.POINTER(RefSpec), C.c_int, C.c_uint64, C.c_void_p,
                                       C.c_uint64, C.POINTER(RefParams), C.c_double, C.c_void_p, C.c_void_p]
        _ref.ref_time_schedule_pass.argtypes = [C.POINTER(RefGen), C.POINTER(RefSpec), C.c_int, C.c_uint64,
                                                C.c_uint64, C.POINTER(RefParams), C.c_int,
                                                C.POINTER(C.c_double), C.POINTER(C.c_int64)]
    return _ref


def ref_check(rc: int) -> None:
    if rc != 0:
        raise RuntimeError(f"reference rc={rc}: {ref_lib().ref_last_error().decode()}")


def ref_gen(input=(0.9, 0.0, 0.0), middle=(0.9, 0.0, 0.0), output=(0.9, 0.0, 0.0), noise=1.0) -> RefGen:
    g = RefGen()
    for i, (r, k, z) in enumerate((input, middle, output)):
        g.rho[i], g.kappa[i], g.zipf[i] = r, k, z
    g.noise_scale = noise
    return g


def ref_spec_from(spec) -> RefSpec:
    """From a product capi.ModelSpec (same field order)."""
    return RefSpec(spec.num_layers, spec.experts_per_layer, spec.top_k, spec.hidden_dim, spec.expert_bytes,
                   spec.group_begin_middle, spec.group_begin_output)


def ref_spec_preset(name: str) -> RefSpec:
    s = RefSpec()
    ref_check(ref_lib().ref_spec_preset(name.encode(), C.byref(s)))
    return s


def ref_router_inputs(gen: RefGen, spec: RefSpec, batch: int, seed: int):
    """generate_trace's router inputs (ref_shim.cpp ref_router_inputs): gate [L,E,H],
    follow [B,L] u8, zipf [L]."""
    L, E, H = spec.num_layers, spec.experts, spec.hidden
    gate = np.empty((L, E, H))
    follow = np.empty((batch, L), np.uint8)
    zipf = np.empty(L)
    ref_check(ref_lib().ref_router_inputs(C.byref(gen), C.byref(spec), batch, seed, gate.ctypes.data,
                                          follow.ctypes.data, zipf.ctypes.data))
    return gate, follow, zipf


def ref_llapor_predict_batch(handle, layer, hidden, active, gate_w, k, threads=16):
    """Reference pca_apply + forward + predict_topk for a batch of layer-(layer-1)
    features (threads over tokens) -> topk [B,k]."""
    hidden = np.ascontiguousarray(hidden, np.float64)
    active = np.ascontiguousarray(active, np.int32)
    gate_w = np.ascontiguousarray(gate_w, np.float64)
    B = hidden.shape[0]
    out = np.empty((B, k), np.int32)
    ref_check(ref_lib().ref_llapor_predict_batch(handle, layer, B, hidden.ctypes.data, active.ctypes.data,
                                                 active.shape[1], gate_w.ctypes.data, k, out.ctypes.data, threads))
    return out


REF_LEGS = ["topk_indices", "aggregate_layer_loads", "pca_apply+forward+predict_topk (input-group net)",
            "pca_apply+forward+predict_topk (middle-group net)", "build_hot_table+plan_residency",
            "schedule_layer (PreSched)", "simulate_pipeline (presched, all layers)", "generate_trace (per token)"]


def ref_time_legs(gen, spec, batch, seed, llapor, budget_bytes, params, min_seconds=0.25):
    """1-core timing of the reference's hot-path functions (ref_shim.cpp ref_time_legs):
    {leg name: (us per call, calls)}."""
    us = np.zeros(8)
    calls = np.zeros(8, np.int64)
    ref_check(ref_lib().ref_time_legs(C.byref(gen), C.byref(spec), batch, seed, llapor, budget_bytes,
                                      C.byref(RefParams(*params)), min_seconds, us.ctypes.data, calls.ctypes.data))
    return {REF_LEGS[i]: (float(us[i]), int(calls[i])) for i in range(8)}


def ref_trace(gen: RefGen, spec: RefSpec, batch: int, seed: int):
    """generate_trace flattened: hidden [B,L,H], gate_weights [B,L,E], active [B,L,k]."""
    L, E, H, K = spec.num_layers, spec.experts, spec.hidden, spec.top_k
    hidden = np.empty((batch, L, H), np.float64)
    gw = np.empty((batch, L, E), np.float64)
    act = np.empty((batch, L, K), np.int32)
    ref_check(ref_lib().ref_generate_trace(C.byref(gen), C.byref(spec), batch, seed,
                                           hidden.ctypes.data_as(C.c_void_p), gw.ctypes.data_as(C.c_void_p),
                                           act.ctypes.data_as(C.c_void_p)))
    return hidden, gw, act


def or_topk(w, k):
    w = np.ascontiguousarray(w, np.float64)
    out = np.empty(max(1, min(k, len(w))), np.int32)
    n = oracle_lib().or_topk(w.ctypes.data_as(C.c_void_p), len(w), k, out.ctypes.data_as(C.c_void_p))
    return list(out[:n])


def or_route(gate, a, zipf, follow, prev_top1, k):
    """One routing decision in f64 (workload.cpp:176-201) -> logits, weights, ids."""
    gate = np.ascontiguousarray(gate, np.float64)
    a = np.ascontiguousarray(a, np.float64)
    E, H = gate.shape
    lg, w, ids = np.empty(E), np.empty(E), np.empty(k, np.int32)
    oracle_lib().or_route(gate.ctypes.data_as(C.c_void_p), a.ctypes.data_as(C.c_void_p), E, H, float(zipf),
                          int(follow), int(prev_top1), k, lg.ctypes.data_as(C.c_void_p),
                          w.ctypes.data_as(C.c_void_p), ids.ctypes.data_as(C.c_void_p))
    return lg, w, ids


def or_route_batch(gate, hidden, follow, zipf, k, threads=1):
    """or_route_trace in one C call (OpenMP over tokens): weights [B,L,E], ids [B,L,k]."""
    gate = np.ascontiguousarray(gate, np.float64)
    hidden = np.ascontiguousarray(hidden, np.float64)
    follow = np.ascontiguousarray(follow, np.uint8)
    zipf = np.ascontiguousarray(zipf, np.float64)
    B, L, H = hidden.shape
    E = gate.shape[1]
    w = np.empty((B, L, E))
    ids = np.empty((B, L, k), np.int32)
    oracle_lib().or_route_batch(gate.ctypes.data, hidden.ctypes.data, follow.ctypes.data, zipf.ctypes.data, B, L, E,
                                H, k, w.ctypes.data, ids.ctypes.data, threads)
    return w, ids


def or_route_trace(gate, hidden, follow, zipf, k):
    """Route a whole trace (gate [L,E,H], hidden [B,L,H], follow [B,L]) in f64."""
    B, L, H = hidden.shape
    E = gate.shape[1]
    logits = np.empty((B, L, E))
    w = np.empty((B, L, E))
    ids = np.empty((B, L, k), np.int32)
    for t in range(B):
        prev = -1
        for l in range(L):
            logits[t, l], w[t, l], ids[t, l] = or_route(gate[l], hidden[t, l], zipf[l], follow[t, l], prev, k)
            prev = ids[t, l, 0]
    return logits, w, ids


def _arr_loads(items):
    a = (OrLoad * max(1, len(items)))()
    for i, (e, l, m) in enumerate(items):
        a[i] = OrLoad(e, l, m)
    return a


def _plan_common(fn, policy_kind, fixed_c, e_cur, e_next, e_next2, params, stats):
    cap = max(1, len(e_cur), len(e_next), len(e_next2))
    cpu, od, pf = (OrLoad * cap)(), (OrLoad * cap)(), (OrLoad * cap)()
    ns = max(1, len(e_cur) + len(e_next))
    sg, sc = (C.c_int64 * ns)(), (C.c_int64 * ns)()
    info = OrPlanInfo()
    rc = fn(policy_kind, fixed_c, _arr_loads(e_cur), len(e_cur), _arr_loads(e_next), len(e_next),
            _arr_loads(e_next2), len(e_next2), C.byref(OrParams(*params)), C.byref(OrStats(*stats)),
            C.byref(info), cpu, od, pf, sg, sc)
    if rc != 0:
        return rc, None
    tl = lambda a, n: [(a[i].expert, a[i].layer, a[i].tokens) for i in range(n)]  # noqa: E731
    return 0, {"split_index": info.split_index, "issued_prefetches": info.issued_prefetches,
               "prefetch_from_widened": bool(info.prefetch_from_widened), "cpu_set": tl(cpu, info.n_cpu),
               "ondemand_seq": tl(od, info.n_od), "prefetch_seq": tl(pf, info.n_pf),
               "t_g_at_split": info.t_g_at_split, "t_c_at_split": info.t_c_at_split, "t_gap": info.t_gap,
               "f": info.f, "f_int": info.f_int, "xi": info.xi, "widened_window": bool(info.widened_window),
               "all_gpu_fallback": bool(info.all_gpu_fallback),
               "sweep_gpu": list(sg[:info.n_sweep]) if policy_kind == 0 else [],
               "sweep_cpu": list(sc[:info.n_sweep]) if policy_kind == 0 else []}


POLICY_KIND = {"presched": 0, "greedy": 1, "ondemand": 2, "oracle": 4}


def _policy(policy):
    if policy.startswith("fixed:"):
        return 3, int(policy[6:])
    return POLICY_KIND[policy], 0


def or_plan_layer(e_cur, e_next, e_next2, params, stats=(1.0, 0.0, 32), policy="presched"):
    kind, c = _policy(policy)
    return _plan_common(oracle_lib().or_plan_layer, kind, c, e_cur, e_next, e_next2, params, stats)


def ref_plan_layer(e_cur, e_next, e_next2, params, stats=(1.0, 0.0, 32), policy="presched"):
    kind, c = _policy(policy)
    return _plan_common(ref_lib().ref_plan_layer, kind, c, e_cur, e_next, e_next2, params, stats)


def _triples(table):
    t = np.asarray(table)
    out = [(l, e, int(t[l, e])) for l in range(t.shape[0]) for e in range(t.shape[1]) if t[l, e] > 0]
    return np.array(out, np.int32).reshape(-1, 3)


def ref_simulate(truth, predicted, params, policy="presched", resident=None, groups=None,
                 options=(1, 8, 1.0, 32)):
    """Reference simulate_policy on dense [L,E] tables (entries > 0 only)."""
    truth = np.asarray(truth)
    L, E = truth.shape
    tr, pr = _triples(truth), _triples(predicted)
    res = np.array([(l, e) for l in range(L) for e in range(E) if resident is not None and resident[l][e]],
                   np.int32).reshape(-1, 2)
    grp = np.ascontiguousarray(groups, np.int32) if groups is not None else None
    cap = 4 * (L * E + L) + 16
    ev = (RefEvent * cap)()
    n = C.c_int()
    ls, le = np.empty(L, np.int64), np.empty(L, np.int64)
    mk = C.c_int64()
    summ = np.empty(4 * L, np.int32)
    kind, c = _policy(policy)
    rc = ref_lib().ref_simulate(L, tr.ctypes.data_as(C.c_void_p), len(tr), pr.ctypes.data_as(C.c_void_p), len(pr),
                                res.ctypes.data_as(C.c_void_p), len(res),
                                grp.ctypes.data_as(C.c_void_p) if grp is not None else None, kind, c,
                                C.byref(RefParams(*params)), C.byref(RefSimOpts(*options)), ev, cap, C.byref(n),
                                ls.ctypes.data_as(C.c_void_p), le.ctypes.data_as(C.c_void_p), C.byref(mk),
                                summ.ctypes.data_as(C.c_void_p))
    if rc != 0:
        return rc, None
    events = [(ev[i].t_start, ev[i].t_end, ev[i].resource, ev[i].kind, ev[i].layer, ev[i].expert, ev[i].tokens)
              for i in range(n.value)]
    return 0, {"events": events, "layer_start": list(map(int, ls)), "layer_end": list(map(int, le)),
               "makespan": mk.value, "plans": [tuple(map(int, summ[4 * i:4 * i + 4])) for i in range(L)]}


def ref_compute_metrics(events, layer_start, layer_end, makespan, output_tokens):
    """Reference compute_metrics -> (scalars (makespan, decode_latency, throughput,
    io_busy, gpu_idle), per_layer_latency [L], cpu_gpu_gap [L])."""
    L = len(layer_start)
    ev = (RefEvent * max(1, len(events)))(*[RefEvent(*e) for e in events])
    ls, le = np.ascontiguousarray(layer_start, np.int64), np.ascontiguousarray(layer_end, np.int64)
    sc, pl, gap = np.empty(5), np.empty(L, np.int64), np.empty(L, np.int64)
    ref_check(ref_lib().ref_compute_metrics(ev, len(events), ls.ctypes.data, le.ctypes.data, L, makespan,
                                            output_tokens, sc.ctypes.data, pl.ctypes.data, gap.ctypes.data))
    return sc, pl, gap


def ref_verify(events, truth, params, resident=None):
    truth = np.asarray(truth)
    L, E = truth.shape
    tr = _triples(truth)
    res = np.array([(l, e) for l in range(L) for e in range(E) if resident is not None and resident[l][e]],
                   np.int32).reshape(-1, 2)
    arr = (RefEvent * max(1, len(events)))(*[RefEvent(*e) for e in events])
    n = C.c_int()
    ref_check(ref_lib().ref_verify_timeline(L, tr.ctypes.data_as(C.c_void_p), len(tr), res.ctypes.data_as(C.c_void_p),
                                            len(res), C.byref(RefParams(*params)), arr, len(events), C.byref(n)))
    return n.value


def or_permute(ids, E):
    ids = np.ascontiguousarray(ids, np.int32)
    B, k = ids.shape
    off = np.empty(E + 1, np.int32)
    src = np.empty(B * k, np.int32)
    inv = np.empty(B * k, np.int32)
    oracle_lib().or_permute(ids.ctypes.data_as(C.c_void_p), B, k, E, off.ctypes.data_as(C.c_void_p),
                            src.ctypes.data_as(C.c_void_p), inv.ctypes.data_as(C.c_void_p))
    return off, src, inv


def or_moe_layer(slabs, H, F, x_bf16, ids, gate, round_h=True, threads=16):
    """slabs: list (index = expert) of uint16 arrays (or None) -> y [B,H] f32."""
    ids = np.ascontiguousarray(ids, np.int32)
    B, k = ids.shape
    E = gate.shape[1]
    ptrs = (C.c_void_p * E)(*[s.ctypes.data if s is not None else None for s in slabs])
    x = np.ascontiguousarray(x_bf16, np.uint16)
    g = np.ascontiguousarray(gate, np.float32)
    y = np.empty((B, H), np.float32)
    oracle_lib().or_moe_layer(ptrs, H, F, B, k, E, x.ctypes.data_as(C.c_void_p), ids.ctypes.data_as(C.c_void_p),
                              g.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p), int(round_h), threads)
    return y


def bl_moe_layer(slabs, H, F, x_bf16, ids, gate, threads=16):
    """CPU-baseline port (oracle/cpu_port.c): same result as or_moe_layer (f32
    accumulation), each routed expert streamed once for all its tokens."""
    lib = oracle_lib()
    ids = np.ascontiguousarray(ids, np.int32)
    B, k = ids.shape
    E = gate.shape[1]
    ptrs = (C.c_void_p * E)(*[s.ctypes.data if s is not None else None for s in slabs])
    x = np.ascontiguousarray(x_bf16, np.uint16)
    g = np.ascontiguousarray(gate, np.float32)
    y = np.empty((B, H), np.float32)
    lib.bl_moe_layer(ptrs, H, F, B, k, E, x.ctypes.data_as(C.c_void_p), ids.ctypes.data_as(C.c_void_p),
                     g.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p), threads)
    return y


def bl_init_slabs(pairs, H, F, seed, threads=16):
    """Synthetic bf16 slabs (or_init_slab values) for [(layer, expert)], one thread per slab."""
    out = [np.empty(3 * H * F, np.uint16) for _ in pairs]
    n = len(pairs)
    if n:
        ptrs = (C.c_void_p * n)(*[a.ctypes.data for a in out])
        ls = np.array([p[0] for p in pairs], np.int32)
        es = np.array([p[1] for p in pairs], np.int32)
        oracle_lib().bl_init_slabs(ptrs, ls.ctypes.data_as(C.c_void_p), es.ctypes.data_as(C.c_void_p), n, H, F,
                                   C.c_uint64(seed), threads)
    return out


def bf16_to_f32(a):
    return (np.asarray(a, np.uint16).astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(a):
    """Round-to-nearest-even (matches the device __float2bfloat16_rn for finite values)."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = u + 0x7FFF + ((u >> 16) & 1)
    return (u >> 16).astype(np.uint16)


def llapor_net_from_ckpt(path):
    """Parse an LLPC v1 checkpoint (predictor.cpp:833-864) -> (spec dict, nets dict layer -> dict)."""
    import struct
    data = pathlib.Path(path).read_bytes()
    pos = [0]

    def rd(fmt):
        v = struct.unpack_from("<" + fmt, data, pos[0])
        pos[0] += struct.calcsize("<" + fmt)
        return v if len(v) > 1 else v[0]

    def vec():
        n = rd("Q")
        v = np.frombuffer(data, np.float64, n, pos[0]).copy()
        pos[0] += 8 * n
        return v

    def mat():
        r, c = rd("i"), rd("i")
        return vec().reshape(r, c)

    def blk():
        return mat(), vec()

    assert data[:4] == b"LLPC"
    pos[0] = 4
    assert rd("I") == 1
    rd("Q")
    spec = dict(zip(["L", "E", "k"], rd("iii")))
    spec["expert_bytes"] = rd("Q")
    spec["H"], spec["gbm"], spec["gbo"] = rd("iii")
    rd("dd"), rd("ii")
    for _ in range(3):
        rd("ddiii")
    rd("ddd"), rd("i"), rd("Q")
    n = rd("I")
    nets = {}
    for i in range(n):
        net = {"target": rd("i"), "group": rd("B"), "E": rd("i")}
        rd("d")
        net["mean"] = vec()
        net["comp"] = mat()
        vec()
        rd("ii")
        net["blocks"] = [blk() for _ in range(rd("I"))]
        net["res"] = [blk() for _ in range(rd("I"))]
        net["gate_w"] = vec()
        net["gate_b"] = rd("d")
        net["out"] = blk()
        if net["blocks"]:
            nets[i] = net
    return spec, nets


def or_llapor_forward(net, hidden_prev, active_prev, gate_prev, k):
    """f64 restated LLaPor forward for one token -> (reduced, logits, topk)."""
    keep = []

    def p(a):
        a = np.ascontiguousarray(a, np.float64)
        keep.append(a)
        return a.ctypes.data

    s = OrNet()
    s.H = net["comp"].shape[1]
    s.P = net["comp"].shape[0]
    s.E = net["E"]
    s.pca_mean, s.pca_comp = p(net["mean"]), p(net["comp"])
    s.n_blocks = len(net["blocks"])
    s.dims[0] = net["blocks"][0][0].shape[1]
    for j, (w, b) in enumerate(net["blocks"]):
        s.dims[j + 1] = w.shape[0]
        s.w[j], s.b[j] = p(w), p(b)
    s.width = s.dims[s.n_blocks]
    s.n_res = len(net["res"])
    for j, (w, b) in enumerate(net["res"]):
        s.rw[j], s.rb[j] = p(w), p(b)
    s.gate_w = p(net["gate_w"] if len(net["gate_w"]) else np.zeros(1))
    s.gate_b = net["gate_b"]
    s.out_w, s.out_b = p(net["out"][0]), p(net["out"][1])
    red = np.empty(s.P)
    lg = np.empty(s.E)
    top = np.empty(k, np.int32)
    act = np.ascontiguousarray(active_prev, np.int32)
    rc = oracle_lib().or_llapor_forward(C.byref(s), p(hidden_prev), act.ctypes.data, len(act), p(gate_prev), k,
                                        red.ctypes.data, lg.ctypes.data, top.ctypes.data)
    assert rc == 0
    return red, lg, top


def or_init_slab(H, F, seed, layer, expert):
    out = np.empty(3 * H * F, np.uint16)
    oracle_lib().or_init_slab(out.ctypes.data, H, F, seed, layer, expert)
    return out


def or_engine_reference(spec, F, weight_seed, hidden, ids, weights, threads=16, n_shared=0):
    """Per-layer MoE outputs the decode engine must produce: hidden [B,L,H] f64 (trace
    order), ids [L,B,k] (routing to evaluate), weights [L,B,E] (full-softmax gate
    weights). x is the bf16 rounding of hidden (the FFN input). Returns y [L,B,H].
    n_shared > 0: DeepSeek-style shared experts (hash-keyed as experts E..E+S-1, gate
    weight 1, every token) are added to each token's output."""
    B, L, H = hidden.shape
    E = spec.experts_per_layer
    S = n_shared
    y = np.empty((L, B, H), np.float32)
    for l in range(L):
        used = set(int(e) for e in np.unique(ids[l])) | set(range(E, E + S))
        slabs = [or_init_slab(H, F, weight_seed, l, e) if e in used else None for e in range(E + S)]
        x = f32_to_bf16(hidden[:, l, :].astype(np.float32))
        ids_l, w_l = ids[l], weights[l].astype(np.float32)
        if S:
            ids_l = np.concatenate([ids_l, np.broadcast_to(np.arange(E, E + S, dtype=np.int32), (B, S))], 1)
            w_l = np.concatenate([w_l, np.ones((B, S), np.float32)], 1)
        y[l] = or_moe_layer(slabs, H, F, x, ids_l, w_l, True, threads)
    return y
