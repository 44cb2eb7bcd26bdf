"""B200-native PreScope MoE-inference hot path (C++/CUDA library behind a C ABI).

This package is the Python-side mirror of the reference's operator API for the hot
path (namespace prescope, /root/reference/proj/include/prescope/*.hpp): thin wrappers
over include/ps_api.h via ctypes. The product is libprescope_b200.so; nothing here
computes anything itself, and every wrapper raises if the library is missing.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import capi
from .capi import check, load

__all__ = ["capi", "load", "check", "spec_preset", "desk_scale", "ffn_dim", "trace_inputs", "plan_layer",
           "parse_policy", "simulate", "verify_timeline", "compute_metrics", "plan_residency", "Plan", "TraceGenConfig",
           "GROUP_DEFAULT_GEN", "Trace", "read_trace", "write_trace"]

# Default generator knobs of the benchmark workloads:
# input/output {rho .9, kappa .5, zipf .5}; middle {rho .95, kappa .6, zipf 1.0}; noise 1.
GROUP_DEFAULT_GEN = {"input": (0.9, 0.5, 0.5), "middle": (0.95, 0.6, 1.0), "output": (0.9, 0.5, 0.5),
                     "noise": 1.0}


def spec_preset(name: str) -> capi.ModelSpec:
    s = capi.ModelSpec()
    check(load().ps_spec_preset(name.encode(), C.byref(s)))
    return s


def desk_scale(full: capi.ModelSpec | str, layers: int, experts: int, hidden: int) -> capi.ModelSpec:
    if isinstance(full, str):
        full = spec_preset(full)
    s = capi.ModelSpec()
    check(load().ps_desk_scale(C.byref(full), layers, experts, hidden, C.byref(s)))
    return s


def ffn_dim(spec: capi.ModelSpec) -> int:
    f = C.c_int()
    check(load().ps_spec_ffn_dim(C.byref(spec), C.byref(f)))
    return f.value


def TraceGenConfig(input=(0.9, 0.0, 0.0), middle=(0.9, 0.0, 0.0), output=(0.9, 0.0, 0.0), noise=1.0):
    """prescope::TraceGenConfig (workload.hpp:80-88): (rho, kappa, zipf_s) per group."""
    c = capi.TraceGenConfig()
    for name, v in (("input", input), ("middle", middle), ("output", output)):
        g = getattr(c, name)
        g.rho, g.kappa, g.zipf_s = v
    c.noise_scale = noise
    return c


def trace_inputs(cfg, spec: capi.ModelSpec, batch: int, seed: int, want_gate=True):
    """Routing inputs of generate_trace (workload.cpp:139-219) without the routing:
    gate [L,E,H] f64, hidden [B,L,H] f64, follow [B,L] u8, zipf per layer [L] f64."""
    L, E, H = spec.num_layers, spec.experts_per_layer, spec.hidden_dim
    gate = np.empty((L, E, H), np.float64) if want_gate else None
    hidden = np.empty((batch, L, H), np.float64)
    follow = np.empty((batch, L), np.uint8)
    zipf = np.empty(L, np.float64)
    ptr = lambda a: a.ctypes.data_as(C.c_void_p) if a is not None else None  # noqa: E731
    check(load().ps_trace_inputs(C.byref(cfg), C.byref(spec), batch, seed, ptr(gate), ptr(hidden), ptr(follow),
                                 ptr(zipf)))
    return gate, hidden, follow, zipf


@dataclass
class Trace:
    """prescope::Trace (workload.hpp:47-66) as dense arrays, index [token, layer]:
    hidden [B,L,H] f64, gate_weights [B,L,E] f64, active [B,L,k] i32 (weight-desc),
    tokens [B,L,E] i32 (tokens_per_expert; 0 = absent)."""
    spec: capi.ModelSpec
    batch_size: int
    seed: int
    hidden: np.ndarray
    gate_weights: np.ndarray
    active: np.ndarray
    tokens: np.ndarray
    checksum: int = 0


def read_trace(path) -> Trace:
    """read_trace (workload.cpp:409-436): raises RuntimeError on TraceFormatError /
    TraceChecksumError / I/O failure, ValueError on an invalid spec."""
    lib = load()
    h = C.c_void_p()
    check(lib.ps_trace_read(str(path).encode(), C.byref(h)))
    try:
        spec, b, seed, cs = capi.ModelSpec(), C.c_int32(), C.c_uint64(), C.c_uint64()
        check(lib.ps_trace_shape(h, C.byref(spec), C.byref(b), C.byref(seed), C.byref(cs)))
        B, L, E, H, k = b.value, spec.num_layers, spec.experts_per_layer, spec.hidden_dim, spec.top_k
        hid = np.empty((B, L, H), np.float64)
        gw = np.empty((B, L, E), np.float64)
        act = np.empty((B, L, k), np.int32)
        tok = np.empty((B, L, E), np.int32)
        check(lib.ps_trace_arrays(h, *(a.ctypes.data_as(C.c_void_p) for a in (hid, gw, act, tok))))
    finally:
        lib.ps_trace_free(h)
    return Trace(spec, B, seed.value, hid, gw, act, tok, cs.value)


def write_trace(trace: Trace, path) -> None:
    """write_trace (workload.cpp:391-407), byte-identical to the reference's writer."""
    arrs = [np.ascontiguousarray(trace.hidden, np.float64), np.ascontiguousarray(trace.gate_weights, np.float64),
            np.ascontiguousarray(trace.active, np.int32), np.ascontiguousarray(trace.tokens, np.int32)]
    check(load().ps_trace_write(str(path).encode(), C.byref(trace.spec), trace.batch_size, trace.seed,
                                *(a.ctypes.data_as(C.c_void_p) for a in arrs)))


def parse_policy(text: str) -> capi.Policy:
    p = capi.Policy()
    check(load().ps_policy_parse(text.encode(), C.byref(p)))
    return p


def _loads(items, default_layer=0):
    arr = (capi.ExpertLoad * max(1, len(items)))()
    for i, it in enumerate(items):
        e, layer, tokens = it
        arr[i] = capi.ExpertLoad(e, layer, tokens, capi.PS_LOC_HOST)
    return arr


@dataclass
class Plan:
    split_index: int
    issued_prefetches: int
    prefetch_from_widened: bool
    cpu_set: list
    ondemand_seq: list
    prefetch_seq: list
    t_g_at_split: int
    t_c_at_split: int
    t_gap: int
    f: float
    f_int: int
    xi: float
    widened_window: bool
    all_gpu_fallback: bool
    sweep_gpu: list = field(default_factory=list)
    sweep_cpu: list = field(default_factory=list)


def plan_layer(e_cur, e_next, e_next2, params, stats=(1.0, 0.0, 32), policy="presched") -> Plan:
    """prescope::plan_layer (scheduler.cpp:271-282). Lists of (expert, layer, tokens);
    params (t_io, t_g, t_attn, beta, startup, alpha)."""
    lib = load()
    cur, nxt, nxt2 = _loads(e_cur), _loads(e_next), _loads(e_next2)
    inp = capi.LayerInputs(cur, len(e_cur), nxt, len(e_next), nxt2, len(e_next2), capi.CostParams(*params),
                           capi.HitStats(*stats))
    cap = max(1, len(e_cur), len(e_next), len(e_next2))
    cpu, od, pf = (capi.ExpertLoad * cap)(), (capi.ExpertLoad * cap)(), (capi.ExpertLoad * cap)()
    ns = max(1, len(e_cur) + len(e_next))
    sg, sc = (C.c_int64 * ns)(), (C.c_int64 * ns)()
    plan = capi.LayerPlan()
    plan.cpu_set, plan.ondemand_seq, plan.prefetch_seq = cpu, od, pf
    plan.trace.sweep_gpu, plan.trace.sweep_cpu = sg, sc
    pol = parse_policy(policy) if isinstance(policy, str) else policy
    check(lib.ps_presched_plan(C.byref(inp), pol, C.byref(plan)))
    tl = lambda a, n: [(a[i].expert, a[i].layer, a[i].tokens) for i in range(n)]  # noqa: E731
    t = plan.trace
    return Plan(plan.split_index, plan.issued_prefetches, bool(plan.prefetch_from_widened),
                tl(cpu, plan.n_cpu), tl(od, plan.n_ondemand), tl(pf, plan.n_prefetch), t.t_g_at_split,
                t.t_c_at_split, t.t_gap, t.f, t.f_int, t.xi, bool(t.widened_window), bool(t.all_gpu_fallback),
                list(sg[:t.n_sweep]), list(sc[:t.n_sweep]))


def _instance(truth, predicted, resident=None, groups=None):
    truth = np.ascontiguousarray(truth, np.int32)
    predicted = np.ascontiguousarray(predicted, np.int32)
    L, E = truth.shape
    res = np.ascontiguousarray(resident if resident is not None else np.zeros((L, E)), np.uint8)
    keep = [truth, predicted, res]
    inst = capi.PipelineInstance(L, E, truth.ctypes.data_as(C.POINTER(C.c_int32)),
                                 predicted.ctypes.data_as(C.POINTER(C.c_int32)),
                                 res.ctypes.data_as(C.POINTER(C.c_uint8)), None)
    if groups is not None:
        g = np.ascontiguousarray(groups, np.int32)
        keep.append(g)
        inst.groups = g.ctypes.data_as(C.POINTER(C.c_int32))
    return inst, keep


def simulate(truth, predicted, params, policy="presched", resident=None, groups=None, options=(1, 8, 1.0, 32),
             plan_fn=None):
    """prescope::simulate_policy / simulate_pipeline (simulator.cpp:61-252) on dense
    [L,E] token tables. Returns dict(events, layer_start, layer_end, makespan, plans)."""
    lib = load()
    inst, keep = _instance(truth, predicted, resident, groups)
    L = inst.num_layers
    cap = 4 * (L * inst.experts + L) + 16
    ev = (capi.TimelineEvent * cap)()
    ls, le = (C.c_int64 * L)(), (C.c_int64 * L)()
    summ = (C.c_int32 * (4 * L))()
    tl = capi.Timeline(ev, cap, 0, ls, le, 0, summ)
    pol = parse_policy(policy) if isinstance(policy, str) else policy
    cb = capi.PLAN_FN(plan_fn) if plan_fn else C.cast(None, capi.PLAN_FN)
    check(lib.ps_simulate_pipeline(C.byref(inst), pol, cb, None, C.byref(capi.CostParams(*params)),
                                   C.byref(capi.SimOptions(*options)), C.byref(tl)))
    events = [(ev[i].t_start, ev[i].t_end, ev[i].resource, ev[i].kind, ev[i].layer, ev[i].expert, ev[i].tokens)
              for i in range(tl.n_events)]
    del keep
    return {"events": events, "layer_start": list(ls), "layer_end": list(le), "makespan": tl.makespan,
            "plans": [tuple(summ[4 * i:4 * i + 4]) for i in range(L)]}


def verify_timeline(events, truth, params, resident=None):
    """prescope::verify_timeline (simulator.cpp:323-394) -> list of violation messages."""
    lib = load()
    inst, keep = _instance(truth, np.zeros_like(np.asarray(truth)), resident)
    arr = (capi.TimelineEvent * max(1, len(events)))(*[capi.TimelineEvent(*e) for e in events])
    n = C.c_int()
    buf = C.create_string_buffer(1 << 16)
    check(lib.ps_verify_timeline(arr, len(events), C.byref(inst), C.byref(capi.CostParams(*params)), C.byref(n),
                                 buf, len(buf)))
    del keep
    msgs = [m for m in buf.value.decode().split("\n") if m]
    assert len(msgs) == n.value or len(buf.value) >= len(buf) - 1
    return msgs


def compute_metrics(events, layer_start, layer_end, makespan, output_tokens):
    """compute_metrics (simulator.cpp:396-426) via ps_compute_metrics -> (ps_metrics,
    per_layer_latency [L], cpu_gpu_gap [L]). events: (t_start, t_end, resource, kind,
    layer, expert, tokens) tuples; makespan: the timeline's own field."""
    L = len(layer_start)
    arr = (capi.TimelineEvent * max(1, len(events)))(*[capi.TimelineEvent(*e) for e in events])
    ls, le = np.ascontiguousarray(layer_start, np.int64), np.ascontiguousarray(layer_end, np.int64)
    m = capi.Metrics()
    pl, gap = np.empty(L, np.int64), np.empty(L, np.int64)
    check(load().ps_compute_metrics(arr, len(events), ls.ctypes.data_as(C.c_void_p), le.ctypes.data_as(C.c_void_p),
                                    L, int(makespan), int(output_tokens), C.byref(m), pl.ctypes.data_as(C.c_void_p),
                                    gap.ctypes.data_as(C.c_void_p)))
    return m, pl, gap


def plan_residency(freq, budget_bytes: int, expert_bytes: int):
    """prescope::plan_residency over a [L,E] frequency table (predictor.cpp:405-433)."""
    f = np.ascontiguousarray(freq, np.int64)
    L, E = f.shape
    out = np.empty((L * E, 2), np.int32)
    n = C.c_int()
    check(load().ps_plan_residency(f.ctypes.data_as(C.c_void_p), L, E, budget_bytes, expert_bytes,
                                   out.ctypes.data_as(C.c_void_p), C.byref(n)))
    return [tuple(map(int, r)) for r in out[:n.value]]
