"""Regenerates the committed golden fixtures from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libprescope_ref.so, built from
/root/reference/proj/src by `make -C oracle ref`):

    python tests/golden/make_golden.py

Outputs (all small, committed):
  golden_scenarios.json   six hand-derived timelines of golden.cpp:61-234, the
                          reference replay of each, and the PreSched plans/timeline
                          on each instance (test_golden.cpp pins the makespans).
  trace_fingerprints.json FNV-1a body checksums of write_trace (workload.cpp:290-406)
                          for the three configs of SURVEY.md §8c + first top-k steps.
  desk_trace_c0.npz       BASELINE config[0]: desk_scale(mixtral,4,8,16), B=32, seed 0,
                          default benchmark knobs: hidden / gate_weights / active.
  presched_cases.json     1000 random LayerInputs x 4 policies with reference plans.
  sim_cases.json          300 random multi-layer PipelineInstances with reference
                          timelines (PreSched, greedy, on-demand, fixed:2).
  llapor_desk.llpc        LLaPor trained by the reference on config[0]-shaped traces
                          (make_llapor + train + save_checkpoint).
  llapor_desk_expected.npz reference pca/logits/top-k for 64 (token, layer) features.
  ref_trace_desk.tsv      a trace file written by the reference's write_trace
                          (workload.cpp:391-407): desk_scale(mixtral,4,8,16), B=3, seed 17,
                          knobs (rho .9, kappa .3, zipf .5) — read/re-write parity.
  ref_trace_h256.tsv      reference trace desk_scale(mixtral,4,8,256), B=8, seed 23,
                          benchmark knobs — replayed through the GPU executor
                          (ps_engine_decode_step_routed, tests/test_gpu_engine.py).
"""
from __future__ import annotations

import ctypes as C
import json
import pathlib
import random
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle as orc  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent
DEFAULT = dict(input=(0.9, 0.5, 0.5), middle=(0.95, 0.6, 1.0), output=(0.9, 0.5, 0.5))


def desk_spec(name, L, E, H):
    s = orc.RefSpec()
    orc.ref_check(orc.ref_lib().ref_desk_scale(name.encode(), L, E, H, C.byref(s)))
    return s


def fingerprints():
    out = []
    cases = [(("mixtral", 6, 8, 16), (0.9, 0.3, 0.5), 12, 17),
             (("mixtral", 4, 8, 16), (0.95, 1.0, 0.0), 48, 13),
             (("mixtral", 4, 8, 16), (0.85, 0.4, 0.7), 8, 41)]
    for (name, L, E, H), knobs, B, seed in cases:
        spec = desk_spec(name, L, E, H)
        gen = orc.ref_gen(knobs, knobs, knobs)
        path = OUT / "_tmp_trace.tsv"
        orc.ref_check(orc.ref_lib().ref_write_trace(C.byref(gen), C.byref(spec), B, seed, str(path).encode()))
        header = json.loads(path.read_text().split("\n", 1)[0])
        path.unlink()
        _, _, act = orc.ref_trace(gen, spec, B, seed)
        out.append({"spec": [name, L, E, H], "knobs": knobs, "batch": B, "seed": seed,
                    "fnv1a": header["checksum"], "top0": act[0, 0].tolist(), "top1": act[0, 1].tolist()})
    return out


def random_loads(rng, layer, lo, hi, max_tokens=20):
    n = rng.randint(lo, hi)
    loads = [(e, layer, rng.randint(1, max_tokens)) for e in range(n)]
    loads.sort(key=lambda x: (x[2], x[0]))
    return loads


def presched_cases(n=1000, seed=7):
    """Same distribution as random_inputs in test_scheduler.cpp:13-28, plus large lists."""
    rng = random.Random(seed)
    cases = []
    for i in range(n):
        big = i % 10 == 0
        hi = 64 if big else 6
        cur, nxt, nxt2 = random_loads(rng, 0, 1, hi), random_loads(rng, 1, 0, hi), random_loads(rng, 2, 0, hi)
        t_io = rng.randint(5, 30)
        params = (t_io, rng.randint(1, min(t_io - 1, 8)), rng.randint(0, 10), rng.uniform(0.5, 4.0),
                  rng.randint(0, 5), rng.randint(0, 20))
        hit = rng.random()
        stats = (hit, 1.0 - hit, 32)
        entry = {"e_cur": cur, "e_next": nxt, "e_next2": nxt2, "params": params, "stats": stats, "plans": {}}
        for pol in ("presched", "greedy", "ondemand", "fixed:2"):
            rc, plan = orc.ref_plan_layer(cur, nxt, nxt2, params, stats, pol)
            assert rc == 0
            entry["plans"][pol] = plan
        cases.append(entry)
    # invalid inputs: the reference rejects them with invalid_argument
    bad = [{"e_cur": [(0, 0, 5), (1, 0, 2)], "e_next": [], "e_next2": [], "params": (10, 2, 3, 1.0, 1, 0)},
           {"e_cur": [(0, 0, 0)], "e_next": [], "e_next2": [], "params": (10, 2, 3, 1.0, 1, 0)},
           {"e_cur": [(0, 0, 2)], "e_next": [], "e_next2": [], "params": (2, 2, 3, 1.0, 1, 0)},
           {"e_cur": [(0, 0, 2)], "e_next": [], "e_next2": [], "params": (10, 2, -3, 1.0, 1, 0)}]
    for b in bad:
        rc, _ = orc.ref_plan_layer(b["e_cur"], b["e_next"], b["e_next2"], b["params"], (1.0, 0.0, 32), "presched")
        b["rc"] = rc
    return {"cases": cases, "invalid": bad}


def sim_cases(n=300, seed=11):
    rng = random.Random(seed)
    out = []
    for i in range(n):
        L = rng.randint(2, 8)
        E = rng.randint(2, 12)
        truth = np.zeros((L, E), np.int32)
        pred = np.zeros((L, E), np.int32)
        for l in range(L):
            for e in rng.sample(range(E), rng.randint(1, E)):
                truth[l, e] = rng.randint(1, 8)
            for e in rng.sample(range(E), rng.randint(0, E)):
                pred[l, e] = rng.randint(1, 8)
        resident = (np.array([[rng.random() < 0.2 for _ in range(E)] for _ in range(L)])).astype(np.uint8)
        groups = [0 if l < max(1, L // 3) else (2 if l >= L - max(1, L // 3) else 1) for l in range(L)]
        t_io = rng.randint(10, 28)
        params = (t_io, rng.randint(1, min(t_io - 1, 8)), rng.randint(2, 20), rng.uniform(0.2, 3.0),
                  rng.randint(0, 3), 0)
        entry = {"truth": truth.tolist(), "predicted": pred.tolist(), "resident": resident.tolist(),
                 "groups": groups, "params": params, "runs": {}}
        for pol in ("presched", "greedy", "ondemand", "fixed:2"):
            rc, r = orc.ref_simulate(truth, pred, params, pol, resident=resident, groups=groups,
                                     options=(1, 64, 1.0, 32))
            assert rc == 0, orc.ref_lib().ref_last_error()
            r["violations"] = orc.ref_verify(r["events"], truth, params, resident)
            entry["runs"][pol] = r
        out.append(entry)
    return out


def desk_trace():
    spec = desk_spec("mixtral", 4, 8, 16)
    gen = orc.ref_gen(**DEFAULT)
    hidden, gw, act = orc.ref_trace(gen, spec, 32, 0)
    np.savez_compressed(OUT / "desk_trace_c0.npz", hidden=hidden, gate_weights=gw, active=act,
                        spec=np.array([spec.num_layers, spec.experts, spec.top_k, spec.hidden,
                                       spec.group_begin_middle, spec.group_begin_output], np.int64),
                        expert_bytes=np.array([spec.expert_bytes], np.uint64))


def llapor():
    spec = desk_spec("mixtral", 4, 8, 16)
    gen = orc.ref_gen(**DEFAULT)
    seeds = (C.c_uint64 * 3)(101, 102, 103)
    path = OUT / "llapor_desk.llpc"
    orc.ref_check(orc.ref_lib().ref_train_llapor(C.byref(gen), C.byref(spec), 256, seeds, 3, 6, 2, 5,
                                                 str(path).encode()))
    h = orc.ref_lib().ref_llapor_load(str(path).encode())
    assert h
    hidden, gw, act = orc.ref_trace(gen, spec, 16, 0)
    rows = []
    reduced, logits, tops = [], [], []
    for t in range(16):
        for l in range(1, spec.num_layers):
            red = np.empty(16)
            lg = np.empty(spec.experts)
            top = np.empty(spec.top_k, np.int32)
            prev_act = np.ascontiguousarray(act[t, l - 1])
            orc.ref_check(orc.ref_lib().ref_llapor_predict(
                h, l, hidden[t, l - 1].ctypes.data, prev_act.ctypes.data, spec.top_k,
                np.ascontiguousarray(gw[t, l - 1]).ctypes.data, spec.top_k, red.ctypes.data, lg.ctypes.data,
                top.ctypes.data))
            rows.append((t, l))
            reduced.append(red.copy())
            logits.append(lg)
            tops.append(top)
    loads = np.empty((spec.num_layers, spec.experts), np.int32)
    orc.ref_check(orc.ref_lib().ref_llapor_predict_loads(h, C.byref(gen), 16, 0, spec.top_k, loads.ctypes.data))
    orc.ref_lib().ref_llapor_free(h)
    np.savez_compressed(OUT / "llapor_desk_expected.npz", rows=np.array(rows), logits=np.array(logits),
                        topk=np.array(tops), predicted_loads=loads, hidden=hidden, gate_weights=gw, active=act)


def ref_trace_file():
    spec = desk_spec("mixtral", 4, 8, 16)
    gen = orc.ref_gen((0.9, 0.3, 0.5), (0.9, 0.3, 0.5), (0.9, 0.3, 0.5))
    orc.ref_check(orc.ref_lib().ref_write_trace(C.byref(gen), C.byref(spec), 3, 17,
                                                str(OUT / "ref_trace_desk.tsv").encode()))


def ref_trace_h256():
    spec = desk_spec("mixtral", 4, 8, 256)
    gen = orc.ref_gen(DEFAULT["input"], DEFAULT["middle"], DEFAULT["output"])
    orc.ref_check(orc.ref_lib().ref_write_trace(C.byref(gen), C.byref(spec), 8, 23,
                                                str(OUT / "ref_trace_h256.tsv").encode()))


def main():
    orc.ref_check(orc.ref_lib().ref_dump_golden(str(OUT / "golden_scenarios.json").encode()))
    (OUT / "trace_fingerprints.json").write_text(json.dumps(fingerprints(), indent=1))
    desk_trace()
    (OUT / "presched_cases.json").write_text(json.dumps(presched_cases()))
    (OUT / "sim_cases.json").write_text(json.dumps(sim_cases()))
    llapor()
    ref_trace_file()
    ref_trace_h256()
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
