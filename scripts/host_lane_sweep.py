#!/usr/bin/env python3
"""Headline workload (Mixtral B=16, 50 % budget) through the host-lane executor for a
few lane thread counts, with and without in-step calibration; one JSON line per point.

  python scripts/host_lane_sweep.py --threads 10,12,13 --steps 10
"""
import argparse
import ctypes as C
import json
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2509_23638_b200 as ps  # noqa: E402
from paper_2509_23638_b200 import engine as eng  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", default="10,12,13")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    import torch
    spec = ps.spec_preset("mixtral")
    gen = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    L, E, H = spec.num_layers, spec.experts_per_layer, spec.hidden_dim
    B, S = 16, args.warmup + args.steps
    gate, hidden, follow, zipf = ps.trace_inputs(gen, spec, B * S, 1000)
    _, wh, wf, _ = ps.trace_inputs(gen, spec, 64, 1000, want_gate=False)
    freq = eng.hot_table(spec, gate, wh, wf, zipf)
    budget = int(round(0.5 * L * E)) * spec.expert_bytes
    resident = ps.plan_residency(freq, budget, spec.expert_bytes)
    lib = ps.load()
    pred = C.c_void_p()
    ps.check(lib.ps_llapor_random(C.byref(spec), 256, 512, 32, 48, 3, C.byref(pred)))
    hid = [torch.as_tensor(np.ascontiguousarray(hidden[s * B:(s + 1) * B].transpose(1, 0, 2), np.float32),
                           device="cuda") for s in range(S)]
    fol = [torch.as_tensor(np.ascontiguousarray(follow[s * B:(s + 1) * B].T), device="cuda") for s in range(S)]
    y = torch.empty(L, B, H, device="cuda")
    for t in [int(x) for x in args.threads.split(",")]:
        e = eng.Engine(spec, gen, max_batch=B, weight_seed=1, gate=gate, budget_bytes=budget, resident=resident,
                       policy="presched", predictor=pred, host_threads=t)
        cost = e.stats()["cost"]
        for cal in (False, True):
            e.set_cost(**cost)
            for s in range(args.warmup):
                e.step_device(hid[s], fol[s], y)
            torch.cuda.synchronize()
            if cal:
                e.calibrate()
            e.reset_stats()
            for s in range(args.warmup, S):
                e.step_device(hid[s], fol[s], y)
            torch.cuda.synchronize()
            st = e.stats()
            ms = st["step_ms_total"] / max(1, st["steps"])
            d = bench.decode_summary(st, ms, 1, B, L)
            d.update({"threads": t, "calibrated": cal})
            print(json.dumps(d), flush=True)
        e.close()
    lib.ps_llapor_free(pred)


if __name__ == "__main__":
    main()
