#!/usr/bin/env python3
"""Headline engine (Mixtral shape, B=16, 50 % budget, host lane): alternate rounds of
device-input steps (step_device) and host-buffer steps (ps_engine_decode_step_host) on
one engine and print per-round wall ms/step and lane stats, to separate the e2e path's
own cost from run-to-run drift."""
import ctypes as C
import json
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2509_23638_b200 as ps  # noqa: E402
from paper_2509_23638_b200 import engine as eng  # noqa: E402


def main():
    import torch
    spec = ps.spec_preset("mixtral")
    gen = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    L, E, H, k = spec.num_layers, spec.experts_per_layer, spec.hidden_dim, spec.top_k
    B, S = 16, 8
    gate, hidden, follow, zipf = ps.trace_inputs(gen, spec, B * S, 1000)
    _, wh, wf, _ = ps.trace_inputs(gen, spec, 64, 1000, want_gate=False)
    freq = eng.hot_table(spec, gate, wh, wf, zipf)
    budget = int(round(0.5 * L * E)) * spec.expert_bytes
    resident = ps.plan_residency(freq, budget, spec.expert_bytes)
    lib = ps.load()
    pred = C.c_void_p()
    ps.check(lib.ps_llapor_random(C.byref(spec), 256, 512, 32, 48, 3, C.byref(pred)))
    e = eng.Engine(spec, gen, max_batch=B, weight_seed=1, gate=gate, budget_bytes=budget, resident=resident,
                   policy="presched", predictor=pred, host_threads=bench.default_host_threads(), compress_host=True)
    hid_d = [torch.as_tensor(np.ascontiguousarray(hidden[s * B:(s + 1) * B].transpose(1, 0, 2), np.float32),
                             device="cuda") for s in range(S)]
    fol_d = [torch.as_tensor(np.ascontiguousarray(follow[s * B:(s + 1) * B].T), device="cuda") for s in range(S)]
    hid_h = [h.cpu().pin_memory() for h in hid_d]
    fol_h = [f.cpu().pin_memory() for f in fol_d]
    y_d = torch.empty(L, B, H, device="cuda")
    y_h = torch.empty(L, B, H).pin_memory()
    ids_h = torch.empty(L, B, k, dtype=torch.int32).pin_memory()
    for s in range(3):
        e.step_device(hid_d[s], fol_d[s], y_d)
    torch.cuda.synchronize()
    e.calibrate()
    for rnd in range(3):
        for mode in ("device", "host", "host_noids"):
            e.reset_stats()
            t0 = time.perf_counter()
            for s in range(3, S):
                if mode == "device":
                    e.step_device(hid_d[s], fol_d[s], y_d)
                    torch.cuda.synchronize()
                else:
                    ps.check(lib.ps_engine_decode_step_host(e.h, C.c_void_p(hid_h[s].data_ptr()),
                                                            C.c_void_p(fol_h[s].data_ptr()), B,
                                                            C.c_void_p(y_h.data_ptr()),
                                                            C.c_void_p(ids_h.data_ptr()) if mode == "host" else None))
            wall = (time.perf_counter() - t0) / (S - 3) * 1e3
            st = e.stats()
            print(json.dumps({"round": rnd, "mode": mode, "wall_ms": wall,
                              "dev_ms": st["step_ms_total"] / max(1, st["steps"]),
                              "cpu_ms": st["cpu_ms_total"] / max(1, st["steps"]),
                              "cpu_experts": st["cpu_experts"] / max(1, st["steps"]),
                              "ondemand": st["ondemand_loads"] / max(1, st["steps"])}), flush=True)
    e.close()


if __name__ == "__main__":
    main()
