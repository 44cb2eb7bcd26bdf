#!/usr/bin/env python3
"""Where a host-lane decode layer's time goes (headline workload): per layer, from the
engine's measured timeline (CUDA events + host clock for the lane): scheduling point
end, lane batch start/end, last load end, layer end. Prints a JSON summary."""
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
    import argparse
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--lookahead", type=int, default=0)
    ap.add_argument("--model", default="mixtral")
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--summary", action="store_true", help="omit the per-layer rows")
    args = ap.parse_args()
    spec = ps.spec_preset(args.model)
    gen = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    L, E, H = spec.num_layers, spec.experts_per_layer, spec.hidden_dim
    B, S = args.batch, 6
    gate, hidden, follow, zipf = ps.trace_inputs(gen, spec, B * S, 1000)
    _, wh, wf, _ = ps.trace_inputs(gen, spec, 64, 1000, want_gate=False)
    freq = eng.hot_table(spec, gate, wh, wf, zipf)
    budget = int(round(0.5 * L * E)) * spec.expert_bytes
    resident = ps.plan_residency(freq, budget, spec.expert_bytes)
    lib = ps.load()
    pred = C.c_void_p()
    p_in, p_mid = (256, 512) if args.model == "mixtral" else (128, 256)
    ps.check(lib.ps_llapor_random(C.byref(spec), p_in, p_mid, 32, 48, 3, C.byref(pred)))
    e = eng.Engine(spec, gen, max_batch=B, weight_seed=1, gate=gate, budget_bytes=budget, resident=resident,
                   policy="presched", predictor=pred, host_threads=bench.default_host_threads(), compress_host=True,
                   lookahead=args.lookahead)
    hid = [torch.as_tensor(np.ascontiguousarray(hidden[s * B:(s + 1) * B].transpose(1, 0, 2), np.float32),
                           device="cuda") for s in range(S)]
    fol = [torch.as_tensor(np.ascontiguousarray(follow[s * B:(s + 1) * B].T), device="cuda") for s in range(S)]
    y = torch.empty(L, B, H, device="cuda")
    for s in range(S - 1):
        e.step_device(hid[s], fol[s], y)
        if s == 2:
            e.calibrate()
    e.step_device(hid[S - 1], fol[S - 1], y)
    torch.cuda.synchronize()
    events, truth, res, ls, le = e.last_timeline()
    rows = []
    for l in range(L):
        ev = [x for x in events if x[4] == l]
        att = [x for x in ev if x[3] == 0]
        cpu = [x for x in ev if x[3] == 2]
        ld = [x for x in ev if x[3] == 3]
        pf = [x for x in events if x[3] == 4 and x[4] == l + 1]
        gpu = [x for x in ev if x[3] == 1]
        io = sorted([x for x in events if x[2] == 2 and x[0] < le[l] and x[1] > ls[l]])
        io_busy = sum(min(x[1], le[l]) - max(x[0], ls[l]) for x in io)
        rows.append({"layer": l, "start": ls[l], "end": le[l], "sched_end": att[0][1] if att else None,
                     "io_busy_in_layer": io_busy, "gpu_expert_starts": [x[0] for x in gpu],
                     "cpu_start": cpu[0][0] if cpu else None, "cpu_end": cpu[0][1] if cpu else None,
                     "n_cpu": len(cpu), "n_load": len(ld), "n_prefetch_next": len(pf),
                     "load_us": [x[1] - x[0] for x in ld + pf], "load_end": max((x[1] for x in ld), default=None),
                     "gpu_end": max((x[1] for x in gpu), default=None)})
    tot = le[-1] - ls[0]
    cpu_busy = sum(r["cpu_end"] - r["cpu_start"] for r in rows if r["cpu_start"] is not None)
    gaps = [(r["cpu_start"] - r["start"]) for r in rows if r["cpu_start"] is not None]
    tails = [(r["end"] - r["cpu_end"]) for r in rows if r["cpu_end"] is not None]
    print(json.dumps({"cost": e.stats()["cost"], "step_us": tot, "cpu_busy_us": cpu_busy, "layer_start_to_lane_start_us_mean": float(np.mean(gaps)),
                      "lane_end_to_layer_end_us_mean": float(np.mean(tails)),
                      "sched_end_minus_start_us_mean": float(np.mean([r["sched_end"] - r["start"] for r in rows
                                                                      if r["sched_end"] is not None])),
                      "n_cpu_mean": float(np.mean([r["n_cpu"] for r in rows])),
                      "n_load_mean": float(np.mean([r["n_load"] for r in rows])),
                      "layers": [] if args.summary else rows}))
    e.close()


if __name__ == "__main__":
    main()
