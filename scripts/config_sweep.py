"""The other BASELINE.json configs through the same engine (one JSON line each):

  config 3  DeepSeek-V2-Lite shape (26 L, 64 experts top-6, H 2048, F 1408): 2k-token
            prefill chunk + B=16 decode, budget 50 %, prefetch/on-demand mix
  config 4  Qwen3-30B-A3B shape (48 L, 128 experts top-8, H 2048, F 768): B=32 decode,
            budget 50 %, LLaPor (random-init, full shape) driving PreSched prefetches

Timing: CUDA events on the engine's compute stream (device time per step), H2D copy
statistics from events on the copy stream.

  python scripts/config_sweep.py --configs qwen3 deepseek --steps 4
"""
import argparse
import ctypes as C
import json
import pathlib
import sys

import numpy as np
import torch

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2509_23638_b200 as ps  # noqa: E402
from paper_2509_23638_b200 import engine as eng  # noqa: E402


def run(model, batch, budget, steps, warmup, policy, calibrate, pca=(128, 256)):
    spec = ps.spec_preset(model)
    L, E, H = spec.num_layers, spec.experts_per_layer, spec.hidden_dim
    gen = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    S = warmup + steps
    gate, hidden, follow, zipf = ps.trace_inputs(gen, spec, batch * S, 2000)
    _, wh, wf, _ = ps.trace_inputs(gen, spec, 64, 2000, want_gate=False)
    freq = eng.hot_table(spec, gate, wh, wf, zipf)
    budget_bytes = int(round(budget * L * E)) * spec.expert_bytes
    resident = ps.plan_residency(freq, budget_bytes, spec.expert_bytes)
    lib = ps.load()
    pred = C.c_void_p()
    ps.check(lib.ps_llapor_random(C.byref(spec), pca[0], pca[1], 32, 48, 3, C.byref(pred)))
    e = eng.Engine(spec, gen, max_batch=max(batch, 2048), weight_seed=1, gate=gate, budget_bytes=budget_bytes,
                   resident=resident, policy=policy, predictor=pred)
    hid = [torch.as_tensor(np.ascontiguousarray(hidden[s * batch:(s + 1) * batch].transpose(1, 0, 2), np.float32),
                           device="cuda") for s in range(S)]
    fol = [torch.as_tensor(np.ascontiguousarray(follow[s * batch:(s + 1) * batch].T), device="cuda")
           for s in range(S)]
    y = torch.empty(L, batch, H, device="cuda")
    for s in range(warmup):
        e.step_device(hid[s], fol[s], y)
    if calibrate:
        e.calibrate()
        for s in range(warmup):
            e.step_device(hid[s], fol[s], y)
    torch.cuda.synchronize()
    e.reset_stats()
    for s in range(warmup, S):
        e.step_device(hid[s], fol[s], y)
    torch.cuda.synchronize()
    st = e.stats()
    ms = st["step_ms_total"] / max(1, st["steps"])
    out = {"config": f"{model} decode B={batch} budget {budget:.0%} policy {policy}"
                     + (" (calibrated costs)" if calibrate else ""),
           "tokens_per_s": batch / (ms / 1e3), "ms_per_step": ms, "moe_layer_us": ms * 1e3 / L,
           "ondemand_loads_per_step": st["ondemand_loads"] / max(1, st["steps"]),
           "prefetches_per_step": st["prefetches_committed"] / max(1, st["steps"]),
           "prefetch_cancelled_per_step": st["prefetches_cancelled"] / max(1, st["steps"]),
           "h2d_gbs": st["h2d_bytes"] / max(1e-9, st["h2d_busy_ms"] / 1e3) / 1e9,
           "h2d_hidden_fraction": (1 - st["compute_wait_ms"] / st["h2d_busy_ms"]) if st["h2d_busy_ms"] else 1.0,
           "ffn_gbs": st["ffn_bytes_total"] / max(1e-9, st["ffn_ms_total"] / 1e3) / 1e9,
           "route_phase_us_per_layer": st["route_phase_ms_total"] * 1e3 / max(1, st["layers"]),
           "cost_us": st["cost"]}
    lines = [out]
    if model == "deepseek":  # 2k-token prefill chunk through the same engine
        T = 2048
        g = torch.Generator(device="cuda").manual_seed(3)
        ph = torch.randn(L, T, H, device="cuda", generator=g)
        ph /= ph.norm(dim=-1, keepdim=True)
        pf = torch.zeros(L, T, dtype=torch.uint8, device="cuda")
        py = torch.empty(L, T, H, device="cuda")
        e.step_device(ph, pf, py)
        torch.cuda.synchronize()
        e.reset_stats()
        e.step_device(ph, pf, py)
        torch.cuda.synchronize()
        st = e.stats()
        ms = st["step_ms_total"]
        lines.append({"config": f"{model} prefill T={T} budget {budget:.0%}", "tokens_per_s": T / (ms / 1e3),
                      "ms_per_step": ms, "moe_layer_us": ms * 1e3 / L,
                      "ondemand_loads_per_step": st["ondemand_loads"], "prefetches_per_step":
                      st["prefetches_committed"], "tc_launches": st["tc_launches"],
                      "ffn_tflops": st["ffn_flops_total"] / max(1e-9, st["ffn_ms_total"] / 1e3) / 1e12,
                      "h2d_gbs": st["h2d_bytes"] / max(1e-9, st["h2d_busy_ms"] / 1e3) / 1e9,
                      "h2d_hidden_fraction": (1 - st["compute_wait_ms"] / st["h2d_busy_ms"])
                      if st["h2d_busy_ms"] else 1.0})
    e.close()
    lib.ps_llapor_free(pred)
    return lines


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["qwen3", "deepseek"])
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--budget", type=float, default=0.5)
    args = ap.parse_args()
    for c in args.configs:
        batch = 32 if c == "qwen3" else 16
        for policy, cal in (("presched", False), ("presched", True), ("ondemand", False)):
            for line in run(c, batch, args.budget, args.steps, args.warmup, policy, cal):
                print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
