#!/usr/bin/env python3
"""The other BASELINE.json configs, measured through the same engine as bench.py
(one JSON line per measurement point; bench.py itself stays on config[1]):

  mixtral-sweep  config[1] sweep: HBM budget {25,50,75,100}% x batch {1,4,16}, GPU-only
                 executor and host expert lane
  deepseek       config[2]: DeepSeek-V2-Lite shape (26 L, 64 routed top-6 + 2 shared,
                 H 2048, F 1408): 2048-token prefill chunk, then batch-16 decode, 50 %
                 budget, prefetch/on-demand mix (+ host lane)
  qwen3          config[3]: Qwen3-30B-A3B shape (48 L, 128 experts top-8, H 2048, F 768)
                 batch-32 decode, 50 % budget, LLaPor-driven prefetch (+ host lane)

Synthetic inputs as in bench.py (reference trace generator, hash-initialised bf16 weights,
random-init LLaPor at full shape). Timing: CUDA events on the engine's compute stream.

  python scripts/configs_bench.py --configs qwen3,deepseek,mixtral-sweep
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2509_23638_b200 as ps  # noqa: E402
from paper_2509_23638_b200 import engine as eng  # noqa: E402


COMPRESS = True


def make_engine(spec, gen, gate, freq, budget, B, predictor, host_threads, n_shared=0):
    L, E = spec.num_layers, spec.experts_per_layer
    budget_bytes = int(round(budget * L * E)) * spec.expert_bytes
    resident = ps.plan_residency(freq, budget_bytes, spec.expert_bytes)
    return eng.Engine(spec, gen, max_batch=B, weight_seed=1, gate=gate, budget_bytes=budget_bytes, resident=resident,
                      policy="presched", predictor=predictor, host_threads=host_threads, n_shared=n_shared,
                      compress_host=COMPRESS)


def timed_steps(torch, e, hid, fol, y, warmup, steps, calibrate=False):
    for s in range(warmup):
        e.step_device(hid[s % len(hid)], fol[s % len(fol)], y)
    torch.cuda.synchronize()
    if calibrate:
        e.calibrate()
    e.reset_stats()
    for s in range(steps):
        e.step_device(hid[(warmup + s) % len(hid)], fol[(warmup + s) % len(fol)], y)
    torch.cuda.synchronize()
    st = e.stats()
    return st, st["step_ms_total"] / max(1, st["steps"])


def decode_points(torch, name, spec, e, B, hid, fol, y, args, extra):
    """GPU-only executor and (if the engine has one) host-lane executor on one engine."""
    out = []
    L = spec.num_layers
    cost = e.stats()["cost"]
    e.set_cost(cost["t_io"], cost["t_g"], cost["t_attn"], 1e9, 0)
    legs = [("gpu_only", False)]
    if e.host_threads:
        legs.append(("host_lane", True))
    for leg, cal in legs:
        if leg == "host_lane":
            e.set_cost(**cost)
        st, ms = timed_steps(torch, e, hid, fol, y, args.warmup, args.steps, calibrate=cal)
        d = bench.decode_summary(st, ms, 1, B, L)
        ffn_gbs = st["ffn_bytes_total"] / (st["ffn_ms_total"] / 1e3) / 1e9 if st["ffn_ms_total"] > 0 else 0.0
        d.update({"config": name, "executor": leg, "batch": B, "ffn_achieved_gbs": ffn_gbs,
                  "ffn_frac_of_hbm": ffn_gbs / bench.measured_peaks()[0], "gpu_launches": st["kernel_launches"]})
        d.update(extra)
        if "cpu_lane" in d:
            d["cpu_lane"]["threads"] = e.host_threads
        out.append(d)
        print(json.dumps(d), flush=True)
    return out


def trace_steps(torch, gen, spec, B, S, seed):
    _, hidden, follow, _ = ps.trace_inputs(gen, spec, B * S, seed, want_gate=False)
    hid = [torch.as_tensor(np.ascontiguousarray(hidden[s * B:(s + 1) * B].transpose(1, 0, 2), np.float32),
                           device="cuda") for s in range(S)]
    fol = [torch.as_tensor(np.ascontiguousarray(follow[s * B:(s + 1) * B].T), device="cuda") for s in range(S)]
    return hid, fol


def finetune(torch, e, pred, spec, gen, B, steps, seed=4242, epochs=3, lr=3e-3):
    """Online LLaPor fine_tune (ps_llapor_fine_tune = predictor.cpp:654-663) on a separate
    warm-up trace before any measurement: decode a step, fine-tune every net on its
    observations, repeat. Replaces the random-init predictor by one trained the way the
    reference's online path trains it."""
    if steps <= 0 or pred is None:
        return
    _, hidden, follow, _ = ps.trace_inputs(gen, spec, B * steps, seed, want_gate=False)
    y = torch.empty(spec.num_layers, B, spec.hidden_dim, device="cuda")
    for s in range(steps):
        h = np.ascontiguousarray(hidden[s * B:(s + 1) * B].transpose(1, 0, 2), np.float32)
        f = np.ascontiguousarray(follow[s * B:(s + 1) * B].T)
        e.step_device(torch.as_tensor(h, device="cuda"), torch.as_tensor(f, device="cuda"), y)
        torch.cuda.synchronize()
        e.fine_tune_predictor(pred, h, steps=epochs, lr=lr)


def setup(model):
    spec = ps.spec_preset(model)
    gen = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    gate, warm_h, warm_f, zipf = ps.trace_inputs(gen, spec, 64, 1000)
    freq = eng.hot_table(spec, gate, warm_h, warm_f, zipf)
    return spec, gen, gate, freq


def llapor(spec, pin, pmid):
    lib = ps.load()
    m = C.c_void_p()
    ps.check(lib.ps_llapor_random(C.byref(spec), pin, pmid, 32, 48, 3, C.byref(m)))
    return m


def run_qwen3(torch, args, ht):
    spec, gen, gate, freq = setup("qwen3")
    B = 32
    pred = llapor(spec, 128, 256)
    e = make_engine(spec, gen, gate, freq, args.budget, B, pred, ht)
    finetune(torch, e, pred, spec, gen, B, args.finetune)
    hid, fol = trace_steps(torch, gen, spec, B, args.warmup + args.steps, 2000)
    y = torch.empty(spec.num_layers, B, spec.hidden_dim, device="cuda")
    tag = (f"LLaPor P=128/256 fine-tuned online on {args.finetune} warm-up steps" if args.finetune
           else "random-init LLaPor P=128/256")
    decode_points(torch, f"qwen3-30b-a3b-shape decode B=32, LLaPor-driven prefetch ({tag})",
                  spec, e, B, hid, fol, y, args, {"budget_fraction": args.budget, "llapor_finetune_steps": args.finetune})
    e.close()
    ps.load().ps_llapor_free(pred)


def run_deepseek(torch, args, ht):
    spec, gen, gate, freq = setup("deepseek")
    T, B = 2048, 16
    pred = llapor(spec, 128, 256)
    e = make_engine(spec, gen, gate, freq, args.budget, T, pred, ht, n_shared=2)
    L, H = spec.num_layers, spec.hidden_dim
    # prefill chunk of T tokens (tcgen05 path; random unit hidden states), then decode
    g = torch.Generator(device="cuda").manual_seed(5)
    ph = torch.randn(L, T, H, device="cuda", generator=g)
    ph /= ph.norm(dim=-1, keepdim=True)
    pf = torch.zeros(L, T, dtype=torch.uint8, device="cuda")
    py = torch.empty(L, T, H, device="cuda")
    cost = e.stats()["cost"]
    for leg in (["gpu_only", "host_lane"] if e.host_threads else ["gpu_only"]):
        e.set_cost(cost["t_io"], cost["t_g"], cost["t_attn"], 1e9 if leg == "gpu_only" else cost["beta"],
                   0 if leg == "gpu_only" else cost["startup"])
        st, ms = timed_steps(torch, e, [ph], [pf], py, 1, 2)
        tf = st["ffn_flops_total"] / (st["ffn_ms_total"] / 1e3) / 1e12 if st["ffn_ms_total"] > 0 else 0.0
        d = bench.decode_summary(st, ms, 1, T, L)
        d.update({"config": "deepseek-v2-lite-shape prefill 2048 tokens (64 routed top-6 + 2 shared)",
                  "executor": leg, "tokens_per_step": T, "ffn_tflops": tf, "tc_launches": st["tc_launches"],
                  "budget_fraction": args.budget})
        print(json.dumps(d), flush=True)
    # the same chunk with every expert resident: one grouped tcgen05 launch per layer,
    # the expert GEMM's own rate (BASELINE config 3's prefill FFN vs the bf16 peak)
    e_full = make_engine(spec, gen, gate, freq, 1.0, T, pred, 0, n_shared=2)
    st, ms = timed_steps(torch, e_full, [ph], [pf], py, 1, 3)
    tf = st["ffn_flops_total"] / (st["ffn_ms_total"] / 1e3) / 1e12 if st["ffn_ms_total"] > 0 else 0.0
    d = bench.decode_summary(st, ms, 1, T, L)
    peak, peak_kind = bench.bf16_peak()
    d.update({"config": "deepseek-v2-lite-shape prefill 2048 tokens, all experts resident (64 routed top-6 + 2 shared)",
              "executor": "all_resident", "tokens_per_step": T, "ffn_tflops": tf, "tc_launches": st["tc_launches"],
              "ffn_frac_of_bf16_peak": tf / peak, "peak_tflops": peak, "peak_kind": peak_kind, "budget_fraction": 1.0})
    print(json.dumps(d), flush=True)
    e_full.close()
    del ph, py
    e.set_cost(**cost)
    finetune(torch, e, pred, spec, gen, B, args.finetune)
    hid, fol = trace_steps(torch, gen, spec, B, args.warmup + args.steps, 3000)
    y = torch.empty(L, B, H, device="cuda")
    decode_points(torch, "deepseek-v2-lite-shape decode B=16 after prefill (64 routed top-6 + 2 shared)"
                  + (f", LLaPor fine-tuned online on {args.finetune} warm-up steps" if args.finetune else ""),
                  spec, e, B, hid, fol, y, args, {"budget_fraction": args.budget, "llapor_finetune_steps": args.finetune})
    e.close()
    ps.load().ps_llapor_free(pred)


def run_mixtral_sweep(torch, args, ht):
    spec, gen, gate, freq = setup("mixtral")
    pred = llapor(spec, 256, 512)
    L, H = spec.num_layers, spec.hidden_dim
    for budget in (0.25, 0.5, 0.75, 1.0):
        e = make_engine(spec, gen, gate, freq, budget, 16, pred, ht if budget < 1.0 else 0)
        for B in (1, 4, 16):
            hid, fol = trace_steps(torch, gen, spec, B, args.warmup + args.steps, 4000 + B)
            y = torch.empty(L, B, H, device="cuda")
            decode_points(torch, f"mixtral-8x7b-shape decode B={B} budget {budget:.0%}", spec, e, B, hid, fol, y,
                          args, {"budget_fraction": budget})
        e.close()
    ps.load().ps_llapor_free(pred)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="qwen3,deepseek,mixtral-sweep")
    ap.add_argument("--budget", type=float, default=0.5)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--host-threads", type=int, default=-1)
    ap.add_argument("--compress", type=int, default=1)
    ap.add_argument("--finetune", type=int, default=0, help="warm-up steps of online LLaPor fine_tune (qwen3)")
    args = ap.parse_args()
    import torch
    torch.cuda.set_device(0)
    ht = args.host_threads if args.host_threads >= 0 else bench.default_host_threads()
    global COMPRESS
    COMPRESS = bool(args.compress)
    runs = {"qwen3": run_qwen3, "deepseek": run_deepseek, "mixtral-sweep": run_mixtral_sweep}
    for c in args.configs.split(","):
        t0 = time.perf_counter()
        runs[c](torch, args, ht)
        print(json.dumps({"config_done": c, "wall_s": time.perf_counter() - t0}), flush=True)


if __name__ == "__main__":
    main()
