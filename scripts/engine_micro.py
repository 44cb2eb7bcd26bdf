"""All-resident engine micro-run (no host offload): per-phase device times of a decode
or prefill step. Small enough to run under `ncu --metrics gpu__time_duration.sum`.

  python scripts/engine_micro.py --model mixtral --batch 16 --steps 3
"""
import argparse
import ctypes as C
import json
import pathlib
import sys

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_2509_23638_b200 as ps  # noqa: E402
from paper_2509_23638_b200 import engine as eng  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="mixtral")
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--layers", type=int, default=0, help="truncate the stack (0 = all)")
    args = ap.parse_args()
    spec = ps.spec_preset(args.model)
    if args.layers:
        spec = ps.desk_scale(spec, args.layers, spec.experts_per_layer, spec.hidden_dim)
    L, E, H = spec.num_layers, spec.experts_per_layer, spec.hidden_dim
    gen = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    B = args.batch
    gate, _, _, _ = ps.trace_inputs(gen, spec, 1, 1000)
    lib = ps.load()
    pred = C.c_void_p()
    ps.check(lib.ps_llapor_random(C.byref(spec), 256, 512, 32, 48, 3, C.byref(pred)))
    e = eng.Engine(spec, gen, max_batch=B, weight_seed=1, gate=gate, budget_bytes=L * E * spec.expert_bytes,
                   resident=[(l, x) for l in range(L) for x in range(E)], predictor=pred)
    g = torch.Generator(device="cuda").manual_seed(1)
    h = torch.randn(L, B, H, device="cuda", generator=g)
    h /= h.norm(dim=-1, keepdim=True)
    f = torch.zeros(L, B, dtype=torch.uint8, device="cuda")
    y = torch.empty(L, B, H, device="cuda")
    e.step_device(h, f, y)
    torch.cuda.synchronize()
    e.reset_stats()
    for _ in range(args.steps):
        e.step_device(h, f, y)
    torch.cuda.synchronize()
    st = e.stats()
    n = max(1, st["layers"])
    print(json.dumps({"model": args.model, "batch": B, "layers": L,
                      "ms_per_step": st["step_ms_total"] / max(1, st["steps"]),
                      "layer_us": st["step_ms_total"] * 1e3 / n,
                      "route_phase_us": st["route_phase_ms_total"] * 1e3 / n,
                      "ffn_us": st["ffn_ms_total"] * 1e3 / n,
                      "combine_us": st["combine_ms_total"] * 1e3 / n,
                      "ffn_gbs": st["ffn_bytes_total"] / max(1e-9, st["ffn_ms_total"] / 1e3) / 1e9,
                      "ffn_tflops": st["ffn_flops_total"] / max(1e-9, st["ffn_ms_total"] / 1e3) / 1e12,
                      "tc_launches": st["tc_launches"],
                      "m_e": e.last_timeline()[1].tolist()}))
    e.close()
    lib.ps_llapor_free(pred)


if __name__ == "__main__":
    main()
