"""Device timeline of one all-resident decode step (CUPTI via torch.profiler): every
kernel and memcpy of the engine's compute stream with start/duration, and the per-layer
breakdown of the scheduling-point phase (K1 route, K4 LLaPor, K2 permute, D2H, host
sync gap) vs the expert FFN. Writes JSON to stdout.

  python scripts/engine_timeline.py --model mixtral --batch 16 --layers 4
"""
import argparse
import ctypes as C
import json
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_2509_23638_b200 as ps  # noqa: E402
from paper_2509_23638_b200 import engine as eng  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="mixtral")
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--layers", type=int, default=6)
    ap.add_argument("--host-experts", type=int, default=0,
                    help="last N experts of every layer live in pinned host DRAM (K4 + loads active)")
    args = ap.parse_args()
    spec = ps.spec_preset(args.model)
    spec = ps.desk_scale(spec, args.layers, spec.experts_per_layer, spec.hidden_dim)
    L, E, H = spec.num_layers, spec.experts_per_layer, spec.hidden_dim
    gen = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    B = args.batch
    gate, _, _, _ = ps.trace_inputs(gen, spec, 1, 1000)
    lib = ps.load()
    pred = C.c_void_p()
    ps.check(lib.ps_llapor_random(C.byref(spec), 256, 512, 32, 48, 3, C.byref(pred)))
    e = eng.Engine(spec, gen, max_batch=B, weight_seed=1, gate=gate, budget_bytes=L * E * spec.expert_bytes,
                   resident=[(l, x) for l in range(L) for x in range(E - args.host_experts)], predictor=pred)
    g = torch.Generator(device="cuda").manual_seed(1)
    h = torch.randn(L, B, H, device="cuda", generator=g)
    h /= h.norm(dim=-1, keepdim=True)
    f = torch.zeros(L, B, dtype=torch.uint8, device="cuda")
    y = torch.empty(L, B, H, device="cuda")
    for _ in range(3):
        e.step_device(h, f, y)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        e.step_device(h, f, y)
        torch.cuda.synchronize()
    evs = [ev for ev in prof.events() if ev.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda ev: ev.time_range.start)
    t0 = evs[0].time_range.start if evs else 0
    rows = [{"name": ev.name[:60], "start_us": ev.time_range.start - t0, "dur_us": ev.time_range.end - ev.time_range.start}
            for ev in evs]
    st = e.stats()
    print(json.dumps({"model": args.model, "batch": B, "layers": L, "step_ms": st["step_ms_total"] / max(1, st["steps"]),
                      "events": rows}))
    e.close()


if __name__ == "__main__":
    main()
