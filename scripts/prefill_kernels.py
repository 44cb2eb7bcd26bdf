"""Per-kernel GPU time of one engine prefill step (torch.profiler / CUPTI kernel records;
no nsys on this image): DeepSeek-V2-Lite shape, 2048-token chunk, all experts resident.

  python scripts/prefill_kernels.py [--model deepseek|mixtral] [--T 2048]
"""
import argparse
import collections
import pathlib
import sys

import torch

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "scripts"))
import configs_bench as cb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="deepseek")
    ap.add_argument("--T", type=int, default=2048)
    ap.add_argument("--timeline", action="store_true")
    args = ap.parse_args()
    spec, gen, gate, freq = cb.setup(args.model)
    n_shared = 2 if args.model == "deepseek" else 0
    pred = cb.llapor(spec, 128, 256)
    e = cb.make_engine(spec, gen, gate, freq, 1.0, args.T, pred, 0, n_shared=n_shared)
    L, H, T = spec.num_layers, spec.hidden_dim, args.T
    g = torch.Generator(device="cuda").manual_seed(5)
    ph = torch.randn(L, T, H, device="cuda", generator=g)
    ph /= ph.norm(dim=-1, keepdim=True)
    pf = torch.zeros(L, T, dtype=torch.uint8, device="cuda")
    py = torch.empty(L, T, H, device="cuda")
    for _ in range(2):
        e.step_device(ph, pf, py)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        e.step_device(ph, pf, py)
    b.record()
    torch.cuda.synchronize()
    step_ms = a.elapsed_time(b) / 3
    print(f"step {step_ms:.2f} ms = {step_ms * 1e3 / L:.1f} us per layer (device clock, CUDA events)")
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        e.step_device(ph, pf, py)
        torch.cuda.synchronize()
    tot = collections.defaultdict(lambda: [0, 0.0])
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            name = ev.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0]
            tot[name][0] += 1
            tot[name][1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
    all_us = sum(v[1] for v in tot.values())
    if args.timeline:  # device ops of layers 1-2 in order, with the idle gap before each
        evs = sorted((ev for ev in prof.events() if ev.device_type == torch.autograd.DeviceType.CUDA),
                     key=lambda ev: ev.time_range.start)
        t_prev = None
        per_layer = max(1, len(evs) // L)
        for ev in evs[per_layer: 3 * per_layer + 1]:
            st, en = ev.time_range.start, ev.time_range.end
            gap = st - t_prev if t_prev is not None else 0.0
            t_prev = en
            name = ev.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0]
            print(f"  gap {gap:8.1f} us  dur {en - st:8.1f} us  {name[:70]}")
    print(f"{args.model} prefill T={T}, {L} layers: {all_us / L:.1f} us of kernels per layer")
    for name, (n, us) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{us / L:9.1f} us/layer  {n / L:5.1f}/layer  {100 * us / all_us:5.1f}%  {name[:100]}")
    e.close()


if __name__ == "__main__":
    main()
