"""Per-kernel GPU time of engine decode steps (torch.profiler / CUPTI kernel records):
BASELINE config shapes through the same engine as bench.py / configs_bench.py.

  python scripts/decode_kernels.py --model qwen3 --batch 32 [--host-threads -1] [--timeline]
"""
import argparse
import collections
import pathlib
import sys

import torch

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "scripts"))
import bench  # noqa: E402
import configs_bench as cb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen3")
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--budget", type=float, default=0.5)
    ap.add_argument("--host-threads", type=int, default=-1)
    ap.add_argument("--timeline", action="store_true")
    args = ap.parse_args()
    spec, gen, gate, freq = cb.setup(args.model)
    pin, pmid = (256, 512) if args.model == "mixtral" else (128, 256)
    pred = cb.llapor(spec, pin, pmid)
    ht = bench.default_host_threads() if args.host_threads < 0 else args.host_threads
    e = cb.make_engine(spec, gen, gate, freq, args.budget, args.batch, pred, ht,
                       n_shared=2 if args.model == "deepseek" else 0)
    L, B = spec.num_layers, args.batch
    hid, fol = cb.trace_steps(torch, gen, spec, B, 6, 3000)
    y = torch.empty(L, B, spec.hidden_dim, device="cuda")
    for s in range(4):
        e.step_device(hid[s], fol[s], y)
        if s == 1:
            e.calibrate()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        e.step_device(hid[4], fol[4], y)
        torch.cuda.synchronize()
    st = e.stats()
    tot = collections.defaultdict(lambda: [0, 0.0])
    evs = []
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            name = ev.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0]
            tot[name][0] += 1
            tot[name][1] += ev.device_time_total
            evs.append((ev.time_range.start, ev.time_range.end, name))
    all_us = sum(v[1] for v in tot.values())
    evs.sort()
    span = evs[-1][1] - evs[0][0] if evs else 0
    print(f"{args.model} decode B={B}: {span / L:.1f} us per layer (first to last device op), "
          f"{all_us / L:.1f} us of device ops per layer")
    for name, (n, us) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{us / L:9.1f} us/layer  {n / L:5.2f}/layer  {100 * us / all_us:5.1f}%  {name[:90]}")
    if args.timeline:
        t0 = evs[0][0]
        for st_, en, name in evs[:60]:
            print(f"  {st_ - t0:9.1f} .. {en - t0:9.1f}  {name[:80]}")
    e.close()


if __name__ == "__main__":
    main()
