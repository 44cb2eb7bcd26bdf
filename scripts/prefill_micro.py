"""Micro-benchmark of the K3 prefill path (tcgen05 grouped GEMM): T tokens routed
uniformly top-k over E experts of shape (H, F); CUDA-event timed; TFLOP/s vs the
measured cuBLAS bf16 peak.

  python scripts/prefill_micro.py --H 4096 --F 14336 --E 8 --k 2 --T 4096
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--H", type=int, default=4096)
    ap.add_argument("--F", type=int, default=14336)
    ap.add_argument("--E", type=int, default=8)
    ap.add_argument("--k", type=int, default=2)
    ap.add_argument("--T", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--ab-env", default="", help="NAME=v1,v2,...: alternate an env knob between timed runs")
    ap.add_argument("--kernel", type=int, default=2, help="ps_set_prefill_kernel mode (0 single, 1 pair, 2 auto, 3 token-N pair)")
    args = ap.parse_args()
    lib = ps.load()
    ps.check(lib.ps_set_prefill_kernel(args.kernel))
    H, F, E, k, T = args.H, args.F, args.E, args.k, args.T
    s = torch.cuda.current_stream()
    sp = C.c_void_p(s.cuda_stream)
    slabs = [torch.empty(3 * H * F, dtype=torch.int16, device="cuda") for _ in range(E)]
    for e, t in enumerate(slabs):
        ps.check(lib.ps_init_expert_slab(C.c_void_p(t.data_ptr()), H, F, 1, 0, e, sp))
    rng = np.random.default_rng(0)
    ids = np.stack([rng.choice(E, k, replace=False) for _ in range(T)]).astype(np.int32)
    rows = T * k
    di = torch.as_tensor(ids, device="cuda")
    x = (torch.randn(T, H, device="cuda") / H ** 0.5).to(torch.bfloat16)
    off = torch.empty(E + 1, dtype=torch.int32, device="cuda")
    src = torch.empty(rows, dtype=torch.int32, device="cuda")
    inv = torch.empty(rows, dtype=torch.int32, device="cuda")
    xp = torch.empty(rows, H, dtype=torch.bfloat16, device="cuda")
    ps.check(lib.ps_permute(C.c_void_p(di.data_ptr()), T, k, E, C.c_void_p(off.data_ptr()),
                            C.c_void_p(src.data_ptr()), C.c_void_p(inv.data_ptr()), C.c_void_p(x.data_ptr()), H,
                            C.c_void_p(xp.data_ptr()), sp))
    counts = np.bincount(ids.ravel(), minlength=E).astype(np.int32)
    offsets = off.cpu().numpy()
    g = ps.capi.ExpertGroup()
    g.n = E
    for e in range(E):
        g.experts[e] = e
        g.slabs[e] = slabs[e].data_ptr()
    h = torch.empty(rows, F, dtype=torch.bfloat16, device="cuda")
    yp = torch.empty(rows, H, dtype=torch.float32, device="cuda")

    def run():
        ps.check(lib.ps_expert_ffn_prefill(C.byref(g), counts.ctypes.data, offsets.ctypes.data,
                                           C.c_void_p(xp.data_ptr()), rows, H, F, C.c_void_p(h.data_ptr()),
                                           C.c_void_p(yp.data_ptr()), sp))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    if args.ab_env:
        import os
        name, vals = args.ab_env.split("=")
        res = {v: [] for v in vals.split(",")}
        for rep in range(args.iters):
            for v in res:  # the host runs ahead of the GPU as in the plain loop (map encoding hidden)
                if name == "kernel":
                    ps.check(lib.ps_set_prefill_kernel(int(v)))
                else:
                    os.environ[name] = v
                run()
                run()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                for _ in range(5):
                    run()
                b.record(s)
                b.synchronize()
                res[v].append(a.elapsed_time(b) / 5)
        flops = 2.0 * rows * 3 * H * F
        for v, t in res.items():
            ms = float(np.median(t))
            print(json.dumps({"H": H, "F": F, "E": E, "k": k, "T": T, name: v, "ms": ms, "tflops": flops / ms / 1e9,
                              "kernel": args.kernel}))
        return
    ts = []
    for _ in range(args.iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        run()
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    import time
    t0 = time.perf_counter()
    for _ in range(20):
        run()
    host_us = (time.perf_counter() - t0) / 20 * 1e6
    torch.cuda.synchronize()
    flops = 2.0 * rows * 3 * H * F
    peaks = ROOT / "MEASURED_PEAKS.json"
    peak = json.loads(peaks.read_text())["bf16_tflops"] if peaks.exists() else 1590.0
    print(json.dumps({"H": H, "F": F, "E": E, "k": k, "T": T, "rows": rows, "ms": ms,
                      "tflops": flops / ms / 1e9, "frac_bf16_peak": flops / ms / 1e9 / peak,
                      "m_per_expert": float(counts.mean()), "kernel": args.kernel,
                      "host_enqueue_us": host_us}))


if __name__ == "__main__":
    main()
