"""Micro-benchmark of K3 (decode SwiGLU FFN) at a given shape: n experts x m tokens,
weights resident in HBM (> L2 in total), CUDA-event timed on the launching stream.

  python scripts/ffn_micro.py --H 4096 --F 14336 --experts 1 2 4 8 --tokens 2 4 --iters 20
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--H", type=int, default=4096)
    ap.add_argument("--F", type=int, default=14336)
    ap.add_argument("--E", type=int, default=8)
    ap.add_argument("--experts", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--tokens", type=int, nargs="+", default=[4])
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--copies", type=int, default=3, help="weight copies rotated to defeat L2")
    args = ap.parse_args()
    lib = ps.load()
    H, F, E = args.H, args.F, args.E
    s = torch.cuda.current_stream()
    sp = C.c_void_p(s.cuda_stream)
    slabs = [[torch.empty(3 * H * F, dtype=torch.int16, device="cuda") for _ in range(E)] for _ in range(args.copies)]
    for c in range(args.copies):
        for e in range(E):
            ps.check(lib.ps_init_expert_slab(C.c_void_p(slabs[c][e].data_ptr()), H, F, 1, c, e, sp))
    peak = json.loads((pathlib.Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
        if (pathlib.Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else 6650.0
    for n in args.experts:
        for m in args.tokens:
            B = m * n  # every token of expert e routes only to e (k=1 layout)
            k = 1
            ids = torch.tensor(np.repeat(np.arange(n), m).astype(np.int32), device="cuda").view(B, 1)
            off = torch.empty(E + 1, dtype=torch.int32, device="cuda")
            src = torch.empty(B, dtype=torch.int32, device="cuda")
            inv = torch.empty(B, dtype=torch.int32, device="cuda")
            ps.check(lib.ps_permute(C.c_void_p(ids.data_ptr()), B, k, E, C.c_void_p(off.data_ptr()),
                                    C.c_void_p(src.data_ptr()), C.c_void_p(inv.data_ptr()), None, H, None, sp))
            counts = np.zeros(E, np.int32)
            counts[:n] = m
            x = torch.randn(B, H, device="cuda").to(torch.bfloat16)
            nsplit = lib.ps_ffn_down_splits(H, F)
            h = torch.empty(B, F, dtype=torch.int16, device="cuda")
            yp = torch.empty(nsplit, B, H, dtype=torch.float32, device="cuda")
            groups = []
            for c in range(args.copies):
                g = ps.capi.ExpertGroup()
                g.n = n
                for i in range(n):
                    g.experts[i] = i
                    g.slabs[i] = slabs[c][i].data_ptr()
                groups.append(g)

            def run(c):
                ps.check(lib.ps_expert_ffn(C.byref(groups[c % args.copies]), counts.ctypes.data,
                                           C.c_void_p(off.data_ptr()), C.c_void_p(src.data_ptr()), k,
                                           C.c_void_p(x.data_ptr()), H, F, C.c_void_p(h.data_ptr()),
                                           C.c_void_p(yp.data_ptr()), nsplit, B, sp))
            for c in range(3):
                run(c)
            t = []
            for it in range(args.iters):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                run(it)
                b.record(s)
                b.synchronize()
                t.append(a.elapsed_time(b))
            ms = float(np.median(t))
            bytes_ = n * 6 * H * F
            print(json.dumps({"experts": n, "tokens_per_expert": m, "us": ms * 1e3, "GBps": bytes_ / ms / 1e6,
                              "frac_hbm": bytes_ / ms / 1e6 / peak}))


if __name__ == "__main__":
    main()
