"""LLaPor forward micro-benchmark at the bench's predictor shape (Mixtral, random net
P=256/512, width 32/48): device time per ps_llapor_forward call for an input-, middle-
and output-group layer. Small enough to run under ncu.

  python scripts/llapor_micro.py --batch 16 --iters 200
"""
import argparse
import ctypes as C
import json
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_2509_23638_b200 as ps  # noqa: E402


def _p(t):
    return C.c_void_p(t.data_ptr())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="mixtral")
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--iters", type=int, default=200)
    args = ap.parse_args()
    lib = ps.load()
    spec = ps.spec_preset(args.model)
    E, H, k = spec.experts_per_layer, spec.hidden_dim, spec.top_k
    m = C.c_void_p()
    ps.check(lib.ps_llapor_random(C.byref(spec), 256, 512, 32, 48, 3, C.byref(m)))
    B = args.batch
    x = torch.randn(B, H, device="cuda")
    pids = torch.randint(0, E, (B, k), dtype=torch.int32, device="cuda")
    pw = torch.softmax(torch.randn(B, E, device="cuda"), 1)
    scratch = torch.empty(lib.ps_llapor_scratch_bytes(m, B), dtype=torch.uint8, device="cuda")
    logits = torch.empty(B, E, device="cuda")
    ids = torch.empty(B, k, dtype=torch.int32, device="cuda")
    cnt = torch.empty(E, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    sp = C.c_void_p(s.cuda_stream)
    out = {"model": args.model, "batch": B}
    layers = {"input": 1, "middle": spec.group_begin_middle + 1, "output": spec.num_layers - 1}
    for name, l in layers.items():
        def call():
            ps.check(lib.ps_llapor_forward(m, l, _p(x), _p(pids), k, _p(pw), B, k, _p(logits), _p(ids), _p(cnt),
                                           _p(scratch), sp))
        for _ in range(5):
            call()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.iters):
            call()
        b.record()
        torch.cuda.synchronize()
        out[f"{name}_us"] = a.elapsed_time(b) * 1e3 / args.iters
    print(json.dumps(out))
    lib.ps_llapor_free(m)


if __name__ == "__main__":
    main()
