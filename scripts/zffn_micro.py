"""Fused z-slab K3 (ps_expert_ffn_zslab: fragments decoded in the consumer warps) vs the two-pass path (ps_zslab_decode into a bf16
slot, then ps_expert_ffn) at the Mixtral expert shape, decode token counts; CUDA events,
same process, alternating. HBM bytes: fused = z bytes; two-pass = z read + bf16 write +
bf16 read. Prints one JSON line per (experts, tokens) case."""
import ctypes as C
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2509_23638_b200 as ps  # noqa: E402


def main():
    lib = ps.load()
    H, F = 4096, 14336
    s = torch.cuda.current_stream()
    sp = C.c_void_p(s.cuda_stream)
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    E = 8
    bits = os.environ.get("PS_ZSLAB_BITS", "auto")  # pins the encoder's code width (3 or 4)
    zs_h, zs_d = [], []
    for e in range(E):
        slab = np.empty(3 * H * F, np.uint16)
        ps.check(lib.ps_init_expert_slab_host(slab.ctypes.data, H, F, 3, 0, e))
        ps.check(lib.ps_host_slab_tile(slab.ctypes.data, H, F))
        cap = lib.ps_zslab_bound(slab.size)
        z = np.zeros(cap, np.uint8)
        nb = C.c_uint64()
        ps.check(lib.ps_zslab_encode_tiled(slab.ctypes.data, H, F, z.ctypes.data, cap, C.byref(nb), 16))
        zs_h.append(z[:nb.value].copy())
        zs_d.append(torch.as_tensor(zs_h[-1], device="cuda"))
    zbytes = float(np.mean([z.size for z in zs_h]))
    slots = [torch.empty(3 * H * F, dtype=torch.int16, device="cuda") for _ in range(E)]
    peaks = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())
    cases = [(1, 2), (1, 8), (2, 4), (4, 4), (8, 4), (8, 8)]
    ncu = "--ncu" in sys.argv  # one fused launch per case for a profiler (no timing)
    if ncu:
        cases = [(2, 4)]
    for n_exp, m in cases:
        B = n_exp * m
        ids = np.array([[t % n_exp] for t in range(B)], np.int32)
        counts = np.bincount(ids.ravel(), minlength=E).astype(np.int32)
        di = torch.as_tensor(ids, device="cuda")
        off = torch.empty(E + 1, dtype=torch.int32, device="cuda")
        src = torch.empty(B, dtype=torch.int32, device="cuda")
        inv = torch.empty(B, dtype=torch.int32, device="cuda")
        ps.check(lib.ps_permute(P(di), B, 1, E, P(off), P(src), P(inv), None, H, None, sp))
        x = (torch.randn(B, H, device="cuda") / H ** 0.5).to(torch.bfloat16).view(torch.int16)
        h = torch.empty(B, F, dtype=torch.int16, device="cuda")
        n_split = lib.ps_ffn_down_splits(H, F)
        yp = torch.empty(n_split, B, H, dtype=torch.float32, device="cuda")
        grp = ps.capi.ExpertGroup()
        grp.n = n_exp
        zp = (C.c_void_p * n_exp)()
        for e in range(n_exp):
            grp.experts[e] = e
            grp.slabs[e] = slots[e].data_ptr()
            zp[e] = zs_d[e].data_ptr()

        def fused():
            ps.check(lib.ps_expert_ffn_zslab(C.byref(grp), zp, counts.ctypes.data, P(off), P(src), 1, P(x), H, F, P(h),
                                             P(yp), n_split, B, sp))

        def two_pass():
            for e in range(n_exp):
                ps.check(lib.ps_zslab_decode(P(zs_d[e]), zs_h[e].ctypes.data, P(slots[e]), sp))
            ps.check(lib.ps_expert_ffn(C.byref(grp), counts.ctypes.data, P(off), P(src), 1, P(x), H, F, P(h), P(yp),
                                       n_split, B, sp))

        def bf16_only():
            ps.check(lib.ps_expert_ffn(C.byref(grp), counts.ctypes.data, P(off), P(src), 1, P(x), H, F, P(h), P(yp),
                                       n_split, B, sp))
        if ncu:
            fused()
            bf16_only()
            torch.cuda.synchronize()
            continue
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        res = {"fused": [], "two_pass": [], "bf16_slot_only": []}
        fns = {"fused": fused, "two_pass": two_pass, "bf16_slot_only": bf16_only}
        for f in fns.values():
            f()
        torch.cuda.synchronize()
        for _ in range(8):
            for name, f in fns.items():
                flush.zero_()  # L2 flush (256 MB > 126 MB L2)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                f()
                b.record(s)
                b.synchronize()
                res[name].append(a.elapsed_time(b) * 1e3)
        med = {k: float(np.median(v)) for k, v in res.items()}
        line = {"code_bits": bits, "experts": n_exp, "tokens_per_expert": m, "us": med,
                "z_bytes_per_expert": zbytes, "bf16_bytes_per_expert": 6.0 * H * F,
                "fused_z_gbs": n_exp * zbytes / med["fused"] / 1e3,
                "fused_bf16_equiv_gbs": n_exp * 6.0 * H * F / med["fused"] / 1e3,
                "fused_frac_of_hbm_z": n_exp * zbytes / med["fused"] / 1e3 / peaks["hbm_gbs"],
                "hbm_bytes_fused": n_exp * zbytes, "hbm_bytes_two_pass": n_exp * (zbytes + 12.0 * H * F)}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
