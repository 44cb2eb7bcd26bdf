"""z-slab decode micro-benchmark (Mixtral expert, 352 MB of bf16): device time per
ps_zslab_decode and the HBM bytes it moves (z-slab read + bf16 written), for both code
widths. One JSON line per width."""
import ctypes as C
import json
import os
import pathlib
import sys

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_2509_23638_b200 as ps  # noqa: E402


def main():
    lib = ps.load()
    H, F = 4096, 14336
    n = 3 * H * F
    slab = np.empty(n, np.uint16)
    ps.check(lib.ps_init_expert_slab_host(slab.ctypes.data, H, F, 1, 0, 0))
    tiled_slab = slab.copy()
    ps.check(lib.ps_host_slab_tile(tiled_slab.ctypes.data, H, F))
    for bits, tiled in [tuple(c.split(":")) for c in os.environ.get("ZMICRO_CASES", "3:0,4:0,3:1").split(",")]:
        tiled = int(tiled)
        os.environ["PS_ZSLAB_BITS"] = bits
        cap = lib.ps_zslab_bound(n)
        z = np.zeros(cap, np.uint8)
        nb = C.c_uint64()
        if tiled:  # the engine's host-lane configuration: z-slab of the lane's tile layout
            ps.check(lib.ps_zslab_encode_tiled(tiled_slab.ctypes.data, H, F, z.ctypes.data, cap, C.byref(nb), 0))
        else:
            ps.check(lib.ps_zslab_encode(slab.ctypes.data, n, z.ctypes.data, cap, C.byref(nb), 0))
        z = z[:nb.value].copy()
        zd = torch.as_tensor(z, device="cuda")
        outs = [torch.empty(n, dtype=torch.int16, device="cuda") for _ in range(3)]
        s = torch.cuda.current_stream()
        for i in range(3):
            ps.check(lib.ps_zslab_decode(C.c_void_p(zd.data_ptr()), z.ctypes.data, C.c_void_p(outs[i].data_ptr()),
                                         C.c_void_p(s.cuda_stream)))
        for ver in os.environ.get("ZMICRO_VERSIONS", "4").split(","):  # PS_ZDECODE A/B, same process
            os.environ["PS_ZDECODE"] = ver
            for o in outs:
                o.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            iters = 20
            for i in range(iters):
                ps.check(lib.ps_zslab_decode(C.c_void_p(zd.data_ptr()), z.ctypes.data,
                                             C.c_void_p(outs[i % 3].data_ptr()), C.c_void_p(s.cuda_stream)))
            b.record()
            torch.cuda.synchronize()
            us = a.elapsed_time(b) * 1e3 / iters
            assert np.array_equal(outs[0].cpu().numpy().view(np.uint16), slab)
            print(json.dumps({"bits": int(bits), "tiled": tiled, "version": ver, "z_bytes": int(nb.value), "us": us,
                              "hbm_gbs": (nb.value + 2 * n) / (us * 1e-6) / 1e9}), flush=True)


if __name__ == "__main__":
    main()
