#!/usr/bin/env python3
"""Host expert lane micro-benchmark (Mixtral expert shape): ps_host_expert_ffn GB/s of
expert weights streamed from pinned host DRAM vs threads and tokens, alone and while
the copy engine runs pinned H2D at full PCIe rate (the engine's concurrent situation).
Writes JSON lines (one per point) to stdout."""
import argparse
import ctypes as C
import json
import pathlib
import sys
import threading
import time

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_2509_23638_b200 as ps  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--H", type=int, default=4096)
    ap.add_argument("--F", type=int, default=14336)
    ap.add_argument("--threads", default="8,12,14,16")
    ap.add_argument("--tokens", default="1,4,8,16")
    ap.add_argument("--slabs", type=int, default=4)
    ap.add_argument("--reps", type=int, default=8)
    ap.add_argument("--isa", default="")
    ap.add_argument("--z", type=int, default=0, help="1: read z-slabs (ps_host_expert_ffn_batch_z)")
    args = ap.parse_args()
    import os
    if args.isa:
        os.environ["PS_HOST_LANE_ISA"] = args.isa
    import torch
    lib = ps.load()
    H, F = args.H, args.F
    nbytes = 6 * H * F
    slabs = [torch.empty(nbytes // 2, dtype=torch.int16).pin_memory() for _ in range(args.slabs)]
    for i, s in enumerate(slabs):
        ps.check(lib.ps_init_expert_slab_host(C.c_void_p(s.data_ptr()), H, F, 1, 0, i))
    zs = []
    if args.z:
        for sl in slabs:
            cap = lib.ps_zslab_bound(nbytes // 2)
            z = torch.empty(cap, dtype=torch.uint8).pin_memory()
            nb = C.c_uint64()
            ps.check(lib.ps_zslab_encode(C.c_void_p(sl.data_ptr()), nbytes // 2, C.c_void_p(z.data_ptr()), cap,
                                         C.byref(nb), 0))
            zs.append(z)
    x = np.zeros((64, H), np.uint16)
    y = np.zeros((64, H), np.float32)

    # background H2D loop (copy engine), like the engine's serial channel
    dma_stop = threading.Event()
    dma_bytes = [0, 0.0]
    src = torch.empty(nbytes // 2, dtype=torch.int16).pin_memory()
    dst = torch.empty(nbytes // 2, dtype=torch.int16, device="cuda")
    stream = torch.cuda.Stream()

    def dma():
        t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            while not dma_stop.is_set():
                dst.copy_(src, non_blocking=True)
                stream.synchronize()
                dma_bytes[0] += nbytes
        dma_bytes[1] = time.perf_counter() - t0

    for threads in [int(t) for t in args.threads.split(",")]:
        lane = C.c_void_p()
        ps.check(lib.ps_host_lane_create(threads, C.byref(lane)))
        isa = {1: "avx512-bf16", 2: "amx-bf16"}[lib.ps_host_lane_isa(lane)]
        for m in [int(t) for t in args.tokens.split(",")]:
            for concurrent in (False, True):
                th = None
                if concurrent:
                    dma_stop.clear()
                    dma_bytes[:] = [0, 0.0]
                    th = threading.Thread(target=dma)
                    th.start()
                    time.sleep(0.05)
                ts = []
                for r in range(args.reps):
                    s = slabs[r % len(slabs)]
                    t0 = time.perf_counter()
                    if args.z:
                        zp = (C.c_void_p * 1)(zs[r % len(zs)].data_ptr())
                        mm, r0 = (C.c_int32 * 1)(m), (C.c_int32 * 1)(0)
                        ps.check(lib.ps_host_expert_ffn_batch_z(lane, 1, zp, mm, r0, H, F, x.ctypes.data,
                                                                y.ctypes.data))
                    else:
                        ps.check(lib.ps_host_expert_ffn(lane, C.c_void_p(s.data_ptr()), H, F, x.ctypes.data, m,
                                                        y.ctypes.data))
                    ts.append(time.perf_counter() - t0)
                dma_gbs = None
                if th:
                    dma_stop.set()
                    th.join()
                    dma_gbs = dma_bytes[0] / dma_bytes[1] / 1e9
                ts.sort()
                print(json.dumps({"threads": threads, "isa": isa, "z": bool(args.z), "tokens": m, "concurrent_h2d": concurrent,
                                  "ms_median": ts[len(ts) // 2] * 1e3, "gbs_median": nbytes / ts[len(ts) // 2] / 1e9,
                                  "gbs_best": nbytes / ts[0] / 1e9, "h2d_gbs_during": dma_gbs}), flush=True)
        lib.ps_host_lane_destroy(lane)


if __name__ == "__main__":
    main()
