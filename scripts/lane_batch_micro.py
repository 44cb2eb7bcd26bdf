#!/usr/bin/env python3
"""Host-lane batch micro-benchmark without a GPU (plain host buffers): one
ps_host_expert_ffn_batch_z call over n experts (tiled z-slabs, the engine's host-lane
format) with m tokens each, as the engine issues a layer's cpu_set. Prints per-expert
time and GB/s of z-slab bytes (the lane's DRAM stream).

  python scripts/lane_batch_micro.py --H 2048 --F 768 --n 9 --m 3     # Qwen3-like layer
  python scripts/lane_batch_micro.py --H 4096 --F 14336 --n 3 --m 4   # Mixtral-like layer
"""
import argparse
import ctypes as C
import json
import pathlib
import sys
import time

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_2509_23638_b200 as ps  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--H", type=int, default=2048)
    ap.add_argument("--F", type=int, default=768)
    ap.add_argument("--n", type=int, default=9)
    ap.add_argument("--m", type=int, default=3)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--sets", type=int, default=8, help="distinct expert sets cycled (> LLC)")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    lib = ps.load()
    H, F, n, m = args.H, args.F, args.n, args.m
    N = 3 * H * F
    zs, zbytes = [], []
    slab = np.empty(N, np.uint16)
    for i in range(args.sets * n):
        ps.check(lib.ps_init_expert_slab_host(slab.ctypes.data, H, F, 1, 0, i))
        t = slab.copy()
        ps.check(lib.ps_host_slab_tile(t.ctypes.data, H, F))
        cap = lib.ps_zslab_bound(N)
        z = np.zeros(cap, np.uint8)
        nb = C.c_uint64()
        ps.check(lib.ps_zslab_encode_tiled(t.ctypes.data, H, F, z.ctypes.data, cap, C.byref(nb), 0))
        zs.append(z[:nb.value].copy())
        zbytes.append(nb.value)
    threads = args.threads or __import__("os").cpu_count()
    lane = C.c_void_p()
    ps.check(lib.ps_host_lane_create(threads, C.byref(lane)))
    rng = np.random.default_rng(0)
    x = rng.integers(0x3c00, 0x3f00, (n * m, H)).astype(np.uint16)
    y = np.zeros((n * m, H), np.float32)
    mm = (C.c_int32 * n)(*([m] * n))
    r0 = (C.c_int32 * n)(*[j * m for j in range(n)])
    ts = []
    for r in range(args.reps + 2):
        s = r % args.sets
        zp = (C.c_void_p * n)(*[zs[s * n + j].ctypes.data for j in range(n)])
        t0 = time.perf_counter()
        ps.check(lib.ps_host_expert_ffn_batch_z(lane, n, zp, mm, r0, H, F, x.ctypes.data, y.ctypes.data))
        if r >= 2:
            ts.append(time.perf_counter() - t0)
    lib.ps_host_lane_destroy(lane)
    ts.sort()
    med = ts[len(ts) // 2]
    zb = float(np.mean(zbytes)) * n
    print(json.dumps({"H": H, "F": F, "n": n, "m": m, "threads": threads, "ms": med * 1e3,
                      "us_per_expert": med * 1e6 / n, "z_gbs": zb / med / 1e9,
                      "bf16_eq_gbs": n * 6.0 * H * F / med / 1e9}))


if __name__ == "__main__":
    main()
