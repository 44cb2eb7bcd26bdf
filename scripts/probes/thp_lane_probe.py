"""Host-lane bandwidth on pinned memory from cudaHostAlloc (4 KiB pages) vs an anonymous
mmap with MADV_HUGEPAGE (transparent 2 MiB pages) registered with cudaHostRegister.
The lane streams 352 MB per expert with 12 threads: 4 KiB pages cost a TLB miss every
4 KiB per stream."""
import ctypes as C
import json
import pathlib
import sys
import time

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[2]))
import paper_2509_23638_b200 as ps  # noqa: E402

libc = C.CDLL("libc.so.6", use_errno=True)
libc.mmap.restype = C.c_void_p
libc.mmap.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_long]
libc.madvise.argtypes = [C.c_void_p, C.c_size_t, C.c_int]


def thp_alloc(nbytes):
    addr = libc.mmap(None, nbytes, 3, 0x22, -1, 0)  # PROT_READ|WRITE, MAP_PRIVATE|ANONYMOUS
    assert addr not in (None, C.c_void_p(-1).value)
    rc = libc.madvise(addr, nbytes, 14)  # MADV_HUGEPAGE
    return addr, rc


def main():
    print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(), flush=True)
    lib = ps.load()
    H, F = 4096, 14336
    nbytes = 6 * H * F
    cudart = torch.cuda.cudart()
    torch.cuda.init()
    res = {}
    for kind in ("cudaHostAlloc", "thp+register"):
        slabs = []
        for e in range(4):
            if kind == "cudaHostAlloc":
                t = torch.empty(nbytes // 2, dtype=torch.int16).pin_memory()
                slabs.append((t, t.data_ptr()))
            else:
                addr, rc = thp_alloc(nbytes)
                ps.check(lib.ps_init_expert_slab_host(C.c_void_p(addr), H, F, 1, 0, e))  # touch
                err = cudart.cudaHostRegister(addr, nbytes, 0)
                slabs.append((None, addr))
                res["madvise_rc"] = rc
                res["register_err"] = int(err) if not isinstance(err, tuple) else int(err[0])
            if kind == "cudaHostAlloc":
                ps.check(lib.ps_init_expert_slab_host(C.c_void_p(slabs[-1][1]), H, F, 1, 0, e))
        meminfo = {l.split(":")[0]: l.split(":")[1].strip() for l in open("/proc/meminfo") if "Huge" in l}
        lane = C.c_void_p()
        ps.check(lib.ps_host_lane_create(12, C.byref(lane)))
        x = np.zeros((16, H), np.uint16)
        y = np.zeros((16, H), np.float32)
        for m in (4, 16):
            ts = []
            for r in range(8):
                t0 = time.perf_counter()
                ps.check(lib.ps_host_expert_ffn(lane, C.c_void_p(slabs[r % 4][1]), H, F, x.ctypes.data, m,
                                                y.ctypes.data))
                ts.append(time.perf_counter() - t0)
            ts.sort()
            res[f"{kind}_m{m}_gbs"] = nbytes / ts[4] / 1e9
        res[f"{kind}_meminfo"] = meminfo
        lib.ps_host_lane_destroy(lane)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
