"""Stand-alone K5 expert cache (ps_cache_*): resident experts from the
HBM arena, the others through staging slots loaded by the serial copy channel; the
slab a caller acquires computes exactly what the same weights uploaded directly compute
(K3 on both, bitwise); prefetch / on-demand / hit / LRU reuse / overflow / cancel."""
import ctypes as C

import numpy as np
import pytest

import oracle as orc
import paper_2509_23638_b200 as ps

pytestmark = pytest.mark.gpu
H, F, L, E = 256, 512, 2, 4


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


class _Cache:
    def __init__(self, torch, n_slots, resident=()):
        self.lib = ps.load()
        self.host = []
        for l in range(L):
            for e in range(E):
                self.host.append(torch.from_numpy(orc.or_init_slab(H, F, 3, l, e).view(np.int16)).pin_memory())
        self.ptrs = (C.c_void_p * (L * E))(*[t.data_ptr() for t in self.host])
        res = np.array(list(resident), np.int32).reshape(-1)
        self.res = res
        cfg = ps.capi.CacheConfig(L, E, 6 * H * F, self.ptrs, res.ctypes.data_as(C.POINTER(C.c_int32)) if len(res)
                                  else None, len(res) // 2, 6 * H * F * max(1, len(res) // 2), n_slots, 0)
        self.h = C.c_void_p()
        ps.check(self.lib.ps_cache_create(C.byref(cfg), C.byref(self.h)))

    def __getattr__(self, name):  # ps_cache_<name>(h, ...)
        fn = getattr(self.lib, "ps_cache_" + name)
        return lambda *a: fn(self.h, *a)

    def stats(self):
        s = ps.capi.CacheStats()
        ps.check(self.lib.ps_cache_get_stats(self.h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in ps.capi.CacheStats._fields_}


def _ffn(torch, slab_ptr, x):
    """K3 on one expert slab (device pointer) for the rows x [m, H] bf16 -> y [m, H]."""
    lib = ps.load()
    m = x.shape[0]
    grp = ps.capi.ExpertGroup()
    grp.n = 1
    grp.experts[0] = 0
    grp.slabs[0] = slab_ptr
    counts = np.array([m], np.int32)
    off = torch.tensor([0, m], dtype=torch.int32, device="cuda")
    src = torch.arange(m, dtype=torch.int32, device="cuda")
    h = torch.empty(m, F, dtype=torch.int16, device="cuda")
    yp = torch.empty(1, m, H, dtype=torch.float32, device="cuda")
    ps.check(lib.ps_expert_ffn(C.byref(grp), counts.ctypes.data, _p(off), _p(src), 1, _p(x), H, F, _p(h), _p(yp), 1, m,
                               C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    return yp[0].cpu().numpy()


def test_cache_prefetch_ondemand_acquire_release(torch_cuda):
    torch = torch_cuda
    c = _Cache(torch, n_slots=2, resident=[(0, 0)])
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    x = torch.as_tensor(orc.f32_to_bf16(np.random.default_rng(0).standard_normal((5, H)).astype(np.float32) / 16)
                        .view(np.int16), device="cuda")

    def check(l, e):
        p = C.c_void_p()
        ps.check(c.acquire(l, e, s, C.byref(p)))
        got = _ffn(torch, p.value, x)
        direct = c.host[l * E + e].cuda()
        assert np.array_equal(got, _ffn(torch, direct.data_ptr(), x)), (l, e)
        return p.value

    try:
        ps.check(c.prefetch(0, 1))
        ps.check(c.ondemand(0, 2))
        a, b = check(0, 1), check(0, 2)
        assert a != b
        ps.check(c.release(0, 1, s))
        ps.check(c.release(0, 2, s))
        ps.check(c.prefetch(0, 1))          # still in its slot: a hit, no copy
        assert c.stats()["slot_hits"] == 1
        ps.check(c.prefetch(0, 0))          # resident: served from the arena
        res = check(0, 0)
        assert res not in (a, b)
        ps.check(c.release(0, 0, s))
        ps.check(c.ondemand(1, 3))          # LRU reuse of one of the two slots
        check(1, 3)
        ps.check(c.ondemand(1, 1))
        check(1, 1)                         # both slots pinned now
        assert c.prefetch(1, 2) == ps.capi.PS_ERUNTIME  # no free slot: the simulator's overflow
        ps.check(c.release(1, 3, s))
        ps.check(c.release(1, 1, s))
        ps.check(c.prefetch(1, 2))
        check(1, 2)
        ps.check(c.release(1, 2, s))
        assert c.acquire(1, 0, s, C.byref(C.c_void_p())) == ps.capi.PS_EINVAL  # never requested
        assert c.release(1, 0, s) == ps.capi.PS_EINVAL
        assert c.prefetch(2, 0) == ps.capi.PS_ERANGE
        st = c.stats()
        assert st["ondemand_loads"] == 3 and st["prefetches"] >= 2 and st["resident_hits"] >= 1
        ps.check(c.sync())
    finally:
        ps.check(c.destroy())


def test_cache_cancel_queued_prefetches(torch_cuda):
    torch = torch_cuda
    c = _Cache(torch, n_slots=6)
    try:
        for e in range(E):
            ps.check(c.prefetch(1, e))
        n = C.c_int()
        ps.check(c.cancel_prefetches(C.byref(n)))
        ps.check(c.sync())
        st = c.stats()
        assert 0 <= n.value <= E and st["prefetches_cancelled"] == n.value
        s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        ok = 0
        for e in range(E):  # issued copies stay acquirable, cancelled ones are gone
            r = c.acquire(1, e, s, C.byref(C.c_void_p()))
            assert r in (ps.capi.PS_OK, ps.capi.PS_EINVAL)
            ok += r == ps.capi.PS_OK
        assert ok == E - n.value
    finally:
        ps.check(c.destroy())
