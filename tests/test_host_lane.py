"""Host expert lane (Resource::Cpu of the reference, simulator.cpp:139-146): the
AVX512-BF16 / AMX-BF16 SwiGLU of ps_host_expert_ffn vs the f64 CPU oracle
(or_expert_ffn, h rounded to bf16 like K3) at the bf16 tolerance. CPU-only tests: the
lane runs on the host, no GPU involved."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle as orc
import paper_2509_23638_b200 as ps

BF16_RTOL = 2e-2


def _has(flag):
    try:
        return flag in open("/proc/cpuinfo").read()
    except OSError:
        return False


needs_bf16 = pytest.mark.skipif(not _has("avx512_bf16"), reason="host CPU lacks AVX512_BF16")


def _lane(threads, isa):
    old = os.environ.get("PS_HOST_LANE_ISA")
    if isa == "avx512":
        os.environ["PS_HOST_LANE_ISA"] = "avx512"
    try:
        h = C.c_void_p()
        ps.check(ps.load().ps_host_lane_create(threads, C.byref(h)))
    finally:
        if old is None:
            os.environ.pop("PS_HOST_LANE_ISA", None)
        else:
            os.environ["PS_HOST_LANE_ISA"] = old
    return h


ISAS = ["avx512"] + (["amx"] if _has("amx_bf16") else [])


@needs_bf16
@pytest.mark.parametrize("isa", ISAS)
@pytest.mark.parametrize("H,F,m", [(256, 512, 1), (256, 512, 5), (256, 512, 16), (256, 512, 17),
                                   (512, 768, 33), (2048, 1408, 3)])
def test_host_expert_ffn_matches_oracle(isa, H, F, m):
    lib = ps.load()
    lane = _lane(3, isa)
    try:
        want = 2 if isa == "amx" else 1
        assert lib.ps_host_lane_isa(lane) == want
        slab = orc.or_init_slab(H, F, 5, 1, 2)
        rng = np.random.default_rng(H + m)
        x = orc.f32_to_bf16(rng.standard_normal((m, H)).astype(np.float32))
        y = np.full((m, H), np.nan, np.float32)
        ps.check(lib.ps_host_expert_ffn(lane, slab.ctypes.data, H, F, x.ctypes.data, m, y.ctypes.data))
        yr = np.empty((m, H), np.float32)
        orc.oracle_lib().or_expert_ffn(slab.ctypes.data, H, F, m, x.ctypes.data, yr.ctypes.data, 1)
        assert np.isfinite(y).all()
        for t in range(m):  # per token: padding rows of a 16-token AMX group must not leak
            assert np.linalg.norm(y[t] - yr[t]) / np.linalg.norm(yr[t]) < BF16_RTOL
    finally:
        lib.ps_host_lane_destroy(lane)


@needs_bf16
def test_host_lane_isas_agree_and_threads_invariant():
    """Row partitioning over threads does not change any value (each output element is
    one thread's fixed-order sum); the two ISAs agree at the bf16 tolerance."""
    lib = ps.load()
    H, F, m = 512, 1024, 9
    slab = orc.or_init_slab(H, F, 1, 0, 0)
    x = orc.f32_to_bf16(np.random.default_rng(0).standard_normal((m, H)).astype(np.float32))
    outs = {}
    for isa in ISAS:
        for threads in (1, 4):
            lane = _lane(threads, isa)
            y = np.empty((m, H), np.float32)
            ps.check(lib.ps_host_expert_ffn(lane, slab.ctypes.data, H, F, x.ctypes.data, m, y.ctypes.data))
            lib.ps_host_lane_destroy(lane)
            outs[(isa, threads)] = y
    for isa in ISAS:
        np.testing.assert_array_equal(outs[(isa, 1)], outs[(isa, 4)])
    a, b = outs[(ISAS[0], 1)], outs[(ISAS[-1], 1)]
    assert np.linalg.norm(a - b) / np.linalg.norm(b) < BF16_RTOL


@needs_bf16
def test_host_lane_argument_errors():
    lib = ps.load()
    lane = _lane(1, "avx512")
    try:
        y = np.empty(64, np.float32)
        x = np.zeros(64, np.uint16)
        slab = np.zeros(3 * 48 * 64, np.uint16)
        assert lib.ps_host_expert_ffn(lane, slab.ctypes.data, 48, 64, x.ctypes.data, 1, y.ctypes.data) == ps.capi.PS_EINVAL
        assert lib.ps_host_expert_ffn(lane, slab.ctypes.data, 64, 64, x.ctypes.data, 0, y.ctypes.data) == ps.capi.PS_OK
        assert lib.ps_host_expert_ffn(lane, None, 64, 64, x.ctypes.data, 1, y.ctypes.data) == ps.capi.PS_EINVAL
    finally:
        lib.ps_host_lane_destroy(lane)
    h = C.c_void_p()
    assert lib.ps_host_lane_create(0, C.byref(h)) == ps.capi.PS_EINVAL


@needs_bf16
@pytest.mark.parametrize("isa", ISAS)
def test_host_expert_ffn_batch_equals_single_calls(isa):
    """A layer's cpu_set in one batch call (rows [row0, row0+m) of shared x/y buffers)
    gives bitwise the per-expert results."""
    lib = ps.load()
    H, F = 256, 384
    ms, row0 = [3, 0, 17, 1], [0, 3, 3, 20]
    slabs = [orc.or_init_slab(H, F, 2, 0, e) for e in range(4)]
    x = orc.f32_to_bf16(np.random.default_rng(7).standard_normal((21, H)).astype(np.float32))
    lane = _lane(4, isa)
    try:
        y = np.full((21, H), np.nan, np.float32)
        arr = (C.c_void_p * 4)(*[s.ctypes.data for s in slabs])
        m_a, r_a = np.array(ms, np.int32), np.array(row0, np.int32)
        ps.check(lib.ps_host_expert_ffn_batch(lane, 4, arr, m_a.ctypes.data, r_a.ctypes.data, H, F, x.ctypes.data,
                                              y.ctypes.data))
        for j in range(4):
            if ms[j] == 0:
                continue
            yj = np.empty((ms[j], H), np.float32)
            ps.check(lib.ps_host_expert_ffn(lane, slabs[j].ctypes.data, H, F, x[row0[j]:].ctypes.data, ms[j],
                                            yj.ctypes.data))
            np.testing.assert_array_equal(y[row0[j]:row0[j] + ms[j]], yj)
    finally:
        lib.ps_host_lane_destroy(lane)


@needs_bf16
@pytest.mark.skipif(not (_has("amx_bf16") and _has("avx512_vbmi2")), reason="z-slab lane path needs AMX-BF16 + VBMI2")
@pytest.mark.parametrize("bits", [3, 4])
@pytest.mark.parametrize("escapes", [0, 3000, 90000])
def test_host_lane_reads_zslabs_bitwise(bits, escapes, monkeypatch):
    """The lane's z-slab path (3- or 4-bit exponent codes decoded per tile, rows starting
    mid-block) gives bitwise the raw-slab results, escapes included (up to ~30 % of the
    values, so segments with many escapes and blocks with long escape lists)."""
    monkeypatch.setenv("PS_ZSLAB_BITS", str(bits))
    lib = ps.load()
    H, F = 256, 384
    ms, row0 = [3, 17, 1], [0, 3, 20]
    slabs, zs = [], []
    rng = np.random.default_rng(11)
    for e in range(3):
        s = orc.or_init_slab(H, F, 2, 1, e)
        if escapes:
            idx = rng.choice(s.size, escapes, replace=False)
            s[idx] = (rng.integers(0, 2, idx.size) << 15 | rng.integers(1, 200, idx.size) << 7 |
                      rng.integers(0, 128, idx.size)).astype(np.uint16)  # finite, wide exponents
        slabs.append(s)
        cap = lib.ps_zslab_bound(s.size)
        z = np.zeros(cap, np.uint8)
        nb = C.c_uint64()
        ps.check(lib.ps_zslab_encode(s.ctypes.data, s.size, z.ctypes.data, cap, C.byref(nb), 2))
        assert z[40:44].view(np.uint32)[0] == bits  # ZHeader.code_bits
        zs.append(z)
    x = orc.f32_to_bf16(rng.standard_normal((21, H)).astype(np.float32))
    lane = _lane(3, "amx")
    try:
        m_a, r_a = np.array(ms, np.int32), np.array(row0, np.int32)
        y_raw = np.full((21, H), np.nan, np.float32)
        y_z = np.full((21, H), np.nan, np.float32)
        ps.check(lib.ps_host_expert_ffn_batch(lane, 3, (C.c_void_p * 3)(*[s.ctypes.data for s in slabs]),
                                              m_a.ctypes.data, r_a.ctypes.data, H, F, x.ctypes.data, y_raw.ctypes.data))
        ps.check(lib.ps_host_expert_ffn_batch_z(lane, 3, (C.c_void_p * 3)(*[z.ctypes.data for z in zs]),
                                                m_a.ctypes.data, r_a.ctypes.data, H, F, x.ctypes.data, y_z.ctypes.data))
        np.testing.assert_array_equal(y_raw, y_z)
    finally:
        lib.ps_host_lane_destroy(lane)


@needs_bf16
@pytest.mark.skipif(not _has("amx_bf16"), reason="tile layout path needs AMX-BF16")
def test_host_lane_tile_layout_bitwise():
    """ps_host_slab_tile + ps_host_expert_ffn_batch_tiled give bitwise the row-major
    batch results (same tile ops in the same order), token groups of 1..17 included."""
    lib = ps.load()
    H, F = 256, 384
    ms, row0 = [1, 17, 0, 5], [0, 1, 18, 18]
    slabs = [orc.or_init_slab(H, F, 3, 2, e) for e in range(4)]
    tiled = [s.copy() for s in slabs]
    for t in tiled:
        ps.check(lib.ps_host_slab_tile(t.ctypes.data, H, F))
    assert not np.array_equal(tiled[0], slabs[0])  # the layout did change
    rng = np.random.default_rng(3)
    x = orc.f32_to_bf16(rng.standard_normal((23, H)).astype(np.float32))
    lane = _lane(3, "amx")
    try:
        m_a, r_a = np.array(ms, np.int32), np.array(row0, np.int32)
        y_raw = np.full((23, H), np.nan, np.float32)
        y_t = np.full((23, H), np.nan, np.float32)
        ps.check(lib.ps_host_expert_ffn_batch(lane, 4, (C.c_void_p * 4)(*[s.ctypes.data for s in slabs]),
                                              m_a.ctypes.data, r_a.ctypes.data, H, F, x.ctypes.data, y_raw.ctypes.data))
        ps.check(lib.ps_host_expert_ffn_batch_tiled(lane, 4, (C.c_void_p * 4)(*[s.ctypes.data for s in tiled]),
                                                    m_a.ctypes.data, r_a.ctypes.data, H, F, x.ctypes.data,
                                                    y_t.ctypes.data))
        np.testing.assert_array_equal(y_raw, y_t)
    finally:
        lib.ps_host_lane_destroy(lane)


@needs_bf16
@pytest.mark.skipif(not (_has("amx_bf16") and _has("avx512_vbmi2")), reason="z-slab lane path needs AMX-BF16 + VBMI2")
@pytest.mark.parametrize("bits", [3, 4])
def test_host_lane_reads_tiled_zslabs_bitwise(bits, monkeypatch):
    """z-slabs of tile-layout slabs (ps_zslab_encode_tiled): the lane's sequential z path
    gives bitwise the row-major raw results; the slab round-trips through untile."""
    monkeypatch.setenv("PS_ZSLAB_BITS", str(bits))
    lib = ps.load()
    H, F = 256, 384
    ms, row0 = [2, 16, 1], [0, 2, 18]
    rng = np.random.default_rng(5)
    slabs, zs = [], []
    for e in range(3):
        s = orc.or_init_slab(H, F, 4, 0, e)
        idx = rng.choice(s.size, 20000, replace=False)
        s[idx] = (rng.integers(0, 2, idx.size) << 15 | rng.integers(1, 255, idx.size) << 7 |
                  rng.integers(0, 128, idx.size)).astype(np.uint16)
        slabs.append(s)
        t = s.copy()
        ps.check(lib.ps_host_slab_tile(t.ctypes.data, H, F))
        back = t.copy()
        ps.check(lib.ps_host_slab_untile(back.ctypes.data, H, F))
        np.testing.assert_array_equal(back, s)
        cap = lib.ps_zslab_bound(s.size)
        z = np.zeros(cap, np.uint8)
        nb = C.c_uint64()
        ps.check(lib.ps_zslab_encode_tiled(t.ctypes.data, H, F, z.ctypes.data, cap, C.byref(nb), 2))
        assert z[40:44].view(np.uint32)[0] == bits and z[44:48].view(np.uint32)[0] == 1
        zs.append(z)
    x = orc.f32_to_bf16(rng.standard_normal((19, H)).astype(np.float32))
    lane = _lane(3, "amx")
    try:
        m_a, r_a = np.array(ms, np.int32), np.array(row0, np.int32)
        y_raw = np.full((19, H), np.nan, np.float32)
        y_z = np.full((19, H), np.nan, np.float32)
        ps.check(lib.ps_host_expert_ffn_batch(lane, 3, (C.c_void_p * 3)(*[s.ctypes.data for s in slabs]),
                                              m_a.ctypes.data, r_a.ctypes.data, H, F, x.ctypes.data, y_raw.ctypes.data))
        ps.check(lib.ps_host_expert_ffn_batch_z(lane, 3, (C.c_void_p * 3)(*[z.ctypes.data for z in zs]),
                                                m_a.ctypes.data, r_a.ctypes.data, H, F, x.ctypes.data, y_z.ctypes.data))
        np.testing.assert_array_equal(y_raw, y_z)
    finally:
        lib.ps_host_lane_destroy(lane)


@needs_bf16
@pytest.mark.skipif(not (_has("amx_bf16") and _has("avx512_vbmi2")), reason="z-slab lane path needs AMX-BF16 + VBMI2")
def test_host_lane_full_mixtral_expert_tiled_z_vs_oracle():
    """The bench's lane configuration at the bench's shape: one Mixtral expert (H=4096,
    F=14336) in the tile layout, read as a 3-bit tiled z-slab (ps_host_expert_ffn_batch_z,
    the engine's default) — bitwise equal to the tiled raw path, and per token within the
    bf16 tolerance of the f64 oracle (4 decode tokens, as a B=16 step routes ~4 per expert)."""
    lib = ps.load()
    H, F, m = 4096, 14336, 4
    s = orc.or_init_slab(H, F, 1, 3, 5)
    t = s.copy()
    ps.check(lib.ps_host_slab_tile(t.ctypes.data, H, F))
    cap = lib.ps_zslab_bound(s.size)
    z = np.zeros(cap, np.uint8)
    nb = C.c_uint64()
    ps.check(lib.ps_zslab_encode_tiled(t.ctypes.data, H, F, z.ctypes.data, cap, C.byref(nb), 0))
    assert z[40:44].view(np.uint32)[0] == 3  # the encoder picks 3-bit codes on these weights
    x = orc.f32_to_bf16((np.random.default_rng(1).standard_normal((m, H)) / np.sqrt(H)).astype(np.float32))
    lane = _lane(os.cpu_count() or 1, "amx")
    try:
        ma, ra = np.array([m], np.int32), np.array([0], np.int32)
        y_t = np.full((m, H), np.nan, np.float32)
        y_z = np.full((m, H), np.nan, np.float32)
        ps.check(lib.ps_host_expert_ffn_batch_tiled(lane, 1, (C.c_void_p * 1)(t.ctypes.data), ma.ctypes.data,
                                                    ra.ctypes.data, H, F, x.ctypes.data, y_t.ctypes.data))
        ps.check(lib.ps_host_expert_ffn_batch_z(lane, 1, (C.c_void_p * 1)(z.ctypes.data), ma.ctypes.data,
                                                ra.ctypes.data, H, F, x.ctypes.data, y_z.ctypes.data))
        np.testing.assert_array_equal(y_t, y_z)
    finally:
        lib.ps_host_lane_destroy(lane)
    yr = np.empty((m, H), np.float32)
    orc.oracle_lib().or_expert_ffn(s.ctypes.data, H, F, m, x.ctypes.data, yr.ctypes.data, 1)
    for tok in range(m):
        assert np.linalg.norm(y_z[tok] - yr[tok]) / np.linalg.norm(yr[tok]) < BF16_RTOL
