"""K3 decode reading z-slabs directly (ps_expert_ffn_zslab): the consumer warps decode
their MMA fragments from the z bytes in registers instead of a separate decode pass into a
bf16 slot. The fragments equal what a TMA load of the decoded slab delivers, so h and the
split-K partial sums must be BITWISE those of ps_zslab_decode + ps_expert_ffn (which the
oracle tests in test_gpu_ops.py pin), for 3- and 4-bit codes, escape-heavy slabs (zeros,
extreme exponents), ragged down splits and 1-8 tokens per expert."""
import ctypes as C

import numpy as np
import pytest

import paper_2509_23638_b200 as ps

pytestmark = pytest.mark.gpu


def _p(t):
    return C.c_void_p(t.data_ptr())


def _s(torch):
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _tiled_z(lib, H, F, seed, expert, escapes):
    slab = np.empty(3 * H * F, np.uint16)
    ps.check(lib.ps_init_expert_slab_host(slab.ctypes.data, H, F, seed, 0, expert))
    if escapes:  # finite escapes: zeros and tiny / large exponents
        rng = np.random.default_rng(100 + expert)
        idx = rng.choice(slab.size, slab.size // 50, replace=False)
        vals = np.array([0x0000, 0x8000, 0x0001, 0x0080, 0x3f80, 0x4700, 0x0c00, 0xb9a0], np.uint16)
        slab[idx] = vals[rng.integers(0, vals.size, idx.size)]
    tiled = slab.copy()
    ps.check(lib.ps_host_slab_tile(tiled.ctypes.data, H, F))
    cap = lib.ps_zslab_bound(slab.size)
    z = np.zeros(cap, np.uint8)
    nb = C.c_uint64()
    ps.check(lib.ps_zslab_encode_tiled(tiled.ctypes.data, H, F, z.ctypes.data, cap, C.byref(nb), 8))
    return slab, z[:nb.value].copy()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("bits", ["3", "4"])
@pytest.mark.parametrize("H,F,E,k,B,one_hot,escapes", [
    (256, 512, 8, 2, 16, False, True),      # 4 tokens per expert, 2-way down split
    (256, 512, 4, 1, 8, True, True),        # one expert with all 8 tokens, the others idle
    (2048, 1408, 16, 6, 16, False, True),   # DeepSeek-V2-Lite expert: down split 1408 = 2.75 stages
    (2048, 768, 32, 8, 16, False, False),   # Qwen3 expert
    (4096, 14336, 2, 1, 16, False, True),   # Mixtral expert, 4-way split, 8 tokens each
])
def test_zslab_ffn_bitwise_equals_decode_then_ffn(torch_cuda, monkeypatch, bits, H, F, E, k, B, one_hot, escapes):
    torch = torch_cuda
    monkeypatch.setenv("PS_ZSLAB_BITS", bits)
    lib = ps.load()
    ids = np.array([[(t * k + j) % E for j in range(k)] for t in range(B)], np.int32)  # B*k/E tokens each
    if one_hot:
        ids[:] = 1
    counts = np.bincount(ids.ravel(), minlength=E).astype(np.int32)
    zs_d, slabs_d = [], []
    for e in range(E):
        slab, z = _tiled_z(lib, H, F, 3, e, escapes)
        hdr = z[:64].view(np.uint32)
        assert hdr[10] == int(bits) and hdr[11] == 1
        zd = torch.as_tensor(z, device="cuda")
        out = torch.empty(slab.size, dtype=torch.int16, device="cuda")
        ps.check(lib.ps_zslab_decode(_p(zd), z.ctypes.data, _p(out), _s(torch)))
        zs_d.append(zd)
        slabs_d.append(out)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(slabs_d[0].cpu().numpy().view(np.uint16), _tiled_z(lib, H, F, 3, 0, escapes)[0])
    di = torch.as_tensor(ids, device="cuda")
    off = torch.empty(E + 1, dtype=torch.int32, device="cuda")
    src = torch.empty(B * k, dtype=torch.int32, device="cuda")
    inv = torch.empty(B * k, dtype=torch.int32, device="cuda")
    ps.check(lib.ps_permute(_p(di), B, k, E, _p(off), _p(src), _p(inv), None, H, None, _s(torch)))
    x = (torch.randn(B, H, device="cuda", generator=torch.Generator("cuda").manual_seed(3)) / H ** 0.5)
    x = x.to(torch.bfloat16).view(torch.int16)
    grp = ps.capi.ExpertGroup()
    grp.n = E
    zp = (C.c_void_p * E)()
    for e in range(E):
        grp.experts[e] = e
        grp.slabs[e] = slabs_d[e].data_ptr()
        zp[e] = zs_d[e].data_ptr()
    n_split = lib.ps_ffn_down_splits(H, F)
    res = []
    for use_z in (False, True, True):
        h = torch.full((B * k, F), -1, dtype=torch.int16, device="cuda")
        yp = torch.full((n_split, B * k, H), 7.0, dtype=torch.float32, device="cuda")
        if use_z:
            ps.check(lib.ps_expert_ffn_zslab(C.byref(grp), zp, counts.ctypes.data, _p(off), _p(src), k, _p(x), H, F,
                                             _p(h), _p(yp), n_split, B * k, _s(torch)))
        else:
            ps.check(lib.ps_expert_ffn(C.byref(grp), counts.ctypes.data, _p(off), _p(src), k, _p(x), H, F, _p(h),
                                       _p(yp), n_split, B * k, _s(torch)))
        torch.cuda.synchronize()
        res.append((h.cpu(), yp.cpu().view(torch.int32)))
    assert torch.isfinite(res[0][1].view(torch.float32)).all()
    for h, yp in res[1:]:
        assert torch.equal(h, res[0][0])
        assert torch.equal(yp, res[0][1])


def test_zslab_ffn_rejects_unsupported(torch_cuda):
    """Argument checks: > 8 tokens for an expert, H/F not multiples of 64."""
    torch = torch_cuda
    lib = ps.load()
    grp = ps.capi.ExpertGroup()
    grp.n = 1
    grp.experts[0] = 0
    zp = (C.c_void_p * 1)()
    zp[0] = 1
    dummy = torch.zeros(16, device="cuda")
    counts = np.array([9], np.int32)
    st = lib.ps_expert_ffn_zslab(C.byref(grp), zp, counts.ctypes.data, _p(dummy), _p(dummy), 1, _p(dummy), 256, 512,
                                 _p(dummy), _p(dummy), 1, 9, _s(torch))
    assert st != 0 and b"8 tokens" in lib.ps_last_error()
    counts = np.array([4], np.int32)
    st = lib.ps_expert_ffn_zslab(C.byref(grp), zp, counts.ctypes.data, _p(dummy), _p(dummy), 1, _p(dummy), 96, 512,
                                 _p(dummy), _p(dummy), 1, 4, _s(torch))
    assert st != 0 and b"multiples of 64" in lib.ps_last_error()


def test_engine_zfuse_bitwise_equals_decode_pass(torch_cuda, monkeypatch):
    """PS_ZFUSE=1: the engine feeds landed 4-bit-code z-slabs (prefetches and on-demand
    loads) straight to K3 instead of decoding them into the slot first — outputs bitwise
    equal, no z_decode launches (batches of <= 8 tokens per expert)."""
    from paper_2509_23638_b200 import engine as eng
    spec = ps.desk_scale("mixtral", 4, 8, 256)
    spec.expert_bytes = 6 * 256 * 512
    cfg = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    gate, hidden, follow, _ = ps.trace_inputs(cfg, spec, 8, 3)
    outs, stats = [], []
    monkeypatch.setenv("PS_ZSLAB_BITS", "4")  # the engine fuses 4-bit-code slabs only
    for fuse in ("0", "1"):
        monkeypatch.setenv("PS_ZFUSE", fuse)
        with eng.Engine(spec, cfg, budget_fraction=0.25, max_batch=8, weight_seed=9, gate=gate, trace_hidden=hidden,
                        trace_follow=follow, compress_host=True, host_threads=2,
                        cost=(1000, 5, 10, 1e9, 0, 0)) as e:  # host lane priced out: every load on the GPU
            for _ in range(2):
                y, ids = e.step_host(hidden, follow)
            outs.append(y)
            stats.append(e.stats())
            assert e.verify_last_step() == []
    np.testing.assert_array_equal(outs[0], outs[1])
    plain, fused = stats
    loads = plain["ondemand_loads"] + plain["prefetches_committed"]
    assert loads > 0 and plain["z_decodes"] > 0
    if fused["z_decodes"] == plain["z_decodes"]:
        pytest.skip("slabs not in the tiled layout on this host (no AMX lane): PS_ZFUSE inactive")
    assert fused["z_decodes"] == 0
