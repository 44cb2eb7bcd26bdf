"""K3 prefill path (tcgen05 / TMEM / TMA grouped GEMM) vs the CPU oracle and vs the
decode path (itself oracle-checked), at ragged per-expert row counts."""
import ctypes as C

import numpy as np
import pytest

import oracle as orc
import paper_2509_23638_b200 as ps

pytestmark = pytest.mark.gpu
BF16_RTOL = 2e-2


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _last_tile_tokens(offsets, perm_src, k):
    """Tokens owning, for every expert, the last routed row, the first row of its last
    128-row M tile (single-CTA kernel) and the first row the second CTA of its last
    256-row pair tile computes (local rows 256*j + 128), when those exist."""
    rows = []
    for e in range(len(offsets) - 1):
        m = int(offsets[e + 1] - offsets[e])
        if m == 0:
            continue
        local = {m - 1, (m - 1) // 128 * 128}
        r2 = (m - 1) // 256 * 256 + 128
        if r2 < m:
            local.add(r2)
        rows += [int(offsets[e]) + r for r in local]
    return np.unique(perm_src[np.array(rows)] // k)


def _prefill_case(torch, H, F, E, k, B, seed, skew=None, check_oracle_rows=None, with_decode=True, last_tiles=False):
    lib = ps.load()
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    rng = np.random.default_rng(seed)
    ids = np.stack([rng.choice(E, k, replace=False) for _ in range(B)]).astype(np.int32)
    if skew is not None:
        ids[: B // 2, 0] = skew
        for t in range(B // 2):
            if skew in ids[t, 1:]:
                ids[t, 1:] = [(skew + 1 + j) % E for j in range(k - 1)]
    logits = rng.standard_normal((B, E))
    gw = np.exp(logits - logits.max(1, keepdims=True))
    gw /= gw.sum(1, keepdims=True)
    x = orc.f32_to_bf16((rng.standard_normal((B, H)) / np.sqrt(H)).astype(np.float32))
    slabs_d = []
    for e in range(E):
        t = torch.empty(3 * H * F, dtype=torch.int16, device="cuda")
        ps.check(lib.ps_init_expert_slab(_p(t), H, F, seed, 0, e, s))
        slabs_d.append(t)
    rows = B * k
    di = torch.as_tensor(ids, device="cuda")
    dx = torch.as_tensor(x.view(np.int16), device="cuda")
    off = torch.empty(E + 1, dtype=torch.int32, device="cuda")
    src = torch.empty(rows, dtype=torch.int32, device="cuda")
    inv = torch.empty(rows, dtype=torch.int32, device="cuda")
    xp = torch.empty(rows, H, dtype=torch.int16, device="cuda")
    ps.check(lib.ps_permute(_p(di), B, k, E, _p(off), _p(src), _p(inv), _p(dx), H, _p(xp), s))
    counts = np.bincount(ids.ravel(), minlength=E).astype(np.int32)
    offsets = off.cpu().numpy()
    grp = ps.capi.ExpertGroup()
    grp.n = E
    for e in range(E):
        grp.experts[e] = e
        grp.slabs[e] = slabs_d[e].data_ptr()
    h = torch.empty(rows, F, dtype=torch.int16, device="cuda")
    yp = torch.full((rows, H), float("nan"), dtype=torch.float32, device="cuda")
    ps.check(lib.ps_expert_ffn_prefill(C.byref(grp), counts.ctypes.data, offsets.ctypes.data, _p(xp), rows, H, F,
                                       _p(h), _p(yp), s))
    y = torch.empty(B, H, dtype=torch.float32, device="cuda")
    dw = torch.as_tensor(gw.astype(np.float32), device="cuda")
    ps.check(lib.ps_combine(_p(yp), 1, _p(inv), _p(di), _p(dw), B, k, E, H, _p(y), s))
    y = y.cpu().numpy()
    out = {"y": y}
    if with_decode:  # decode path on the same inputs
        h2 = torch.empty(rows, F, dtype=torch.int16, device="cuda")
        yp2 = torch.empty(1, rows, H, dtype=torch.float32, device="cuda")
        ps.check(lib.ps_expert_ffn(C.byref(grp), counts.ctypes.data, _p(off), _p(src), k, _p(dx), H, F, _p(h2),
                                   _p(yp2), 1, rows, s))
        y2 = torch.empty(B, H, dtype=torch.float32, device="cuda")
        ps.check(lib.ps_combine(_p(yp2), 1, _p(inv), _p(di), _p(dw), B, k, E, H, _p(y2), s))
        out["y_decode"] = y2.cpu().numpy()
    if check_oracle_rows:
        sel = np.arange(min(B, check_oracle_rows))
        if last_tiles:  # + every expert's last rows: its last 128-row tile, the 2nd CTA of its last pair tile
            sel = np.union1d(sel, _last_tile_tokens(offsets, src.cpu().numpy(), k))
        slabs_h = [t.cpu().numpy().view(np.uint16) if e in set(ids[sel].ravel()) else None
                   for e, t in enumerate(slabs_d)]
        out["y_oracle"] = orc.or_moe_layer(slabs_h, H, F, x[sel], ids[sel], gw[sel].astype(np.float32), True)
        out["sel"] = sel
    return out


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.fixture(params=[0, 1, 3], ids=["single_cta", "cta_pair", "token_n_pair"])
def prefill_kernel(request):
    """Every tcgen05 kernel explicitly (ps_set_prefill_kernel), auto mode restored after."""
    lib = ps.load()
    ps.check(lib.ps_set_prefill_kernel(request.param))
    yield request.param
    ps.check(lib.ps_set_prefill_kernel(2))


@pytest.mark.parametrize("H,F,E,k,B,skew", [(256, 512, 8, 2, 512, None), (256, 384, 8, 2, 300, 3),
                                             (512, 1024, 16, 4, 160, None), (256, 256, 4, 1, 1, None)])
def test_prefill_vs_oracle_small(torch_cuda, prefill_kernel, H, F, E, k, B, skew):
    out = _prefill_case(torch_cuda, H, F, E, k, B, 7, skew, check_oracle_rows=B)
    assert np.isfinite(out["y"]).all()
    assert _rel(out["y"], out["y_oracle"]) < BF16_RTOL
    assert _rel(out["y"], out["y_decode"]) < BF16_RTOL


def test_prefill_deepseek_shape(torch_cuda, prefill_kernel):
    """DeepSeek-V2-Lite expert shape (H=2048, F=1408), 64 experts top-6, 2k-token chunk;
    oracle rows include every expert's last (padded) M tile and 2nd pair CTA."""
    out = _prefill_case(torch_cuda, 2048, 1408, 64, 6, 2048, 3, check_oracle_rows=6, last_tiles=True)
    assert _rel(out["y"], out["y_decode"]) < BF16_RTOL
    sel = out["sel"]
    for i, t in enumerate(sel):  # per token: a bad padded-tile row cannot hide in a norm over many rows
        assert _rel(out["y"][t], out["y_oracle"][i]) < BF16_RTOL, t


def test_prefill_mixtral_shape(torch_cuda, prefill_kernel):
    """Mixtral expert shape (H=4096, F=14336), 8 experts top-2, 1k tokens (m_e ~ 256);
    oracle rows include every expert's last (padded) M tile and 2nd pair CTA."""
    out = _prefill_case(torch_cuda, 4096, 14336, 8, 2, 1024, 5, check_oracle_rows=2, last_tiles=True)
    assert _rel(out["y"], out["y_decode"]) < BF16_RTOL
    sel = out["sel"]
    for i, t in enumerate(sel):  # per token: a bad padded-tile row cannot hide in a norm over many rows
        assert _rel(out["y"][t], out["y_oracle"][i]) < BF16_RTOL, t


def _explicit_counts_case(torch, H, F, counts, seed, reps=1):
    """k = 1 routing with exactly counts[e] tokens on expert e; y of the prefill path
    (every launch of `reps`) and the oracle on all rows."""
    lib = ps.load()
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    E = len(counts)
    rng = np.random.default_rng(seed)
    ids = rng.permutation(np.repeat(np.arange(E, dtype=np.int32), counts))[:, None].copy()
    B = ids.shape[0]
    x = orc.f32_to_bf16((rng.standard_normal((B, H)) / np.sqrt(H)).astype(np.float32))
    slabs_d = []
    for e in range(E):
        t = torch.empty(3 * H * F, dtype=torch.int16, device="cuda")
        ps.check(lib.ps_init_expert_slab(_p(t), H, F, seed, 0, e, s))
        slabs_d.append(t)
    di = torch.as_tensor(ids, device="cuda")
    dx = torch.as_tensor(x.view(np.int16), device="cuda")
    off = torch.empty(E + 1, dtype=torch.int32, device="cuda")
    src = torch.empty(B, dtype=torch.int32, device="cuda")
    inv = torch.empty(B, dtype=torch.int32, device="cuda")
    xp = torch.empty(B, H, dtype=torch.int16, device="cuda")
    ps.check(lib.ps_permute(_p(di), B, 1, E, _p(off), _p(src), _p(inv), _p(dx), H, _p(xp), s))
    cnt = np.asarray(counts, dtype=np.int32)
    offsets = off.cpu().numpy()
    grp = ps.capi.ExpertGroup()
    grp.n = E
    for e in range(E):
        grp.experts[e] = e
        grp.slabs[e] = slabs_d[e].data_ptr()
    h = torch.empty(B, F, dtype=torch.int16, device="cuda")
    gate = np.zeros((B, E), np.float32)
    gate[np.arange(B), ids[:, 0]] = 1.0
    ones = torch.as_tensor(gate, device="cuda")
    ys = []
    for _ in range(reps):
        yp = torch.full((B, H), float("nan"), dtype=torch.float32, device="cuda")
        ps.check(lib.ps_expert_ffn_prefill(C.byref(grp), cnt.ctypes.data, offsets.ctypes.data, _p(xp), B, H, F,
                                           _p(h), _p(yp), s))
        y = torch.empty(B, H, dtype=torch.float32, device="cuda")
        ps.check(lib.ps_combine(_p(yp), 1, _p(inv), _p(di), _p(ones), B, 1, E, H, _p(y), s))
        ys.append(y.cpu().numpy())
    slabs_h = [t.cpu().numpy().view(np.uint16) for t in slabs_d]
    y_ref = orc.or_moe_layer(slabs_h, H, F, x, ids, gate, True)
    return ys, y_ref


def test_prefill_token_n_ragged_counts(torch_cuda):
    """Token-N kernel at every N-tile boundary case: 1, 15, 16, 17, 255, 256, 257, 300,
    513 rows (last token tile N = 16 .. 256, 1-3 token tiles per expert), one launch for
    gate_up + down; every row vs the oracle, and the launch repeated 70 times (map-ring
    slots reused: the per-slot gate_up counters only grow) with bit-identical outputs."""
    lib = ps.load()
    ps.check(lib.ps_set_prefill_kernel(3))
    try:
        ys, y_ref = _explicit_counts_case(torch_cuda, 256, 384, [1, 15, 16, 17, 255, 256, 257, 300, 513], 11, reps=70)
    finally:
        ps.check(lib.ps_set_prefill_kernel(2))
    for t in range(y_ref.shape[0]):
        assert _rel(ys[0][t], y_ref[t]) < BF16_RTOL, t
    for y in ys[1:]:
        assert np.array_equal(y, ys[0])


@pytest.mark.parametrize("H,F,E,k,B", [(2048, 1408, 64, 6, 2048), (256, 384, 9, 1, 1500), (512, 512, 16, 4, 300)])
def test_prefill_device_schedule_matches_host_schedule(torch_cuda, H, F, E, k, B):
    """ps_expert_ffn_prefill_dev (tile schedule built on the device from K2's offsets, the
    engine's early resident-group launch) gives bitwise the h / y of the host-count call,
    with experts that get no rows in the group (they cost nothing) and ragged counts."""
    torch = torch_cuda
    lib = ps.load()
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    rng = np.random.default_rng(B + E)
    p = rng.dirichlet(np.ones(E) * 0.3)
    p[E // 3] = 0.0  # an expert nobody routes to
    p /= p.sum()
    ids = np.stack([rng.choice(E, k, replace=False, p=p) for _ in range(B)]).astype(np.int32)
    x = orc.f32_to_bf16((rng.standard_normal((B, H)) / np.sqrt(H)).astype(np.float32))
    slabs = []
    for e in range(E):
        t = torch.empty(3 * H * F, dtype=torch.int16, device="cuda")
        ps.check(lib.ps_init_expert_slab(_p(t), H, F, 5, 0, e, s))
        slabs.append(t)
    rows = B * k
    di = torch.as_tensor(ids, device="cuda")
    dx = torch.as_tensor(x.view(np.int16), device="cuda")
    off = torch.empty(E + 1, dtype=torch.int32, device="cuda")
    src = torch.empty(rows, dtype=torch.int32, device="cuda")
    inv = torch.empty(rows, dtype=torch.int32, device="cuda")
    xp = torch.empty(rows, H, dtype=torch.int16, device="cuda")
    ps.check(lib.ps_permute(_p(di), B, k, E, _p(off), _p(src), _p(inv), _p(dx), H, _p(xp), s))
    counts = np.bincount(ids.ravel(), minlength=E).astype(np.int32)
    offsets = off.cpu().numpy()
    grp = ps.capi.ExpertGroup()
    grp.n = E
    for e in range(E):
        grp.experts[e] = e
        grp.slabs[e] = slabs[e].data_ptr()
    outs = []
    for dev in (False, True, True):
        h = torch.zeros(rows, F, dtype=torch.int16, device="cuda")
        yp = torch.full((rows, H), float("nan"), dtype=torch.float32, device="cuda")
        if dev:
            ps.check(lib.ps_expert_ffn_prefill_dev(C.byref(grp), _p(off), _p(xp), rows, H, F, _p(h), _p(yp), s))
        else:
            ps.check(lib.ps_set_prefill_kernel(3))
            ps.check(lib.ps_expert_ffn_prefill(C.byref(grp), counts.ctypes.data, offsets.ctypes.data, _p(xp), rows,
                                               H, F, _p(h), _p(yp), s))
            ps.check(lib.ps_set_prefill_kernel(2))
        outs.append((h.cpu().numpy(), yp.cpu().numpy()))
    assert np.isfinite(outs[0][1]).all()
    for h, yp in outs[1:]:
        assert np.array_equal(h, outs[0][0])
        assert np.array_equal(yp, outs[0][1])


def test_prefill_map_table_overflow_restarts(tmp_path):
    """The token-N kernel's persistent tensor-map table (weights by slab, tokens by chunk
    size) empties itself after a device sync when full: in a process whose table holds only
    64 maps, 12 prefill calls with 12 different chunk sizes (and both entry points) still
    match the oracle. Subprocess: the capacity is read once per process."""
    import subprocess
    import sys
    code = r"""
import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, %r)
sys.path.insert(0, %r)
import oracle as orc, paper_2509_23638_b200 as ps
from test_gpu_prefill import _explicit_counts_case, _rel
lib = ps.load()
for i in range(12):
    counts = [5 + 17 * i, 33, 1 + i, 64]
    ys, y_ref = _explicit_counts_case(torch, 256, 256, counts, 100 + i, reps=1)
    assert _rel(ys[0], y_ref) < 2e-2, (i, _rel(ys[0], y_ref))
print("ok")
""" % (str(_tests_dir()), str(_tests_dir().parent))
    env = dict(__import__("os").environ, PS_MAPTABLE_CAP="64")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def _tests_dir():
    import pathlib
    return pathlib.Path(__file__).resolve().parent
