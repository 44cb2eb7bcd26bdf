"""Per-layer K5 ABI (ps_engine_step_begin / ps_engine_layer_forward / ps_engine_step_end,
the reference's per-layer seam plan_fn(inputs, l), simulator.cpp:136) and caller-supplied
expert weights (ps_engine_config.expert_weights): a host model that interleaves its own
attention kernels on its own stream gets bit-identical outputs to the whole-step call."""
import ctypes as C

import numpy as np
import pytest

import oracle as orc
import paper_2509_23638_b200 as ps
from paper_2509_23638_b200 import engine as eng

pytestmark = pytest.mark.gpu
BF16_RTOL = 2e-2


def _spec(L=4, E=8, H=256, F=512, preset="mixtral"):
    spec = ps.desk_scale(preset, L, E, H)
    spec.expert_bytes = 6 * H * F
    return spec


def _inputs(spec, B, seed=3):
    cfg = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    gate, hidden, follow, zipf = ps.trace_inputs(cfg, spec, B, seed)
    return cfg, gate, hidden, follow, zipf


def _host_slabs(spec, seed, n_shared=0):
    lib = ps.load()
    H, F = spec.hidden_dim, ps.ffn_dim(spec)
    out = []
    for l in range(spec.num_layers):
        for e in range(spec.experts_per_layer + n_shared):
            a = np.empty(3 * H * F, np.uint16)
            ps.check(lib.ps_init_expert_slab_host(a.ctypes.data, H, F, seed, l, e))
            out.append(a)
    return out


def _per_layer(torch, e, hid_lbh, fol_lb, attn_stream):
    """Host-model loop: 'attention' on the caller's stream produces x_l (a copy stands in
    for it), then the MoE layer on that stream."""
    L, B, H = hid_lbh.shape
    x = torch.empty(B, H, dtype=torch.float32, device="cuda")
    y = torch.empty(L, B, H, dtype=torch.float32, device="cuda")
    ids = torch.empty(L, B, e.spec.top_k, dtype=torch.int32, device="cuda")
    e.step_begin(B)
    with torch.cuda.stream(attn_stream):
        for l in range(L):
            x.copy_(hid_lbh[l])  # attention(l) -> x_l on the caller's stream
            e.layer_forward(l, x, fol_lb[l], y[l], ids[l], stream=attn_stream)
    e.step_end()
    torch.cuda.synchronize()
    return y.cpu().numpy(), ids.cpu().numpy()


@pytest.mark.parametrize("compress,budget", [(False, 0.5), (True, 0.25), (False, 1.0)])
def test_layer_api_bit_identical_to_decode_step(torch_cuda, compress, budget):
    torch = torch_cuda
    spec = _spec()
    B = 8
    cfg, gate, hidden, follow, _ = _inputs(spec, B)
    hid = torch.as_tensor(np.ascontiguousarray(hidden.transpose(1, 0, 2), np.float32), device="cuda")
    fol = torch.as_tensor(np.ascontiguousarray(follow.T), device="cuda")
    kw = dict(budget_fraction=budget, max_batch=B, weight_seed=9, gate=gate, trace_hidden=hidden,
              trace_follow=follow, policy="ondemand", compress_host=compress)
    with eng.Engine(spec, cfg, **kw) as e1:
        y1 = torch.empty(spec.num_layers, B, spec.hidden_dim, device="cuda")
        ids1 = torch.empty(spec.num_layers, B, spec.top_k, dtype=torch.int32, device="cuda")
        e1.step_device(hid, fol, y1, ids1)
        torch.cuda.synchronize()
        st1 = e1.stats()
    with eng.Engine(spec, cfg, **kw) as e2:
        s = torch.cuda.Stream()
        y2, ids2 = _per_layer(torch, e2, hid, fol, s)
        st2 = e2.stats()
        assert e2.verify_last_step() == []
    np.testing.assert_array_equal(ids1.cpu().numpy(), ids2)
    np.testing.assert_array_equal(y1.cpu().numpy(), y2)
    assert st1["ondemand_loads"] == st2["ondemand_loads"] and st2["steps"] == 1


def test_layer_api_presched_host_lane_llapor_vs_oracle(torch_cuda):
    """Per-layer calls with the full executor (PreSched, LLaPor, host expert lane,
    z-slabs) over two steps: outputs vs the oracle, timeline invariants."""
    torch = torch_cuda
    lib = ps.load()
    spec = _spec(L=4)
    B = 8
    cfg, gate, hidden, follow, zipf = _inputs(spec, 2 * B, seed=7)
    m = C.c_void_p()
    ps.check(lib.ps_llapor_random(C.byref(spec), 32, 64, 32, 48, 1, C.byref(m)))
    try:
        with eng.Engine(spec, cfg, budget_fraction=0.25, max_batch=B, weight_seed=9, gate=gate, trace_hidden=hidden,
                        trace_follow=follow, predictor=m, host_threads=2, cost=(1000, 5, 10, 1.0, 1, 0),
                        compress_host=True) as e:
            for s in range(2):
                h, f = hidden[s * B:(s + 1) * B], follow[s * B:(s + 1) * B]
                hid = torch.as_tensor(np.ascontiguousarray(h.transpose(1, 0, 2), np.float32), device="cuda")
                fol = torch.as_tensor(np.ascontiguousarray(f.T), device="cuda")
                y, ids = _per_layer(torch, e, hid, fol, torch.cuda.Stream())
                assert e.verify_last_step() == []
                _, ref_w, ref_ids = orc.or_route_trace(gate, h, f, zipf, spec.top_k)
                assert np.array_equal(ids, ref_ids.transpose(1, 0, 2))
                y_ref = orc.or_engine_reference(spec, ps.ffn_dim(spec), 9, h, ids, ref_w.transpose(1, 0, 2))
                assert np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref) < BF16_RTOL
            assert e.stats()["cpu_experts"] > 0
    finally:
        lib.ps_llapor_free(m)


@pytest.mark.parametrize("n_shared", [0, 2])
def test_caller_supplied_expert_weights(torch_cuda, n_shared):
    """expert_weights = the caller's host slabs (here the same synthetic values, made on
    the host): outputs bit-identical to the engine's own hash-initialised weights, for
    resident, loaded (raw and z-slab) and shared experts; a perturbed slab changes y."""
    spec = _spec(E=8, preset="deepseek" if n_shared else "mixtral")
    B = 8
    cfg, gate, hidden, follow, _ = _inputs(spec, B)
    slabs = _host_slabs(spec, 9, n_shared)
    kw = dict(budget_fraction=0.5, max_batch=B, gate=gate, trace_hidden=hidden, trace_follow=follow,
              policy="ondemand", n_shared=n_shared, compress_host=True)
    with eng.Engine(spec, cfg, weight_seed=9, **kw) as e1:
        y1, ids1 = e1.step_host(hidden, follow)
    with eng.Engine(spec, cfg, weight_seed=12345, expert_weights=slabs, **kw) as e2:
        y2, ids2 = e2.step_host(hidden, follow)
    np.testing.assert_array_equal(ids1, ids2)
    np.testing.assert_array_equal(y1, y2)
    E = spec.experts_per_layer + n_shared
    l0, e0 = 0, int(ids1[0, 0, 0])
    slabs[l0 * E + e0] = slabs[l0 * E + e0].copy()
    slabs[l0 * E + e0][:1000] = 0
    with eng.Engine(spec, cfg, weight_seed=9, expert_weights=slabs, **kw) as e3:
        y3, _ = e3.step_host(hidden, follow)
    assert not np.array_equal(y3[0], y1[0]) and np.array_equal(y3[1:], y1[1:])


def test_layer_api_errors(torch_cuda):
    torch = torch_cuda
    spec = _spec(L=3)
    B = 4
    cfg, gate, hidden, follow, _ = _inputs(spec, B)
    x = torch.as_tensor(hidden[:, 0].astype(np.float32), device="cuda")
    y = torch.empty_like(x)
    with eng.Engine(spec, cfg, budget_fraction=0.5, max_batch=B, weight_seed=1, gate=gate) as e:
        with pytest.raises(ps.capi.PsError):
            e.layer_forward(0, x, None, y)  # no step in progress
        e.step_begin(B)
        with pytest.raises(ps.capi.PsError):
            e.layer_forward(1, x, None, y)  # out of order
        e.layer_forward(0, x, None, y)
        with pytest.raises(ps.capi.PsError):
            e.step_end()  # layers 1, 2 missing
        # a new step recovers (step_begin settles the abandoned one)
        e.step_begin(B)
        for l in range(3):
            e.layer_forward(l, x, None, y)
        e.step_end()


def test_cpp_host_model_layer_loop(torch_cuda, tmp_path):
    """tests/cpp/layer_loop.cpp: a C++ host model (no Python, no torch) drives the engine
    per layer with its own stream and expert weights; bit-identical to the whole step."""
    import subprocess
    from conftest import ROOT
    exe = tmp_path / "layer_loop"
    lib_dir = ROOT / "paper_2509_23638_b200"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"), "-I", "/usr/local/cuda/include",
                    str(ROOT / "tests/cpp/layer_loop.cpp"), "-L", str(lib_dir), "-lprescope_b200",
                    "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib_dir}",
                    "-Wl,-rpath,/usr/local/cuda/lib64", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert "layer loop ok" in out.stdout
