"""Edge cases of the GPU ops through the C ABI (the reference's tests cover empty and
ragged inputs and maximum sizes): empty batches, the maximum expert count
and top-k, an expert that receives every token, ragged prefill chunks."""
import ctypes as C

import numpy as np
import pytest

import oracle as orc
import paper_2509_23638_b200 as ps
from paper_2509_23638_b200 import engine as eng

pytestmark = pytest.mark.gpu


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def test_empty_batch_is_a_no_op(torch_cuda):
    torch = torch_cuda
    lib = ps.load()
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    E, k, H = 8, 2, 64
    x = torch.zeros(1, H, device="cuda")
    g = torch.randn(E, H, device="cuda")
    w = torch.full((1, E), 7.0, device="cuda")
    ids = torch.full((1, k), -5, dtype=torch.int32, device="cuda")
    ps.check(lib.ps_route_topk(_p(x), _p(g), None, None, None, 0, 0, H, E, k, None, _p(w), _p(ids), None, None, s))
    off = torch.full((E + 1,), -1, dtype=torch.int32, device="cuda")
    src = torch.empty(1, dtype=torch.int32, device="cuda")
    inv = torch.empty(1, dtype=torch.int32, device="cuda")
    ps.check(lib.ps_permute(_p(ids), 0, k, E, _p(off), _p(src), _p(inv), None, H, None, s))
    y = torch.full((1, H), 3.0, device="cuda")
    ps.check(lib.ps_combine(_p(y), 1, _p(inv), _p(ids), _p(w), 0, k, E, H, _p(y), s))
    torch.cuda.synchronize()
    assert (w == 7.0).all() and (ids == -5).all() and (y == 3.0).all()  # untouched
    assert (off.cpu() == 0).all()  # empty histogram


@pytest.mark.parametrize("E,k,B", [(256, 16, 33), (256, 1, 5), (2, 2, 7)])
def test_route_and_permute_at_the_size_limits(torch_cuda, E, k, B):
    """kMaxE = 256 experts, kMaxK = 16, and k = E: top-k bit-exact vs topk_indices on the
    kernel's weights, permutation bit-exact vs the oracle."""
    torch = torch_cuda
    rng = np.random.default_rng(E + k)
    H = 128
    x = torch.as_tensor(rng.standard_normal((B, H)).astype(np.float32), device="cuda")
    g = torch.as_tensor((rng.standard_normal((E, H)) / np.sqrt(H)).astype(np.float32), device="cuda")
    bias = torch.zeros(E, device="cuda")
    _, w, ids, counts, _ = eng.route(x, g, bias, None, None, k)
    w, ids, counts = w.cpu().numpy(), ids.cpu().numpy(), counts.cpu().numpy()
    for t in range(B):
        assert list(ids[t]) == orc.or_topk(w[t].astype(np.float64), k)
    assert np.array_equal(counts, np.bincount(ids.ravel(), minlength=E))
    lib = ps.load()
    di = torch.as_tensor(ids, device="cuda")
    off = torch.empty(E + 1, dtype=torch.int32, device="cuda")
    src = torch.empty(B * k, dtype=torch.int32, device="cuda")
    inv = torch.empty(B * k, dtype=torch.int32, device="cuda")
    ps.check(lib.ps_permute(_p(di), B, k, E, _p(off), _p(src), _p(inv), None, H, None,
                            C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    o_off, o_src, o_inv = orc.or_permute(ids, E)
    assert np.array_equal(off.cpu().numpy(), o_off) and np.array_equal(src.cpu().numpy(), o_src)
    assert np.array_equal(inv.cpu().numpy(), o_inv)


def test_engine_all_tokens_on_one_expert_and_ragged_prefill(torch_cuda):
    """A routed trace where every token picks expert 3 (one expert with m = B, the others
    ragged) through the decode GEMV and, for B = 300, the tcgen05 prefill path."""
    spec = ps.desk_scale("mixtral", 3, 8, 256)
    spec.expert_bytes = 6 * 256 * 512
    cfg = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    for B in (16, 300):
        gate, hidden, follow, _ = ps.trace_inputs(cfg, spec, B, 9)
        L, E, k = spec.num_layers, spec.experts_per_layer, spec.top_k
        rng = np.random.default_rng(B)
        act = np.zeros((B, L, k), np.int32)
        act[:, :, 0] = 3
        act[:, :, 1] = rng.choice([e for e in range(E) if e != 3], (B, L))
        gw = rng.random((B, L, E))
        gw /= gw.sum(-1, keepdims=True)
        with eng.Engine(spec, cfg, budget_fraction=0.5, max_batch=B, weight_seed=2, gate=gate) as e:
            y = e.step_routed(hidden, act, gw.astype(np.float32))
            st = e.stats()
        y_ref = orc.or_engine_reference(spec, ps.ffn_dim(spec), 2, hidden, act.transpose(1, 0, 2),
                                        gw.transpose(1, 0, 2))
        assert np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref) < 2e-2
        if B > 64:
            assert st["tc_launches"] > 0
