"""Online LLaPor fine-tuning through the engine (§8f row 4): decode a step, fine_tune the
nets on that step's observations (ps_engine_last_routing + the step's hidden states),
decode again with the updated nets (their GPU copies refresh lazily) — outputs stay
correct, and the refreshed GPU net equals the fine-tuned model saved to LLPC (vs the f64
restatement of the reference's forward)."""
import ctypes as C

import numpy as np
import pytest

import oracle as orc
import paper_2509_23638_b200 as ps
from paper_2509_23638_b200 import engine as eng
from oracle.llpc import random_nets, write_llpc

pytestmark = pytest.mark.gpu
BF16_RTOL = 2e-2


def test_engine_online_fine_tune_round_trip(torch_cuda, tmp_path):
    torch = torch_cuda
    lib = ps.load()
    spec = ps.desk_scale("mixtral", 4, 8, 256)
    spec.expert_bytes = 6 * 256 * 512
    path = tmp_path / "nets.llpc"
    write_llpc(path, spec, random_nets(spec, 32, 64, 32, 48, seed=4))
    m = C.c_void_p()
    ps.check(lib.ps_llapor_load(str(path).encode(), C.byref(m), None))
    B = 16
    cfg = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    gate, hidden, follow, zipf = ps.trace_inputs(cfg, spec, 2 * B, 8)
    try:
        with eng.Engine(spec, cfg, budget_fraction=0.25, max_batch=B, weight_seed=9, gate=gate, trace_hidden=hidden,
                        trace_follow=follow, predictor=m) as e:
            h0 = hidden[:B]
            e.step_host(h0, follow[:B])
            before = e.last_predictions().copy()
            e.fine_tune_predictor(m, np.ascontiguousarray(h0.transpose(1, 0, 2)), steps=3, lr=3e-3)
            y, ids = e.step_host(hidden[B:], follow[B:])
            _, ref_w, _ = orc.or_route_trace(gate, hidden[B:], follow[B:], zipf, spec.top_k)
            y_ref = orc.or_engine_reference(spec, ps.ffn_dim(spec), 9, hidden[B:], ids, ref_w.transpose(1, 0, 2))
            assert np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref) < BF16_RTOL
        saved = tmp_path / "tuned.llpc"
        ps.check(lib.ps_llapor_save(m, str(saved).encode()))
        assert saved.read_bytes() != path.read_bytes()
        _, onets = orc.llapor_net_from_ckpt(saved)
        # GPU forward of the refreshed net 2 == the f64 forward of the saved fine-tuned net 2
        x = np.ascontiguousarray(hidden[:B, 1], np.float32)
        act = np.ascontiguousarray(ids[1], np.int32)
        gw = np.ascontiguousarray(ref_w[:, 1], np.float32)
        xd, ad, gd = (torch.as_tensor(a, device="cuda") for a in (x, act, gw))
        lg = torch.empty(B, spec.experts_per_layer, device="cuda")
        scratch = torch.empty(lib.ps_llapor_scratch_bytes(m, B), dtype=torch.uint8, device="cuda")
        ps.check(lib.ps_llapor_forward(m, 2, C.c_void_p(xd.data_ptr()), C.c_void_p(ad.data_ptr()), spec.top_k,
                                       C.c_void_p(gd.data_ptr()), B, spec.top_k, C.c_void_p(lg.data_ptr()), None,
                                       None, C.c_void_p(scratch.data_ptr()), None))
        torch.cuda.synchronize()
        g = lg.cpu().numpy()
        for t in range(B):
            _, r, _ = orc.or_llapor_forward(onets[2], x[t].astype(np.float64), act[t], gw[t].astype(np.float64),
                                            spec.top_k)
            assert (np.abs(g[t] - r) / np.maximum(1.0, np.abs(r))).max() < 1e-4
        assert before.shape == (spec.num_layers, spec.experts_per_layer)
    finally:
        lib.ps_llapor_free(m)
