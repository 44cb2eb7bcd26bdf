"""Expert parallelism on the GPU.

* Engine over a real NCCL communicator (world 1: send/recv to self) must reproduce the
  non-EP engine bit for bit (same rows, same kernels, exact unit-weight unpermute).
* The EP data path for world G in {2, 4}, emulated on one GPU through the per-op C ABI:
  each virtual rank remaps + permutes + packs its counts, the test moves the segments
  (the all-to-all), each owner runs only its experts on the received rows, unpermutes,
  the outputs travel back and are combined at home — compared with the CPU oracle."""
import ctypes as C

import numpy as np
import pytest

import oracle as orc
import paper_2509_23638_b200 as ps
from paper_2509_23638_b200 import engine as eng

pytestmark = pytest.mark.gpu
BF16_RTOL = 2e-2


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


@pytest.mark.parametrize("compress", [False, True])
def test_engine_ep_world1_matches_engine(torch_cuda, compress):
    spec = ps.desk_scale("mixtral", 4, 8, 256)
    spec.expert_bytes = 6 * 256 * 512
    cfg = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    B = 16
    gate, hidden, follow, _ = ps.trace_inputs(cfg, spec, B, 4)
    outs = []
    for use_ep in (False, True):
        comm = eng.EpComm() if use_ep else None
        try:
            with eng.Engine(spec, cfg, budget_fraction=0.5, max_batch=B, weight_seed=3, gate=gate,
                            trace_hidden=hidden, trace_follow=follow, ep=comm, compress_host=compress) as e:
                outs.append(e.step_host(hidden, follow))
        finally:
            if comm:
                comm.close()
    np.testing.assert_array_equal(outs[0][1], outs[1][1])
    np.testing.assert_allclose(outs[0][0], outs[1][0], rtol=0, atol=0)


@pytest.mark.parametrize("G", [2, 4])
def test_ep_data_path_emulated_ranks(torch_cuda, G):
    torch = torch_cuda
    lib = ps.load()
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    H, F, E, k, B = 256, 512, 8, 2, 12  # B tokens per rank
    El = (E + G - 1) // G
    rng = np.random.default_rng(G)
    slabs = []
    for e in range(E):
        t = torch.empty(3 * H * F, dtype=torch.int16, device="cuda")
        ps.check(lib.ps_init_expert_slab(_p(t), H, F, 9, 0, e, s))
        slabs.append(t)
    ranks = []
    for r in range(G):  # home side: route (given), remap, permute+gather, pack counts
        ids = np.stack([rng.choice(E, k, replace=False) for _ in range(B)]).astype(np.int32)
        lg = rng.standard_normal((B, E))
        w = np.exp(lg - lg.max(1, keepdims=True))
        w /= w.sum(1, keepdims=True)
        x = orc.f32_to_bf16((rng.standard_normal((B, H)) / np.sqrt(H)).astype(np.float32))
        d = {"ids": ids, "w": w.astype(np.float32), "x": x, "dids": torch.as_tensor(ids, device="cuda"),
             "dx": torch.as_tensor(x.view(np.int16), device="cuda")}
        vids = torch.empty(B * k, dtype=torch.int32, device="cuda")
        ps.check(lib.ps_ep_remap_ids(_p(d["dids"]), B * k, E, G, _p(vids), s))
        off_v = torch.empty(G * El + 1, dtype=torch.int32, device="cuda")
        perm_v = torch.empty(B * k, dtype=torch.int32, device="cuda")
        inv_v = torch.empty(B * k, dtype=torch.int32, device="cuda")
        send_x = torch.empty(B * k, H, dtype=torch.int16, device="cuda")
        ps.check(lib.ps_permute(_p(vids), B, k, G * El, _p(off_v), _p(perm_v), _p(inv_v), _p(d["dx"]), H, _p(send_x),
                                s))
        cnt = torch.empty(G, 2 * El, dtype=torch.int32, device="cuda")
        ps.check(lib.ps_ep_pack_counts(_p(off_v), None, E, G, _p(cnt), s))
        d.update(off_v=off_v.cpu().numpy(), inv_v=inv_v, send_x=send_x, cnt=cnt.cpu().numpy())
        ranks.append(d)
    y_back = [torch.empty(B * k, H, dtype=torch.float32, device="cuda") for _ in range(G)]
    for o in range(G):  # owner side
        recv_cnt = np.stack([ranks[sr]["cnt"][o, :El] for sr in range(G)]).astype(np.int32)
        segs = [ranks[sr]["send_x"][ranks[sr]["off_v"][o * El]:ranks[sr]["off_v"][(o + 1) * El]] for sr in range(G)]
        recv_x = torch.cat(segs) if sum(len(t) for t in segs) else torch.empty(0, H, dtype=torch.int16, device="cuda")
        rows = recv_x.shape[0]
        off_loc = np.empty(El + 1, np.int32)
        perm = np.empty(max(1, rows), np.int32)
        seg = np.empty(G + 1, np.int32)
        ps.check(lib.ps_ep_recv_plan(recv_cnt.ctypes.data, G, El, off_loc.ctypes.data, perm.ctypes.data,
                                     seg.ctypes.data))
        if rows == 0:
            continue
        og = np.zeros(E + 1, np.int32)
        counts = np.zeros(E, np.int32)
        run = 0
        for e in range(E):
            og[e] = run
            if e % G == o:
                counts[e] = off_loc[e // G + 1] - off_loc[e // G]
                run += counts[e]
        og[E] = run
        inv = np.empty(rows, np.int32)
        inv[perm[:rows]] = np.arange(rows, dtype=np.int32)
        d_og = torch.as_tensor(og, device="cuda")
        d_perm = torch.as_tensor(perm[:rows].copy(), device="cuda")
        d_inv = torch.as_tensor(inv, device="cuda")
        grp = ps.capi.ExpertGroup()
        for e in range(E):
            if e % G == o:
                grp.experts[grp.n] = e
                grp.slabs[grp.n] = slabs[e].data_ptr()
                grp.n += 1
        h = torch.empty(rows, F, dtype=torch.int16, device="cuda")
        yp = torch.empty(1, rows, H, dtype=torch.float32, device="cuda")
        ps.check(lib.ps_expert_ffn(C.byref(grp), counts.ctypes.data, _p(d_og), _p(d_perm), 1, _p(recv_x), H, F, _p(h),
                                   _p(yp), 1, rows, s))
        ones = torch.ones(rows, dtype=torch.float32, device="cuda")
        zeros = torch.zeros(rows, dtype=torch.int32, device="cuda")
        y_recv = torch.empty(rows, H, dtype=torch.float32, device="cuda")
        ps.check(lib.ps_combine(_p(yp), 1, _p(d_inv), _p(zeros), _p(ones), rows, 1, 1, H, _p(y_recv), s))
        for sr in range(G):  # all-to-all back into each home's owner-major send order
            a, b = ranks[sr]["off_v"][o * El], ranks[sr]["off_v"][(o + 1) * El]
            y_back[sr][a:b] = y_recv[seg[sr]:seg[sr + 1]]
    slabs_h = [t.cpu().numpy().view(np.uint16) for t in slabs]
    for r, d in enumerate(ranks):  # home combine vs oracle
        y = torch.empty(B, H, dtype=torch.float32, device="cuda")
        dw = torch.as_tensor(d["w"], device="cuda")
        ps.check(lib.ps_combine(_p(y_back[r]), 1, _p(d["inv_v"]), _p(d["dids"]), _p(dw), B, k, E, H, _p(y), s))
        y_ref = orc.or_moe_layer(slabs_h, H, F, d["x"], d["ids"], d["w"], True)
        rel = np.linalg.norm(y.cpu().numpy() - y_ref) / np.linalg.norm(y_ref)
        assert rel < BF16_RTOL, (r, rel)
