"""Expert-parallel host logic across 2 processes (gloo, world_size 2, CPU): the
owner-major send order and the receive plan (ps_ep_recv_plan) must route every routed
(token, slot) row to its owner exactly once, grouped by local expert, sources in rank
order, tokens ascending — the contract the GPU dispatch/combine kernels rely on."""
import ctypes as C
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2509_23638_b200 as ps

E, K, B = 8, 2, 7


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        lib = ps.load()
        G = world
        El = (E + G - 1) // G
        rng = np.random.default_rng(100 + rank)
        ids = np.stack([rng.choice(E, K, replace=False) for _ in range(B)]).astype(np.int32)
        # sender: owner-major virtual id, stable over (token, slot) -> destination segments
        v = (ids % G) * El + ids // G
        order = np.argsort(v.ravel(), kind="stable")
        rows = [(rank, int(i // K), int(i % K), int(ids.ravel()[i])) for i in order]
        send_rows = [sum(1 for r in rows if r[3] % G == d) for d in range(G)]
        cnt = np.zeros((G, El), np.int32)
        for r in rows:
            cnt[r[3] % G, r[3] // G] += 1
        recv_cnt = torch.empty(G * El, dtype=torch.int32)
        dist.all_to_all_single(recv_cnt, torch.from_numpy(cnt.ravel().copy()))
        recv_cnt = recv_cnt.numpy().reshape(G, El)
        recv_rows = [int(recv_cnt[s].sum()) for s in range(G)]
        meta = torch.tensor(rows, dtype=torch.int32).reshape(-1, 4)
        got = torch.empty(sum(recv_rows), 4, dtype=torch.int32)
        dist.all_to_all_single(got, meta, output_split_sizes=recv_rows, input_split_sizes=send_rows)
        got = got.numpy()
        off = np.empty(El + 1, np.int32)
        perm = np.empty(max(1, len(got)), np.int32)
        seg = np.empty(G + 1, np.int32)
        ps.check(lib.ps_ep_recv_plan(recv_cnt.ctypes.data, G, El, off.ctypes.data, perm.ctypes.data, seg.ctypes.data))
        assert seg.tolist() == [0] + list(np.cumsum(recv_rows))
        assert sorted(perm[:len(got)].tolist()) == list(range(len(got)))
        for j in range(El):
            block = got[perm[off[j]:off[j + 1]]]
            assert (block[:, 3] == j * G + rank).all()          # owner
            assert (np.diff(block[:, 0]) >= 0).all()            # sources in rank order
            for s in range(G):
                toks = block[block[:, 0] == s][:, 1]
                assert (np.diff(toks) >= 0).all()               # tokens ascending
        assert lib.ps_ep_local_experts(E, G, rank) == El
        # every (token, slot) of every rank lands on exactly one owner
        total = torch.tensor([len(got)])
        dist.all_reduce(total)
        assert int(total) == world * B * K
        q.put((rank, "ok"))
    except Exception as ex:  # pragma: no cover
        q.put((rank, repr(ex)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_ep_dispatch_plan_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
