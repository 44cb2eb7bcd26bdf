"""The real expert-parallel engine (ps_engine with a ps_ep_comm) at G = 2, 4, 8 ranks in
ONE process on one GPU, over the in-process transport (ps_ep_loopback_create: the
NCCL all-to-all contract built from CUDA events and device copies). Each rank owns
experts e % G with its own HBM budget/cache/loader, routes its own B tokens, dispatches
rows to the owners, runs its experts, returns outputs, combines at home — the exact
engine code that runs over NCCL across GPUs. Every rank's outputs are
compared with the CPU oracle on that rank's tokens (§8e oracle: the single-GPU result),
ids with the reference router."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle as orc
import paper_2509_23638_b200 as ps
from paper_2509_23638_b200 import engine as eng

pytestmark = pytest.mark.gpu
BF16_RTOL = 2e-2


def _ep_run(spec, G, B, budget, seed=5, compress=False, steps=2, host_threads=0, cost=None):
    L, E = spec.num_layers, spec.experts_per_layer
    cfg = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    gate, hidden, follow, zipf = ps.trace_inputs(cfg, spec, B * G, seed)
    freq = eng.hot_table(spec, gate, hidden, follow, zipf)
    comms = eng.EpComm.loopback(G)
    engines = []
    try:
        for r in range(G):
            f = freq.copy()
            for x in range(E):
                if x % G != r:
                    f[:, x] = -1
            n_owned = sum(1 for x in range(E) if x % G == r) * L
            budget_bytes = int(round(budget * n_owned)) * spec.expert_bytes
            resident = [(l, x) for (l, x) in ps.plan_residency(f, budget_bytes, spec.expert_bytes) if x % G == r]
            engines.append(eng.Engine(spec, cfg, max_batch=B, weight_seed=9, gate=gate, budget_bytes=budget_bytes,
                                      resident=resident, ep=comms[r], compress_host=compress,
                                      host_threads=host_threads, cost=cost))

        def rank_step(r):
            sl = slice(r * B, (r + 1) * B)
            out = None
            for _ in range(steps):
                out = engines[r].step_host(hidden[sl], follow[sl])
            return out

        with ThreadPoolExecutor(G) as pool:
            outs = list(pool.map(rank_step, range(G)))
        stats = [e.stats() for e in engines]
    finally:
        for e in engines:
            e.close()
        for c in comms:
            c.close()
    F = ps.ffn_dim(spec)
    for r in range(G):
        sl = slice(r * B, (r + 1) * B)
        y, ids = outs[r]
        _, ref_w, ref_ids = orc.or_route_trace(gate, hidden[sl], follow[sl], zipf, spec.top_k)
        assert np.array_equal(ids, ref_ids.transpose(1, 0, 2)), f"rank {r}: ids differ from the reference router"
        y_ref = orc.or_engine_reference(spec, F, 9, hidden[sl], ids, ref_w.transpose(1, 0, 2))
        for l in range(L):
            rel = np.linalg.norm(y[l] - y_ref[l]) / np.linalg.norm(y_ref[l])
            assert rel < BF16_RTOL, (r, l, rel)
    return stats


@pytest.mark.parametrize("G,budget,compress", [(2, 0.5, False), (4, 0.5, True), (8, 0.25, False), (8, 1.0, False)])
def test_ep_engine_loopback_mixtral_like(torch_cuda, G, budget, compress):
    spec = ps.desk_scale("mixtral", 3, 8, 256)
    spec.expert_bytes = 6 * 256 * 512
    stats = _ep_run(spec, G, 8, budget, compress=compress)
    if budget < 1.0:  # every rank loads its non-resident experts over its own loader
        assert sum(s["ondemand_loads"] + s["prefetches_committed"] for s in stats) > 0
    else:
        assert all(s["h2d_bytes"] == 0 for s in stats)


def test_ep_engine_loopback_qwen3_like(torch_cuda):
    spec = ps.desk_scale("qwen3", 3, 128, 256)
    spec.expert_bytes = 6 * 256 * 128
    _ep_run(spec, 4, 16, 0.5)


def test_ep_engine_loopback_prefill_chunk(torch_cuda):
    """B > 64 per rank: prefill mode through EP (gathered received rows, tcgen05 path)."""
    spec = ps.desk_scale("mixtral", 3, 8, 256)
    spec.expert_bytes = 6 * 256 * 512
    stats = _ep_run(spec, 2, 160, 1.0, steps=1)
    assert sum(s["tc_launches"] for s in stats) > 0


def test_ep_engine_loopback_mixtral_expert_shape(torch_cuda):
    """Full Mixtral expert shape (H=4096, F=14336), G=2, z-slab loads, 50 % budget."""
    full = ps.spec_preset("mixtral")
    spec = ps.desk_scale("mixtral", 3, 8, 4096)
    spec.expert_bytes = full.expert_bytes
    _ep_run(spec, 2, 16, 0.5, compress=True, steps=1)


@pytest.mark.parametrize("G", [2, 4])
def test_ep_engine_loopback_with_host_lane(torch_cuda, G):
    """The same executor at every G: each rank's PreSched cpu_set runs on its own host
    expert lane from the rows routed to it by all ranks (copied to the host after the
    dispatch), with PCIe priced far above the lane."""
    spec = ps.desk_scale("mixtral", 3, 8, 256)
    spec.expert_bytes = 6 * 256 * 512
    stats = _ep_run(spec, G, 8, 0.25, host_threads=2, cost=(1000, 5, 10, 1.0, 1, 0))
    assert sum(s["cpu_experts"] for s in stats) > 0
