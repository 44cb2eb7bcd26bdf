"""Small engine run for compute-sanitizer (memcheck / racecheck / synccheck): every
kernel and copy path of the decode engine once — resident group, on-demand loads,
prefetch, host expert lane, shared experts, prefill chunk (tcgen05) — at desk shapes.

  compute-sanitizer --tool memcheck python scripts/sanitize_engine.py
"""
import pathlib
import sys

import torch  # noqa: F401  (CUDA context + pinned allocator parity with the tests)

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_2509_23638_b200 as ps  # noqa: E402
from paper_2509_23638_b200 import engine as eng  # noqa: E402


def run(preset, L, E, H, F, B, budget, **kw):
    spec = ps.desk_scale(preset, L, E, H)
    spec.expert_bytes = 6 * H * F
    gen = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    gate, hidden, follow, _ = ps.trace_inputs(gen, spec, B, 3)
    with eng.Engine(spec, gen, budget_fraction=budget, max_batch=B, weight_seed=9, gate=gate, trace_hidden=hidden,
                    trace_follow=follow, **kw) as e:
        for _ in range(2):
            e.step_host(hidden, follow)
        print(preset, B, budget, kw, e.stats()["ondemand_loads"], e.stats()["cpu_experts"])


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="all", choices=["all", "prefill_single", "prefill_pair", "prefill_tn"],
                    help="prefill_*: only that tcgen05 kernel (to attribute sanitizer reports)")
    args = ap.parse_args()
    if args.only != "all":
        lib = ps.load()
        ps.check(lib.ps_set_prefill_kernel({"prefill_single": 0, "prefill_pair": 1, "prefill_tn": 3}[args.only]))
        run("mixtral", 3, 8, 256, 512, 512, 1.0)
        run("mixtral", 3, 8, 256, 512, 1200, 1.0)  # m_e ~ 300: equal-width multi-tile experts
        print("sanitize run done")
        return
    cost = (1000, 5, 10, 1.0, 1, 0)
    run("mixtral", 3, 8, 256, 512, 8, 0.25)
    run("mixtral", 3, 8, 256, 512, 8, 0.25, host_threads=2, cost=cost)
    run("deepseek", 3, 64, 256, 256, 8, 0.2, n_shared=2, host_threads=2, cost=cost)
    run("mixtral", 3, 8, 256, 512, 256, 0.5)
    run("mixtral", 3, 8, 256, 512, 8, 0.25, compress_host=True)
    run("mixtral", 3, 8, 256, 512, 256, 0.5, compress_host=True)
    run("qwen3", 3, 128, 256, 256, 32, 0.5, host_threads=2, cost=cost)  # split router, ranged lane rows
    lib = ps.load()
    for kern, name in ((0, "single-CTA"), (1, "CTA-pair"), (3, "token-N")):  # every tcgen05 prefill kernel
        ps.check(lib.ps_set_prefill_kernel(kern))
        print("prefill kernel", name)
        run("mixtral", 3, 8, 256, 512, 512, 1.0)
        run("deepseek", 3, 16, 256, 256, 512, 1.0, n_shared=2)
    ps.check(lib.ps_set_prefill_kernel(2))
    ep_loopback(2)
    print("sanitize run done")


def ep_loopback(G):
    """The EP engine over the in-process transport (G ranks, one thread each)."""
    from concurrent.futures import ThreadPoolExecutor
    spec = ps.desk_scale("mixtral", 3, 8, 256)
    spec.expert_bytes = 6 * 256 * 512
    gen = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    B = 8
    gate, hidden, follow, _ = ps.trace_inputs(gen, spec, B * G, 3)
    comms = eng.EpComm.loopback(G)
    es = [eng.Engine(spec, gen, max_batch=B, weight_seed=9, gate=gate, budget_bytes=spec.expert_bytes * 2,
                     resident=[(0, r)], ep=comms[r]) for r in range(G)]
    with ThreadPoolExecutor(G) as pool:
        list(pool.map(lambda r: es[r].step_host(hidden[r * B:(r + 1) * B], follow[r * B:(r + 1) * B]), range(G)))
    for e in es:
        e.close()
    for c in comms:
        c.close()
    print("ep loopback", G)


if __name__ == "__main__":
    main()
