#!/usr/bin/env python3
"""Headline benchmark: Mixtral-8x7B-shape MoE decode under a fixed HBM expert budget.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Step = one decode step of the MoE hot path over all 32 layers for a batch of B tokens:
K1 route -> K4 LLaPor (prediction of l+1) -> K2 permute -> PreSched plan -> resident
experts' FFN + PCIe loads of the missing experts (pinned host DRAM -> HBM on the copy
engine, dual on-demand buffer, PreSched prefetches) -> K3 FFN per landed expert -> K2
combine. Synthetic inputs: routing trace of the reference generator (same RNG), random
bf16 weights of the named shapes (hash-initialised; no checkpoints offline).

`value` = B / device time per step (CUDA events on the engine's compute stream), inputs
already in HBM. `e2e` = the same through the host-buffer C-ABI call
(ps_engine_decode_step_host: H2D inputs, step, D2H outputs), host wall-clock around the
blocking call. `roofline` = the decode FFN kernel (K3), the dominant kernel, vs the
measured HBM copy bandwidth. `cpu_baseline` = the same step on the host cores: the
oracle port of the SwiGLU FFN/combine + the reference's own scheduling code.
N>1: expert parallelism (torchrun, one rank per GPU): rank r owns experts e % N == r with the
same budget fraction of its shard, decodes its own B tokens (weak scaling) and exchanges
routed rows with NCCL all-to-all over NVLink.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import pathlib
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "decode tokens/sec & MoE-layer us at Mixtral-8x7B shape, fixed HBM expert budget"
PCIE_H2D_PEAK_GBS = 55.5  # measured pinned H2D on this pool (scripts/probe.sh, gpurun_out/probe.log)


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


def bf16_peak():
    """Dense bf16 TF/s denominator for the prefill leg: MEASURED_PEAKS.json's sustained
    figure when it has one (the leg is a long tensor-bound step that runs into the power
    cap: SM clocks ~1200 MHz under sw_power_cap were sampled during it), else its plain
    bf16 figure, else the profiling guide's fallback."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        sus = [v for k, v in d.items() if "bf16" in k and "sustain" in k and isinstance(v, (int, float))]
        if sus:
            return float(sus[0]), "measured_sustained"
        if isinstance(d.get("bf16_tflops"), (int, float)):
            return float(d["bf16_tflops"]), "measured"
    return 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.rows)}


def make_workload(args):
    import paper_2509_23638_b200 as ps
    spec = ps.spec_preset(args.model)
    gen = ps.TraceGenConfig(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    return ps, spec, gen


def host_info():
    from oracle.cpu_arm import cpu_model
    return {"cpu_model": cpu_model(), "nproc": os.cpu_count()}


def cpu_sample(args, ffn_layers=(0, 1)):
    """Bounded CPU sample for our arm's `cpu_baseline`: one decode step of the reference
    CPU path (oracle/cpu_arm.py: the reference router, LLaPor at full shape and
    simulate_policy(presched) through oracle/_ref for the WHOLE step, plus the expert
    port on `ffn_layers` only, scaled to all layers), after one warm-up step; and the
    1-core table of the reference's hot-path functions."""
    from oracle.cpu_arm import RefArm
    arm = RefArm(args.model, args.batch, args.budget, steps=2, weight_seed=args.weight_seed,
                 ffn_layers=list(ffn_layers))
    try:
        arm.step(0)
        sec, ph, _ = arm.step(1)
        scale = arm.L / len(arm.ffn_layers)
        step_s = sec - ph["experts"] + ph["experts"] * scale
        legs = arm.legs_1core()
        t0 = time.perf_counter()
        from oracle import or_route_batch
        or_route_batch(arm.gate, arm.hidden[:arm.B], arm.follow[:arm.B], arm.zipf, arm.k, 1)
        route_us = (time.perf_counter() - t0) * 1e6 / (arm.B * arm.L)
    finally:
        arm.close()
    legs_us = {"router (workload.cpp:176-202, f64 restatement), per token-layer": round(route_us, 3)}
    legs_us.update({k: round(v[0], 3) for k, v in legs.items()})
    desc = (f"one B={args.batch} decode step of the reference CPU path: router + LLaPor (P=256/512) + "
            f"simulate_policy(presched) for all {arm.L} layers through oracle/_ref, experts+combine "
            f"(oracle/cpu_port.c, {arm.threads} threads) on {len(ffn_layers)} of {arm.L} layers scaled "
            f"x{scale:g}; phases {', '.join(f'{k} {v * 1e3:.1f} ms' for k, v in ph.items() if k != 'makespan_ticks')}")
    return step_s, desc, legs_us, arm.threads


def run_reference_arm(args):
    """--impl reference: the reference CPU path of the bench workload on this box's host
    cores, WHOLE decode steps (W warm-up + K timed), loading only oracle/ (the
    unmodified reference in oracle/_ref + the oracle/cpu_port.c expert port)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle as orc
    if not orc.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libprescope_ref.so not built"}))
        return
    from oracle.cpu_arm import RefArm
    # our arm's workload at N GPUs is a global batch of N x batch tokens per step (weak
    # scaling): the reference arm steps the same global batch on the host cores
    gb = args.batch * max(1, args.gpus)
    t_init = time.perf_counter()
    arm = RefArm(args.model, gb, args.budget, steps=args.warmup + args.steps, weight_seed=args.weight_seed)
    t_init = time.perf_counter() - t_init
    phases = {}
    times = []
    wall0 = time.perf_counter()
    for s in range(args.warmup + args.steps):
        sec, ph, _ = arm.step(s)
        if s >= args.warmup:
            times.append(sec)
            for k, v in ph.items():
                phases[k] = phases.get(k, 0.0) + v / args.steps
    wall = time.perf_counter() - wall0
    legs = arm.legs_1core()
    threads = arm.threads
    L = arm.L
    arm.close()
    step_s = sum(times) / len(times)
    value = gb / step_s
    desc = (f"whole B={gb} decode steps ({args.steps} timed after {args.warmup} warm-up, no extrapolation): "
            f"reference router + LLaPor P=256/512 + simulate_policy(presched) via oracle/_ref, experts+combine via "
            f"oracle/cpu_port.c on all {L} layers, {threads} host threads")
    cfg = {"workload": f"{args.model}-shape MoE decode, {L} layers, batch {gb}, budget {args.budget:.0%}: "
                       "the reference's CPU path (oracle/_ref) + CPU expert port",
           "decode_batch": args.batch, "global_batch": gb, "budget_fraction": args.budget}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16 weights, f32/f64 accumulate",
            "data": "synthetic (reference generate_trace, hash-init bf16 weights, random-init LLaPor)",
            "config": cfg, "moe_layer_us": step_s / L * 1e6,
            "phases_ms_per_step": {k: round(v * 1e3, 3) for k, v in phases.items() if k != "makespan_ticks"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "reference",
                             "sample": desc, "host": host_info(),
                             "legs_1core_us": {k: round(v[0], 3) for k, v in legs.items()}},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "consistency": {"timed_s": sum(times), "wall_s_steps": wall, "init_s": t_init,
                            "fits_in_driver_run": True}}
    print(json.dumps(line))


def workload_config(args, spec, executor="gpu_only"):
    import paper_2509_23638_b200 as ps
    L, E = spec.num_layers, spec.experts_per_layer
    n_res = int(round(args.budget * L * E))
    return {"workload": f"{args.model}-shape MoE decode: {L} layers, {E} experts top-{spec.top_k}, H={spec.hidden_dim}, "
                        f"F={ps.ffn_dim(spec)}, batch {args.batch}, HBM expert budget {args.budget:.0%} "
                        f"({n_res}/{L * E} experts resident, hot-table residency from a warm-up trace), "
                        f"other experts in pinned host DRAM, policy {args.policy}"

                        + (", PreSched cpu_set on the host expert lane (AMX-BF16, reading the z-slabs)" if executor == "host_lane" else
                           ", GPU-only executor")
                        + (", loads as lossless z-slabs decoded on the GPU" if getattr(args, "compress", 0)
                           else "")
                        + f", predictor {getattr(args, 'predictor', 'llapor')}"
                        + ((f" (full shape, fine-tuned online on {args.llapor_finetune} warm-up steps of a separate "
                            "trace: ps_llapor_fine_tune = predictor.cpp:654-663)" if getattr(args, "llapor_finetune", 0)
                            else " (random-init at full shape)")
                           if getattr(args, "predictor", "llapor") == "llapor" else ""),
            "expert_shape": f"{args.model}-8x7b" if args.model == "mixtral" else args.model,
            "decode_batch": args.batch, "global_batch": args.batch * args.gpus,
            "parallelism": (f"ep{args.gpus}" if args.gpus > 1 else "single"),
            "executor": executor,
            "budget_fraction": args.budget, "policy": args.policy,
            "extra_leg": (f"host_lane_lookahead: PreSched + lookahead {args.lookahead}"
                          + (" + steal_late" if getattr(args, "steal_late", 0) else "")
                          if getattr(args, "lookahead", 0) or getattr(args, "steal_late", 0) else None),
            "l2": "inputs larger than L2 (each expert slab 336 MiB > 126 MB L2)"}


def run_ours(args):
    import torch

    import paper_2509_23638_b200 as ps
    from paper_2509_23638_b200 import engine as eng

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    _, spec, gen = make_workload(args)
    L, E, H, k = spec.num_layers, spec.experts_per_layer, spec.hidden_dim, spec.top_k
    B = args.batch
    S = args.warmup + args.steps
    # routing inputs: one trace (one set of gate matrices for all ranks), B*S tokens per
    # rank sliced into S decode steps; rank r decodes its own tokens (weak scaling)
    gate, hidden_all, follow_all, zipf = ps.trace_inputs(gen, spec, B * S * world, 1000)
    hidden = hidden_all[rank * B * S:(rank + 1) * B * S]
    follow = follow_all[rank * B * S:(rank + 1) * B * S]
    # hot table from a separate warm-up trace with the same gate matrices (perf mode)
    _, warm_h, warm_f, _ = ps.trace_inputs(gen, spec, 64, 1000, want_gate=False)
    freq = eng.hot_table(spec, gate, warm_h, warm_f, zipf)
    ep = None
    if world > 1:
        # Expert parallelism: rank r owns experts e % world == r and the
        # same budget fraction of its shard; tokens are exchanged with NCCL all-to-all.
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(eng.EpComm.unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        ep = eng.EpComm(rank, world, local, bytes(uid.cpu().numpy().tobytes()))
        freq = freq.copy()
        for x in range(E):
            if x % world != rank:
                freq[:, x] = -1  # never resident here
        n_owned = sum(1 for x in range(E) if x % world == rank) * L
        budget_bytes = int(round(args.budget * n_owned)) * spec.expert_bytes
    else:
        budget_bytes = int(round(args.budget * L * E)) * spec.expert_bytes
    resident = [(l, x) for (l, x) in ps.plan_residency(freq, budget_bytes, spec.expert_bytes)
                if x % world == rank]

    lib = ps.load()
    predictor = C.c_void_p()
    ps.check(lib.ps_llapor_random(C.byref(spec), 256, 512, 32, 48, 3, C.byref(predictor)))
    host_threads = args.host_threads if args.host_threads >= 0 else default_host_threads(world)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info(local)[0]
    t_create = time.perf_counter()
    e = eng.Engine(spec, gen, max_batch=B, weight_seed=args.weight_seed, gate=gate, budget_bytes=budget_bytes,
                   resident=resident, policy=args.policy, predictor=predictor, device=local, ep=ep,
                   host_threads=host_threads, compress_host=bool(args.compress),
                   predictor_kind=args.predictor, lookahead=args.lookahead, steal_late=bool(args.steal_late))
    t_create = time.perf_counter() - t_create
    torch.cuda.synchronize()
    hbm_engine = free0 - torch.cuda.mem_get_info(local)[0]
    t_ft = 0.0
    if args.llapor_finetune and args.predictor == "llapor":
        # online LLaPor fine_tune on a separate warm-up trace (not the measured steps), before
        # any timed region: the reference trains its predictor, random init is the weak case
        sys.path.insert(0, str(ROOT / "scripts"))
        import configs_bench
        t_ft = time.perf_counter()
        configs_bench.finetune(torch, e, predictor, spec, gen, B, args.llapor_finetune, seed=4242 + rank)
        t_ft = time.perf_counter() - t_ft
    thp_gb = anon_huge_gb()  # the host arenas ask for transparent huge pages (lane TLB reach)
    measured_cost = e.stats()["cost"]

    # device-resident step inputs (layer-major), outputs
    hid_d = [torch.as_tensor(np.ascontiguousarray(hidden[s * B:(s + 1) * B].transpose(1, 0, 2), np.float32),
                             device="cuda") for s in range(S)]
    fol_d = [torch.as_tensor(np.ascontiguousarray(follow[s * B:(s + 1) * B].T), device="cuda") for s in range(S)]
    y_d = torch.empty(L, B, H, dtype=torch.float32, device="cuda")

    def decode_leg(calibrate=False):
        for s in range(args.warmup):
            e.step_device(hid_d[s], fol_d[s], y_d)
        torch.cuda.synchronize()
        if calibrate:
            e.calibrate()  # measured t_io / t_g / t_attn / host-lane beta, C (fit_cost_params)
        e.reset_stats()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            t0 = time.perf_counter()
            for s in range(args.warmup, S):
                e.step_device(hid_d[s], fol_d[s], y_d)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
        st = e.stats()
        dev_ms = st["step_ms_total"] / max(1, st["steps"])
        if dist:
            t = torch.tensor([dev_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dev_ms = float(t.item())
            dist.barrier()
        return st, dev_ms, wall, clk.summary()

    # GPU-only executor: PreSched with beta = 1e9 (cpu_set always empty).
    e.set_cost(measured_cost["t_io"], measured_cost["t_g"], measured_cost["t_attn"], 1e9, 0)
    e.set_lookahead(0, False)
    legs = {"gpu_only": decode_leg()}
    if e.host_threads:
        # Host expert lane: PreSched with the host's measured cpu_cost (beta*m + C) —
        # plain PreSched (the reference executor), then the headline configuration with
        # the executor extensions (--lookahead / --steal-late) on the same engine.
        e.set_cost(**measured_cost)
        legs["host_lane"] = decode_leg(calibrate=True)
        head_cost = e.stats()["cost"]
        if args.lookahead or args.steal_late:
            e.set_cost(**measured_cost)
            e.set_lookahead(args.lookahead, bool(args.steal_late))
            legs["host_lane_lookahead"] = decode_leg(calibrate=True)
            # the e2e leg below measures the headline executor: plain PreSched again
            e.set_lookahead(0, False)
            e.set_cost(**head_cost)
    head = "host_lane" if "host_lane" in legs else "gpu_only"
    st, dev_ms, wall, clocks = legs[head]

    # end-to-end through the host-buffer C-ABI entry point (pinned host buffers), same executor
    hid_h = [torch.from_numpy(np.ascontiguousarray(hidden[s * B:(s + 1) * B], np.float32)).pin_memory()
             for s in range(S)]
    fol_h = [torch.from_numpy(np.ascontiguousarray(follow[s * B:(s + 1) * B])).pin_memory() for s in range(S)]
    hid_lm = [torch.from_numpy(np.ascontiguousarray(h.numpy().transpose(1, 0, 2))).pin_memory() for h in hid_h]
    fol_lm = [torch.from_numpy(np.ascontiguousarray(f.numpy().T)).pin_memory() for f in fol_h]
    y_h = torch.empty(L, B, H, dtype=torch.float32).pin_memory()
    ids_h = torch.empty(L, B, k, dtype=torch.int32).pin_memory()
    def step_host(s):
        ps.check(lib.ps_engine_decode_step_host(e.h, C.c_void_p(hid_lm[s].data_ptr()),
                                                C.c_void_p(fol_lm[s].data_ptr()), B,
                                                C.c_void_p(y_h.data_ptr()), C.c_void_p(ids_h.data_ptr())))
    for s in range(args.warmup):  # untimed warm-up of the host-buffer entry point (its staging)
        step_host(s)
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for s in range(args.warmup, S):
        ps.check(lib.ps_engine_decode_step_host(e.h, C.c_void_p(hid_lm[s].data_ptr()),
                                                C.c_void_p(fol_lm[s].data_ptr()), B,
                                                C.c_void_p(y_h.data_ptr()), C.c_void_p(ids_h.data_ptr())))
    e2e_s = (time.perf_counter() - t0) / args.steps
    if dist:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d_in = hid_lm[0].numel() * 4 + fol_lm[0].numel()
    d2h_out = y_h.numel() * 4 + ids_h.numel() * 4
    # Extra leg (after the headline's e2e): the same plain PreSched executor with the LLaPor
    # nets fine-tuned online (ps_llapor_fine_tune = predictor.cpp:654-663) on a separate
    # warm-up trace. The trained nets predict the hot, resident experts, PreSched then issues
    # no prefetches and the few loads are on-demand (so little H2D time is hidden), and the
    # lane takes the rest: faster in paired runs (profiles/README.md), reported beside.
    if args.ft_leg and e.host_threads and args.predictor == "llapor" and not args.llapor_finetune:
        sys.path.insert(0, str(ROOT / "scripts"))
        import configs_bench
        t_ft = time.perf_counter()
        configs_bench.finetune(torch, e, predictor, spec, gen, B, args.ft_leg, seed=4242 + rank)
        t_ft = time.perf_counter() - t_ft
        e.set_cost(**measured_cost)
        e.set_lookahead(0, False)
        legs["host_lane_llapor_ft"] = decode_leg(calibrate=True)
    e.close()
    # In-bench checksum (outside every timed region): the last e2e step's outputs vs the
    # CPU oracle — ids of all layers vs the f64 reference router, y of two layers vs the
    # oracle SwiGLU/combine on the same bf16 weights (tests/ hold the full parity suite).
    checksum = None
    if rank == 0 and not args.no_checksum:
        checksum = step_checksum(args, spec, gate, hidden[(S - 1) * B:S * B], follow[(S - 1) * B:S * B],
                                 zipf, y_h.numpy(), ids_h.numpy())

    # BASELINE config 5 (N > 1 only): Mixtral EP with a GLOBAL batch of 64 decode tokens
    # and a 4096-token prefill chunk, split over the ranks, same budget and executor.
    config5 = None
    if world > 1 and not args.no_config5:
        config5 = config5_legs(args, spec, gen, gate, zipf, ep, resident, budget_bytes, predictor, host_threads,
                               local, rank, world, dist)

    # Same steps with every expert resident (budget 100 %): the HBM-bound MoE layer.
    all_res = None
    prefill = None
    if not args.no_all_resident and world == 1:
        PT = args.prefill_tokens
        e2 = eng.Engine(spec, gen, max_batch=max(B, PT), weight_seed=args.weight_seed, gate=gate,
                        budget_bytes=L * E * spec.expert_bytes, resident=[(l, x) for l in range(L) for x in range(E)],
                        policy=args.policy, predictor=predictor, device=local)
        for s in range(args.warmup):
            e2.step_device(hid_d[s], fol_d[s], y_d)
        torch.cuda.synchronize()
        e2.reset_stats()
        for s in range(args.warmup, S):
            e2.step_device(hid_d[s], fol_d[s], y_d)
        torch.cuda.synchronize()
        st2 = e2.stats()
        if PT > 0:
            # Prefill chunk of PT tokens through the same engine (tcgen05 path): random
            # unit hidden states routed by the same gate matrices; inputs > L2.
            g = torch.Generator(device="cuda").manual_seed(5)
            ph = torch.randn(L, PT, H, device="cuda", generator=g)
            ph /= ph.norm(dim=-1, keepdim=True)
            pf = torch.zeros(L, PT, dtype=torch.uint8, device="cuda")
            py = torch.empty(L, PT, H, dtype=torch.float32, device="cuda")
            for _ in range(2):
                e2.step_device(ph, pf, py)
            torch.cuda.synchronize()
            e2.reset_stats()
            with ClockSampler(local) as pclk:
                for _ in range(args.prefill_steps):
                    e2.step_device(ph, pf, py)
                torch.cuda.synchronize()
            st3 = e2.stats()
            ms3 = st3["step_ms_total"] / max(1, st3["steps"])
            peak_tf, peak_tf_kind = bf16_peak()
            tf = st3["ffn_flops_total"] / (st3["ffn_ms_total"] / 1e3) / 1e12 if st3["ffn_ms_total"] > 0 else 0.0
            prefill = {"tokens_per_step": PT, "value": N_world(dist) * PT / (ms3 / 1e3), "unit": "tokens/s",
                       "ms_per_step": ms3, "moe_layer_us": ms3 * 1e3 / L,
                       "ffn_tflops": tf, "ffn_frac_of_bf16_peak": tf / peak_tf, "peak_tflops": peak_tf,
                       "peak_kind": peak_tf_kind,
                       "tc_launches": st3["tc_launches"], "clocks": pclk.summary(),
                       "route_phase_us_per_layer": st3["route_phase_ms_total"] * 1e3 / max(1, st3["layers"]),
                       "data": "random unit hidden states, all experts resident"}
            del ph, py
        e2.close()
        ms2 = st2["step_ms_total"] / max(1, st2["steps"])
        ach2 = st2["ffn_bytes_total"] / (st2["ffn_ms_total"] / 1e3) / 1e9 if st2["ffn_ms_total"] > 0 else 0.0
        layer_bytes = st2["ffn_bytes_total"] / max(1, st2["steps"]) / L
        all_res = {"value": N_world(dist) * B / (ms2 / 1e3), "unit": "tokens/s", "ms_per_step": ms2,
                   "moe_layer_us": ms2 * 1e3 / L, "ffn_achieved_gbs": ach2,
                   "ffn_frac_of_hbm": ach2 / measured_peaks()[0],
                   "layer_frac_of_hbm": layer_bytes / (ms2 / 1e3 / L) / 1e9 / measured_peaks()[0],
                   "route_phase_us_per_layer": st2["route_phase_ms_total"] * 1e3 / max(1, st2["layers"]),
                   "combine_us_per_layer": st2["combine_ms_total"] * 1e3 / max(1, st2["layers"]),
                   "gpu_launches": st2["kernel_launches"]}
    lib.ps_llapor_free(predictor)
    if ep is not None:
        ep.close()

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    N = world
    value = N * B / (dev_ms / 1e3)
    peak_hbm, peak_kind = measured_peaks()
    ffn_ms = st["ffn_ms_total"]
    ffn_launches = max(1, st["ffn_launches"])  # one persistent K3 kernel (gate_up + down) per launch
    # algorithmic bytes of the FFN launches = sum over launched experts with m_e > 0 of
    # 3*H*F*2 (weights; activations are <0.1% at decode)
    ffn_bytes = ffn_bytes_total(st, spec)
    achieved = ffn_bytes / (ffn_ms / 1e3) / 1e9 if ffn_ms > 0 else 0.0
    # DRAM traffic per launch from the committed ncu --set full capture of the same kernel
    # (profiles/r01_ffn_decode_traffic.json): measured bytes / algorithmic bytes, applied
    # to this run's algorithmic bytes per launch.
    traffic, traffic_src = None, None
    tpath = ROOT / "profiles" / "r01_ffn_decode_traffic.json"
    if tpath.exists():
        tj = json.loads(tpath.read_text())
        traffic = tj["traffic_over_algorithmic"] * ffn_bytes / ffn_launches
        traffic_src = f"{tj['source']}: traffic/algorithmic = {tj['traffic_over_algorithmic']:.4f}"
    leg_summary = {name: decode_summary(lst, lms, N, B, L) for name, (lst, lms, _, _) in legs.items()}
    for name in ("host_lane", "host_lane_lookahead", "host_lane_llapor_ft"):
        if "cpu_lane" in leg_summary.get(name, {}):
            leg_summary[name]["cpu_lane"]["threads"] = host_threads
    cpu_step_s, cpu_desc, cpu_legs, cpu_threads = (cpu_sample(args) if not args.no_cpu_baseline
                                                   else (None, "skipped", None, 0))
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": N, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (reference trace generator, hash-init bf16 weights)",
        "config": workload_config(args, spec, head),
        "moe_layer_us": dev_ms * 1e3 / L,
        "e2e": {"value": N * B / e2e_s, "unit": "tokens/s", "h2d_bytes_per_step": h2d_in,
                "d2h_bytes_per_step": d2h_out, "timing": "host wall-clock around ps_engine_decode_step_host"},
        "roofline": {"kernel": "K3 decode SwiGLU expert FFN (gate_up + down)", "bound": "hbm",
                     "achieved": achieved, "peak": peak_hbm, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / peak_hbm, "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic_bytes_per_launch": ffn_bytes / ffn_launches,
                     "avg_launch_us": ffn_ms * 1e3 / ffn_launches},
        "h2d": leg_summary[head]["h2d"],
        "executor": head,
        "host_lane": leg_summary.get("host_lane"),
        "host_lane_lookahead": leg_summary.get("host_lane_lookahead"),
        "host_lane_llapor_ft": (dict(leg_summary["host_lane_llapor_ft"], llapor_finetune_steps=args.ft_leg,
                                     llapor_finetune_s=t_ft) if "host_lane_llapor_ft" in leg_summary else None),
        "gpu_only": leg_summary["gpu_only"],
        "cpu_baseline": ({"value": args.batch / cpu_step_s, "unit": "tokens/s", "cores": cpu_threads,
                          "kind": "reference", "sample": cpu_desc, "host": host_info(),
                          "legs_1core_us": cpu_legs} if cpu_step_s else None),
        "checksum": checksum,
        "all_resident": all_res,
        "prefill": prefill,
        "clocks": clocks,
        "gpu_launches": st["kernel_launches"],
        "nccl_init": nccl_init_lines() if world > 1 else None,
        "config5_ep": config5,
        "hbm_footprint_gb": {"budget_resident_experts": budget_bytes / 1e9,
                             "resident_arena": len(resident) * spec.expert_bytes / 1e9,
                             "engine_total_device": hbm_engine / 1e9,
                             "note": "engine_total_device = device memory the engine allocated at create "
                                     "(resident arena + 2 on-demand and the prefetch staging slots with "
                                     "their z-slab landing buffers + routing/FFN scratch), cudaMemGetInfo delta"},
        "host_memory": {"anon_huge_pages_gb": thp_gb, "note": "transparent huge pages backing the pinned host "
                        "arenas after engine create (/proc/self/smaps_rollup); the lane streams them"},
        "wall_s_timed": wall, "engine_create_s": t_create, "llapor_finetune_s": t_ft,
        "cost_params_us": st["cost"],
    }
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


def config5_legs(args, spec, gen, gate, zipf, ep, resident, budget_bytes, predictor, host_threads, local, rank, world,
                 dist):
    """EP decode at a global batch of 64 and a 4096-token prefill chunk (BASELINE config 5):
    each rank routes 64/N (4096/N) tokens of one trace, dispatches them to the owners over
    NCCL, runs its experts through its own cache/loader/lane, combines at home. Device
    time per step is the max over ranks; value = global tokens / that time."""
    import torch

    import paper_2509_23638_b200 as ps
    from paper_2509_23638_b200 import engine as eng
    L, H = spec.num_layers, spec.hidden_dim
    Bd, Tp = 64 // world, 4096 // world
    e = eng.Engine(spec, gen, max_batch=max(Bd, Tp), weight_seed=args.weight_seed, gate=gate,
                   budget_bytes=budget_bytes, resident=resident, policy=args.policy, predictor=predictor,
                   device=local, ep=ep, host_threads=host_threads, compress_host=bool(args.compress))
    out = {}
    try:
        S = args.warmup + args.steps
        _, hd, fd, _ = ps.trace_inputs(gen, spec, 64 * S, 2000, want_gate=False)

        def timed(inputs, steps, warm):
            y = torch.empty(L, inputs[0][0].shape[1], H, dtype=torch.float32, device="cuda")
            for i in range(warm):
                e.step_device(inputs[i][0], inputs[i][1], y)
            torch.cuda.synchronize()
            e.reset_stats()
            dist.barrier()
            for i in range(warm, warm + steps):
                e.step_device(inputs[i % len(inputs)][0], inputs[i % len(inputs)][1], y)
            torch.cuda.synchronize()
            st = e.stats()
            t = torch.tensor([st["step_ms_total"] / max(1, st["steps"])], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item()), st

        dec = []
        for s_ in range(S):
            tok = hd[s_ * 64 + rank * Bd:s_ * 64 + (rank + 1) * Bd]
            fol = fd[s_ * 64 + rank * Bd:s_ * 64 + (rank + 1) * Bd]
            dec.append((torch.as_tensor(np.ascontiguousarray(tok.transpose(1, 0, 2), np.float32), device="cuda"),
                        torch.as_tensor(np.ascontiguousarray(fol.T), device="cuda")))
        ms, st = timed(dec, args.steps, args.warmup)
        out["decode_global_batch_64"] = {"value": 64 / (ms / 1e3), "unit": "tokens/s", "ms_per_step": ms,
                                         "tokens_per_rank": Bd, "cpu_experts_per_step_rank0": st["cpu_experts"] /
                                         max(1, st["steps"]), "ondemand_loads_per_step_rank0":
                                         st["ondemand_loads"] / max(1, st["steps"])}
        g = torch.Generator(device="cuda").manual_seed(11 + rank)
        ph = torch.randn(L, Tp, H, device="cuda", generator=g)
        ph /= ph.norm(dim=-1, keepdim=True)
        pf = torch.zeros(L, Tp, dtype=torch.uint8, device="cuda")
        ms, st = timed([(ph, pf)], max(2, args.prefill_steps), 2)
        out["prefill_4096"] = {"value": 4096 / (ms / 1e3), "unit": "tokens/s", "ms_per_step": ms,
                               "tokens_per_rank": Tp, "tc_launches_rank0": st["tc_launches"]}
    finally:
        e.close()
    return out


def nccl_init_lines(limit=6):
    """This process's NCCL INIT debug lines (NCCL_DEBUG_FILE set in main): communicator
    size, rank and transport as NCCL reports them."""
    import glob
    import socket
    pat = os.environ.get("NCCL_DEBUG_FILE", "").replace("%h", socket.gethostname()).replace("%p", str(os.getpid()))
    lines = []
    for path in glob.glob(pat) if pat else []:
        for ln in open(path, errors="replace"):
            if "Init COMPLETE" in ln or "nRanks" in ln or "comm 0x" in ln:
                lines.append(ln.strip())
    return lines[:limit]


def step_checksum(args, spec, gate, hidden, follow, zipf, y, ids, layers=None):
    import oracle as orc
    L, E, H, k = spec.num_layers, spec.experts_per_layer, spec.hidden_dim, spec.top_k
    F = spec.expert_bytes // (6 * H)
    layers = layers or [0, L - 1]
    _, ref_w, ref_ids = orc.or_route_trace(gate, hidden, follow, zipf, k)
    ids_ok = bool(np.array_equal(ids, ref_ids.transpose(1, 0, 2)))
    rel = []
    for l in layers:
        used = sorted(set(int(x) for x in np.unique(ids[l])))
        slabs = orc.bl_init_slabs([(l, x) for x in used], H, F, args.weight_seed)
        by_e = dict(zip(used, slabs))
        x = orc.f32_to_bf16(hidden[:, l].astype(np.float32))
        y_ref = orc.or_moe_layer([by_e.get(x_) for x_ in range(E)], H, F, x, ids[l],
                                 ref_w[:, l].astype(np.float32), True, os.cpu_count() or 1)
        rel.append(float(np.linalg.norm(y[l] - y_ref) / np.linalg.norm(y_ref)))
    return {"tokens": int(hidden.shape[0]), "ids_match_reference_router": ids_ok, "layers": layers,
            "y_rel_err_vs_oracle": rel, "tolerance": 2e-2, "ok": ids_ok and max(rel) < 2e-2,
            "source": "last e2e step (ps_engine_decode_step_host) vs oracle/or_route_trace + or_moe_layer"}


def default_host_threads(world=1):
    """Host expert lane threads: one per core, at most 16 (the engine and I/O threads
    mostly sleep on futexes/blocking events): on the B200 box's 16-core host 16 threads
    stream 178-182 GB/s vs 170-177 with 15 and 168-175 with 14 in alternating runs
    (profiles/r01_bench_lane_threads_14_15_16.jsonl; 14 beat 12 before,
    r01_bench_threads.jsonl); 0 without AVX512_BF16."""
    try:
        if "avx512_bf16" not in open("/proc/cpuinfo").read():
            return 0
    except OSError:
        return 0
    # one lane per rank (EP: every rank's lane computes its own cpu_set): the host's
    # cores split between the ranks of this node
    return max(1, min(16, (os.cpu_count() or 1) // max(1, world)))


def decode_summary(st, dev_ms, N, B, L):
    """Per-executor decode numbers: throughput, PCIe, hidden fraction, host lane."""
    steps = max(1, st["steps"])
    h2d_gbs = st["h2d_bytes"] / (st["h2d_busy_ms"] / 1e3) / 1e9 if st["h2d_busy_ms"] > 0 else 0.0
    out = {"value": N * B / (dev_ms / 1e3), "unit": "tokens/s", "ms_per_step": dev_ms,
           "host_outside_device_ms_per_step": {"prologue": st["host_head_ms_total"] / steps,
                                               "drain_and_measurement": st["host_tail_ms_total"] / steps},
           "moe_layer_us": dev_ms * 1e3 / L,
           "h2d": {"achieved_gbs": h2d_gbs, "peak_gbs": PCIE_H2D_PEAK_GBS, "frac": h2d_gbs / PCIE_H2D_PEAK_GBS,
                   "bytes_per_step": st["h2d_bytes"] / steps,
                   # expert bytes delivered per second of copy time (z-slabs: > the link rate)
                   "expert_gbs": st["h2d_expert_bytes"] / (st["h2d_busy_ms"] / 1e3) / 1e9 if st["h2d_busy_ms"] > 0
                   else 0.0,
                   "z_ratio": st["h2d_bytes"] / st["h2d_expert_bytes"] if st["h2d_expert_bytes"] > 0 else None,
                   "ondemand_loads_per_step": st["ondemand_loads"] / steps,
                   "prefetches_per_step": st["prefetches_committed"] / steps,
                   "prefetch_hits_per_step": st["prefetch_hits"] / steps,
                   # committed prefetches the target layer actually routed tokens to
                   "prefetch_use_rate": (st["prefetches_used"] / st["prefetches_committed"]
                                         if st["prefetches_committed"] else None),
                   "lookahead_prefetches_per_step": st["lookahead_prefetches"] / steps,
                   "stolen_prefetches_per_step": st["stolen_prefetches"] / steps,
                   # 1 - (compute-stream stall on copy events) / (copy-engine busy time)
                   "hidden_fraction": (1.0 - st["compute_wait_ms"] / st["h2d_busy_ms"]) if st["h2d_busy_ms"] > 0
                   else 1.0},
           "cost_params_us": st["cost"], "calibration_fit_cost_params": bool(st["calibration_fit"])}
    # host DRAM: everything non-resident is read from it, by the lane (its z-slab reads)
    # or by the PCIe DMA; roofline = the host's measured read bandwidth
    # (scripts/probes/host_stream.c on the GPU box, profiles/r02_host_stream.jsonl)
    step_s = dev_ms / 1e3
    lane_gbs = st["cpu_read_bytes"] / steps / step_s / 1e9
    dma_gbs = st["h2d_bytes"] / steps / step_s / 1e9
    peak = host_dram_peak()
    out["host_dram"] = {"lane_read_gbs": lane_gbs, "pcie_dma_read_gbs": dma_gbs, "total_gbs": lane_gbs + dma_gbs,
                        "peak_gbs": peak, "frac": (lane_gbs + dma_gbs) / peak if peak else None,
                        "peak_source": "profiles/r02_host_stream.jsonl (16-thread AVX-512 read stream, 32 GB)"}
    if st["cpu_experts"]:
        out["cpu_lane"] = {"experts_per_step": st["cpu_experts"] / steps,
                           "busy_ms_per_step": st["cpu_ms_total"] / steps,
                           "achieved_gbs": st["cpu_bytes_total"] / (st["cpu_ms_total"] / 1e3) / 1e9,
                           "threads": None}
    return out


def anon_huge_gb():
    try:
        for line in open("/proc/self/smaps_rollup"):
            if line.startswith("AnonHugePages:"):
                return int(line.split()[1]) / 1e6  # kB -> GB
    except OSError:
        pass
    return None


def host_dram_peak():
    """Best host-DRAM read bandwidth measured on the pool's GPU boxes (GB/s), if recorded."""
    p = ROOT / "profiles" / "r02_host_stream.jsonl"
    try:
        return max(json.loads(l)["best_gbs"] for l in p.read_text().splitlines() if l.strip())
    except (OSError, ValueError, KeyError):
        return None


def N_world(dist):
    return dist.get_world_size() if dist else 1


def ffn_bytes_total(st, spec):
    return st["ffn_bytes_total"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--model", default="mixtral")
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--budget", type=float, default=0.5)
    ap.add_argument("--policy", default="presched")
    ap.add_argument("--weight-seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-all-resident", action="store_true")
    ap.add_argument("--no-checksum", action="store_true")
    ap.add_argument("--no-config5", action="store_true", help="N>1: skip the BASELINE config-5 EP legs")
    ap.add_argument("--prefill-tokens", type=int, default=4096)
    ap.add_argument("--prefill-steps", type=int, default=5)
    ap.add_argument("--predictor", default="llapor", choices=["llapor", "gate", "perfect", "none"],
                    help="next-layer load predictor feeding PreSched (the reference's PredictFn menu)")
    ap.add_argument("--compress", type=int, default=1,
                    help="1: non-resident experts cross PCIe as lossless z-slabs (decoded on the GPU)")
    ap.add_argument("--lookahead", type=int, default=3, choices=[0, 1, 2, 3],
                    help="extra leg host_lane_lookahead: PreSched + lookahead top-up of the serial channel "
                         "(0 with --steal-late 0: no extra leg; the headline is always plain PreSched)")
    ap.add_argument("--steal-late", type=int, default=1,
                    help="1: the host lane computes committed prefetches whose copies land too late")
    ap.add_argument("--llapor-finetune", type=int, default=0,
                    help="warm-up steps of online LLaPor fine_tune on a separate trace before measuring")
    ap.add_argument("--ft-leg", type=int, default=16,
                    help="extra leg host_lane_llapor_ft: plain PreSched after N warm-up steps of online "
                         "LLaPor fine_tune (0: skip)")
    ap.add_argument("--host-threads", type=int, default=-1,
                    help="host expert lane threads (-1 auto, 0 = GPU-only executor)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # One process per GPU: relaunch under torchrun (the driver does this itself).
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), str(pathlib.Path(__file__).resolve()),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if world > 1 and args.impl == "ours":
        # NCCL init lines (communicator size/ranks) go to a per-process file; rank 0
        # copies its own into the JSON line (stdout carries only the JSON line).
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/tmp/ps_bench_nccl.%h.%p.log")
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
