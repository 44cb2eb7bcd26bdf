"""TEST / BASELINE INFRASTRUCTURE ONLY: the CPU arm of bench.py (`--impl reference` and
the `cpu_baseline` leg). Loads only oracle/ (liboracle.so + the UNMODIFIED reference in
oracle/_ref) — never the product library.

One decode step of the reference's CPU path for the bench workload, timed whole:

  1. router  — generate_trace's router (workload.cpp:176-202) on the reference trace's
               hidden states: or_route_batch (the f64 restatement, bit-exact to the
               trace's gate weights — asserted every step), OpenMP over tokens;
  2. LLaPor  — the reference's pca_apply + forward + predict_topk (predictor.cpp:
               116-124, 166-247, 669-672) through oracle/_ref on random-init nets at the
               bench's full shape (P=256/512, widths 32/48, written as an LLPC checkpoint
               and read by the reference's load_checkpoint), nets[l+1] on layer-l
               features for every (token, layer) (experiment.cpp:82-112), host threads
               over tokens;
  3. plan    — the reference's simulate_policy(presched) (simulator.cpp:61-242) over the
               step's true and predicted loads with the hot-table residency
               (predictor.cpp:405-433) of the same warm-up trace the GPU arm uses;
  4. experts — the SwiGLU experts + combine the reference does not have (SURVEY.md §8a
               a17/a18), as oracle/cpu_port.c's port (each routed expert streamed once,
               f32 AVX-512, all host cores) on the same hash-initialised bf16 weights.
"""
from __future__ import annotations

import os
import tempfile
import time

import numpy as np

from . import (bl_init_slabs, bl_moe_layer, f32_to_bf16, or_route_batch, ref_check, ref_gen, ref_lib,
               ref_llapor_predict_batch, ref_router_inputs, ref_simulate, ref_spec_preset, ref_time_legs, ref_trace)
from .llpc import random_nets, write_llpc

# TraceGenConfig defaults of the bench: (rho, kappa, zipf) per group
DEFAULT_GEN = {"input": (0.9, 0.5, 0.5), "middle": (0.95, 0.6, 1.0), "output": (0.9, 0.5, 0.5)}
# PreSched costs for the simulate leg: the GPU arm's calibrated host-lane executor values
# (BENCH_r01: t_io 4485, t_g 70, t_attn 59 us, beta 0.35 us/token, C 2013 us)
SIM_PARAMS = (4485, 70, 59, 0.35, 2013, 0)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class RefArm:
    """The reference CPU path of the bench workload. `ffn_layers`: the layers whose
    experts are materialised and computed (None = all: a whole step)."""

    def __init__(self, model="mixtral", batch=16, budget=0.5, steps=1, seed=1000, weight_seed=1,
                 threads=None, ffn_layers=None, p_in=256, p_mid=512):
        self.threads = threads or os.cpu_count() or 1
        self.spec = spec = ref_spec_preset(model)
        self.L, self.E, self.k, self.H = spec.num_layers, spec.experts, spec.top_k, spec.hidden
        self.F = spec.expert_bytes // (6 * self.H)
        self.B = batch
        self.gen = ref_gen(*[DEFAULT_GEN[g] for g in ("input", "middle", "output")])
        n_tok = batch * steps
        self.hidden, self.gw, self.act = ref_trace(self.gen, spec, n_tok, seed)
        self.gate, self.follow, self.zipf = ref_router_inputs(self.gen, spec, n_tok, seed)
        # hot-table residency from the GPU arm's warm-up trace (64 tokens, same seed)
        budget_bytes = int(round(budget * self.L * self.E)) * spec.expert_bytes
        self.budget_bytes = budget_bytes
        pairs = np.empty(2 * self.L * self.E, np.int32)
        import ctypes as C
        n = C.c_int()
        ref_check(ref_lib().ref_residency(C.byref(self.gen), C.byref(spec), 64, seed, budget_bytes,
                                          pairs.ctypes.data, C.byref(n)))
        self.resident = np.zeros((self.L, self.E), bool)
        for i in range(n.value):
            self.resident[pairs[2 * i], pairs[2 * i + 1]] = True
        # LLaPor nets at the bench's full shape, read by the reference's load_checkpoint
        fd, self._llpc = tempfile.mkstemp(suffix=".llpc")
        os.close(fd)
        write_llpc(self._llpc, spec, random_nets(spec, p_in, p_mid, 32, 48, seed=7))
        self.llapor = ref_lib().ref_llapor_load(self._llpc.encode())
        if not self.llapor:
            raise RuntimeError("reference load_checkpoint failed: " + ref_lib().ref_last_error().decode())
        os.unlink(self._llpc)
        self.ffn_layers = list(range(self.L)) if ffn_layers is None else list(ffn_layers)
        t0 = time.perf_counter()
        keys = [(l, e) for l in self.ffn_layers for e in range(self.E)]
        self.slabs = dict(zip(keys, bl_init_slabs(keys, self.H, self.F, weight_seed, self.threads)))
        self.init_s = time.perf_counter() - t0

    def close(self):
        if self.llapor:
            ref_lib().ref_llapor_free(self.llapor)
            self.llapor = None
        self.slabs = {}

    def step(self, s):
        """Step s (tokens s*B ... s*B+B-1): returns (seconds, {phase: seconds}, y [L',B,H])."""
        B, L, E, k, H, F = self.B, self.L, self.E, self.k, self.H, self.F
        sl = slice(s * B, (s + 1) * B)
        hid = self.hidden[sl]
        ph = {}
        t0 = time.perf_counter()
        w, ids = or_route_batch(self.gate, hid, self.follow[sl], self.zipf, k, self.threads)
        t1 = time.perf_counter()
        truth = np.zeros((L, E), np.int32)
        pred = np.zeros((L, E), np.int32)
        for l in range(L):
            truth[l] = np.bincount(ids[:, l].ravel(), minlength=E)
            if l + 1 < L:
                top = ref_llapor_predict_batch(self.llapor, l + 1, hid[:, l], ids[:, l], w[:, l], k, self.threads)
                pred[l + 1] = np.bincount(top.ravel(), minlength=E)
        t2 = time.perf_counter()
        rc, sim = ref_simulate(truth, pred, SIM_PARAMS, "presched", self.resident)
        if rc != 0:
            raise RuntimeError(f"reference simulate_policy rc={rc}: {ref_lib().ref_last_error().decode()}")
        t3 = time.perf_counter()
        ys = []
        for l in self.ffn_layers:
            x = f32_to_bf16(hid[:, l].astype(np.float32))
            slabs = [self.slabs[(l, e)] if truth[l, e] else None for e in range(E)]
            ys.append(bl_moe_layer(slabs, H, F, x, ids[:, l], w[:, l].astype(np.float32), self.threads))
        t4 = time.perf_counter()
        # the arm routes exactly as the reference trace did
        assert np.array_equal(ids, self.act[sl]) and np.array_equal(w, self.gw[sl]), "router restatement drifted"
        ph = {"router": t1 - t0, "llapor": t2 - t1, "presched_simulate": t3 - t2, "experts": t4 - t3,
              "makespan_ticks": sim["makespan"]}
        return t4 - t0, ph, np.stack(ys) if ys else None

    def legs_1core(self, min_seconds=0.25):
        """us per call of the reference's hot-path functions on one core."""
        return ref_time_legs(self.gen, self.spec, self.B, 1000, self.llapor, self.budget_bytes, SIM_PARAMS,
                             min_seconds)
