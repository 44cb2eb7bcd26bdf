"""Python handle for the decode engine (K5) and the per-op GPU wrappers.

Mirrors the reference's experiment flow (experiment.cpp:310-360): routing trace ->
hot-expert table -> plan_residency under the HBM budget -> per-layer PreSched-driven
execution. Device buffers come from torch (plumbing); all compute is the CUDA library.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import capi
from .capi import check, load


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2509_23638_b200 GPU ops need a CUDA device (no CPU fallback)")
    return torch


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _stream(torch):
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def route(x, gate, bias, follow, prev_ids, k, want_logits=True):
    """K1 on device tensors: x [B,H] f32, gate [E,H] f32 -> (logits, weights, ids, counts, x_bf16)."""
    torch = _torch()
    B, H = x.shape
    E = gate.shape[0]
    dev = x.device
    logits = torch.empty(B, E, dtype=torch.float32, device=dev) if want_logits else None
    weights = torch.empty(B, E, dtype=torch.float32, device=dev)
    ids = torch.empty(B, k, dtype=torch.int32, device=dev)
    counts = torch.empty(E, dtype=torch.int32, device=dev)
    xb = torch.empty(B, H, dtype=torch.int16, device=dev)
    pk = prev_ids.shape[1] if prev_ids is not None else 0
    check(load().ps_route_topk(_ptr(x), _ptr(gate), _ptr(bias), _ptr(follow), _ptr(prev_ids), pk, B, H, E, k,
                               _ptr(logits), _ptr(weights), _ptr(ids), _ptr(counts), _ptr(xb), _stream(torch)))
    return logits, weights, ids, counts, xb


def hot_table(spec: capi.ModelSpec, gate: np.ndarray, hidden: np.ndarray, follow: np.ndarray,
              zipf: np.ndarray) -> np.ndarray:
    """Activation frequency per (layer, expert) of a routing trace, routed on the GPU
    (build_hot_table, predictor.cpp:405-424). hidden [B,L,H], follow [B,L]."""
    torch = _torch()
    L, E, k = spec.num_layers, spec.experts_per_layer, spec.top_k
    g = torch.as_tensor(np.ascontiguousarray(gate, np.float32), device="cuda")
    hid = torch.as_tensor(np.ascontiguousarray(hidden.transpose(1, 0, 2), np.float32), device="cuda")
    fol = torch.as_tensor(np.ascontiguousarray(follow.T), device="cuda")
    bias = torch.as_tensor(np.array([[-z * np.log(e + 1.0) for e in range(E)] for z in zipf], np.float32),
                           device="cuda")
    freq = np.zeros((L, E), np.int64)
    prev = None
    for l in range(L):
        _, _, ids, counts, _ = route(hid[l], g[l], bias[l], fol[l], prev, k, want_logits=False)
        prev = ids
        freq[l] = counts.cpu().numpy()
    return freq


class EpComm:
    """NCCL communicator for expert parallelism (ps_ep_comm). `unique_id` (128 bytes)
    comes from rank 0's EpComm.unique_id() and is broadcast by the caller (e.g. with
    torch.distributed); world=1 needs no broadcast."""

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(load().ps_ep_unique_id(buf, 128))
        return buf.raw

    def __init__(self, rank: int = 0, world: int = 1, device: int = 0, unique_id: bytes | None = None):
        uid = unique_id if unique_id is not None else EpComm.unique_id()
        self.h = C.c_void_p()
        check(load().ps_ep_comm_create(uid, rank, world, device, C.byref(self.h)))
        self.rank, self.world = rank, world

    @classmethod
    def loopback(cls, world: int, device: int = 0):
        """`world` communicators of the in-process transport (ps_ep_loopback_create), one
        per host thread of this process: the EP engine at G > 1 on one GPU."""
        arr = (C.c_void_p * world)()
        check(load().ps_ep_loopback_create(world, device, arr))
        out = []
        for r in range(world):
            c = cls.__new__(cls)
            c.h = C.c_void_p(arr[r])
            c.rank, c.world = r, world
            out.append(c)
        return out

    def owned(self, E: int):
        return [e for e in range(E) if e % self.world == self.rank]

    def close(self):
        if self.h:
            check(load().ps_ep_comm_destroy(self.h))
            self.h = None


class Engine:
    """ps_engine handle. gate: [L,E,H] router matrices (from ps.trace_inputs)."""

    def __init__(self, spec: capi.ModelSpec, gen_cfg, *, max_batch: int, weight_seed: int = 0,
                 gate: np.ndarray, budget_fraction: float | None = None, budget_bytes: int | None = None,
                 resident=None, trace_hidden=None, trace_follow=None, policy: str = "presched",
                 predictor=None, cost=None, prefetch_slots: int = 8, device: int = 0, ep=None,
                 n_shared: int = 0, host_threads: int = 0, compress_host: bool = False,
                 predictor_kind: str = "auto", stats_ranking=None, expert_weights=None, lookahead: int = 0,
                 steal_late: bool = False):
        from . import parse_policy, plan_residency, trace_inputs  # noqa: F401
        self.lib = load()
        self.spec = spec
        L, E, H = spec.num_layers, spec.experts_per_layer, spec.hidden_dim
        if budget_bytes is None:
            budget_bytes = int(round((budget_fraction or 0.0) * L * E)) * spec.expert_bytes
        self.budget_bytes = budget_bytes
        zipf = np.array([[gen_cfg.input, gen_cfg.middle, gen_cfg.output][self._group(l)].zipf_s for l in range(L)])
        if resident is None:
            if trace_hidden is None:
                resident = []
            else:
                self.freq = hot_table(spec, gate, trace_hidden, trace_follow, zipf)
                resident = plan_residency(self.freq, budget_bytes, spec.expert_bytes)
        self.resident = list(resident)
        res = np.array(self.resident, np.int32).reshape(-1, 2)
        self._res = res
        cfg = capi.EngineConfig()
        cfg.spec = spec
        cfg.gen = gen_cfg
        cfg.weight_seed = weight_seed
        cfg.budget_bytes = budget_bytes
        cfg.resident = res.ctypes.data_as(C.POINTER(C.c_int32))
        cfg.n_resident = len(res)
        cfg.max_batch = max_batch
        cfg.prefetch_slots = prefetch_slots
        cfg.policy = parse_policy(policy)
        if cost is not None:
            cfg.cost = capi.CostParams(*cost)
        cfg.predictor = predictor
        cfg.device = device
        cfg.host_pinned = 1
        cfg.ep = ep.h if isinstance(ep, EpComm) else ep
        cfg.n_shared = n_shared
        cfg.host_threads = host_threads
        cfg.compress_host = int(bool(compress_host))
        cfg.lookahead = lookahead
        cfg.steal_late = int(bool(steal_late))
        kinds = {"auto": 0, "llapor": 1, "gate": 2, "stats": 3, "perfect": 4, "none": 5}
        cfg.predictor_kind = kinds[predictor_kind]
        if stats_ranking is not None:
            self._rank = np.ascontiguousarray(stats_ranking, np.int32).reshape(-1)
            cfg.stats_ranking = self._rank.ctypes.data_as(C.POINTER(C.c_int32))
        if expert_weights is not None:  # caller-supplied slabs: list [L*(E+n_shared)] of uint16 arrays / None
            self._weights = list(expert_weights)
            self._wptrs = (C.c_void_p * len(self._weights))(
                *[w.ctypes.data if w is not None else None for w in self._weights])
            cfg.expert_weights = C.cast(self._wptrs, C.POINTER(C.c_void_p))
        self.host_threads = host_threads
        h = C.c_void_p()
        check(self.lib.ps_engine_create(C.byref(cfg), C.byref(h)))
        self.h = h
        g32 = np.ascontiguousarray(gate, np.float32)
        check(self.lib.ps_engine_set_router(self.h, g32.ctypes.data_as(C.c_void_p)))
        self.max_batch = max_batch

    def _group(self, l):
        s = self.spec
        return 0 if l < s.group_begin_middle else (1 if l < s.group_begin_output else 2)

    def step_host(self, hidden: np.ndarray, follow: np.ndarray):
        """One decode step from host buffers. hidden [B,L,H] (trace order), follow [B,L].
        Returns y [L,B,H] f32 and ids [L,B,k]."""
        B, L, H = hidden.shape
        hid = np.ascontiguousarray(hidden.transpose(1, 0, 2), np.float32)
        fol = np.ascontiguousarray(follow.T, np.uint8)
        y = np.empty((L, B, H), np.float32)
        ids = np.empty((L, B, self.spec.top_k), np.int32)
        check(self.lib.ps_engine_decode_step_host(self.h, hid.ctypes.data_as(C.c_void_p),
                                                   fol.ctypes.data_as(C.c_void_p), B,
                                                   y.ctypes.data_as(C.c_void_p), ids.ctypes.data_as(C.c_void_p)))
        return y, ids

    def step_routed(self, hidden, active, gate_weights):
        """Replay a trace's routing (prescope::Trace arrays, [B,L,...] trace order): hidden
        [B,L,H], active [B,L,k], gate_weights [B,L,E]. Returns y [L,B,H] f32."""
        torch = _torch()
        B, L, H = hidden.shape
        hid = torch.as_tensor(np.ascontiguousarray(hidden.transpose(1, 0, 2), np.float32), device="cuda")
        ids = torch.as_tensor(np.ascontiguousarray(active.transpose(1, 0, 2), np.int32), device="cuda")
        w = torch.as_tensor(np.ascontiguousarray(gate_weights.transpose(1, 0, 2), np.float32), device="cuda")
        y = torch.empty(L, B, H, dtype=torch.float32, device="cuda")
        check(self.lib.ps_engine_decode_step_routed(self.h, _ptr(hid), _ptr(ids), _ptr(w), B, _ptr(y)))
        torch.cuda.synchronize()
        return y.cpu().numpy()

    def step_device(self, hidden_lbh, follow_lb, y_lbh, ids_lbk=None):
        """One decode step on device tensors (layer-major)."""
        B = hidden_lbh.shape[1]
        check(self.lib.ps_engine_decode_step(self.h, _ptr(hidden_lbh), _ptr(follow_lb), B, _ptr(y_lbh),
                                             _ptr(ids_lbk)))

    def step_begin(self, B: int):
        """Per-layer ABI: start a decode pass of B tokens (ps_engine_step_begin)."""
        check(self.lib.ps_engine_step_begin(self.h, B))

    def layer_forward(self, layer: int, x_bh, follow_b, y_bh, ids_bk=None, stream=None):
        """One MoE layer on device tensors (ps_engine_layer_forward); `stream`: a
        torch.cuda.Stream the layer is ordered with (default: torch's current stream)."""
        torch = _torch()
        st = stream if stream is not None else torch.cuda.current_stream()
        check(self.lib.ps_engine_layer_forward(self.h, layer, _ptr(x_bh), _ptr(follow_b), _ptr(y_bh), _ptr(ids_bk),
                                               C.c_void_p(st.cuda_stream)))

    def step_end(self):
        check(self.lib.ps_engine_step_end(self.h))

    def stats(self) -> dict:
        s = capi.EngineStats()
        check(self.lib.ps_engine_get_stats(self.h, C.byref(s)))
        d = {f: getattr(s, f) for f, _ in capi.EngineStats._fields_ if f != "cost"}
        c = s.cost
        d["cost"] = dict(t_io=c.t_io, t_g=c.t_g, t_attn=c.t_attn, beta=c.beta, startup=c.startup)
        return d

    def last_timeline(self, cap: int = 1 << 16):
        """Measured timeline of the last step: (events, truth [L,E], resident [L,E],
        layer_start, layer_end) — events as (t_start, t_end, resource, kind, layer,
        expert, tokens) in us from the step start."""
        L, E = self.spec.num_layers, self.spec.experts_per_layer
        ev = (capi.TimelineEvent * cap)()
        ls, le = (C.c_int64 * L)(), (C.c_int64 * L)()
        tl = capi.Timeline(ev, cap, 0, ls, le, 0, None)
        truth = np.zeros((L, E), np.int32)
        res = np.zeros((L, E), np.uint8)
        check(self.lib.ps_engine_last_timeline(self.h, C.byref(tl), truth.ctypes.data_as(C.c_void_p),
                                               res.ctypes.data_as(C.c_void_p)))
        events = [(ev[i].t_start, ev[i].t_end, ev[i].resource, ev[i].kind, ev[i].layer, ev[i].expert, ev[i].tokens)
                  for i in range(tl.n_events)]
        return events, truth, res, list(ls), list(le)

    def verify_last_step(self):
        """verify_timeline (simulator.cpp:323-394) on the measured timeline of the last
        step (measured mode: transfer durations are not the modelled t_io)."""
        events, truth, res, _, _ = self.last_timeline()
        from . import _instance
        inst, keep = _instance(truth, np.zeros_like(truth), res)
        arr = (capi.TimelineEvent * max(1, len(events)))(*[capi.TimelineEvent(*x) for x in events])
        n = C.c_int()
        buf = C.create_string_buffer(1 << 16)
        st = self.stats()["cost"]
        params = capi.CostParams(st["t_io"], st["t_g"], st["t_attn"], st["beta"], st["startup"], 0)
        check(self.lib.ps_verify_timeline_ex(arr, len(events), C.byref(inst), C.byref(params), 1, C.byref(n), buf,
                                             len(buf)))
        del keep
        return [m for m in buf.value.decode().split("\n") if m]

    def calibrate(self):
        """Replace PreSched costs with the measured means (ps_engine_calibrate)."""
        c = capi.CostParams()
        check(self.lib.ps_engine_calibrate(self.h, C.byref(c)))
        return dict(t_io=c.t_io, t_g=c.t_g, t_attn=c.t_attn, beta=c.beta, startup=c.startup)

    def last_predictions(self):
        """[L,E] predicted token counts of the last step (row l: predicted at layer l-1)."""
        out = np.zeros((self.spec.num_layers, self.spec.experts_per_layer), np.int32)
        check(self.lib.ps_engine_last_predictions(self.h, out.ctypes.data_as(C.c_void_p)))
        return out

    def last_routing(self, B: int):
        """(ids [L,B,k] i32, gate weights [L,B,E] f32) of the last completed step."""
        L, E, k = self.spec.num_layers, self.spec.experts_per_layer, self.spec.top_k
        ids = np.empty((L, B, k), np.int32)
        w = np.empty((L, B, E), np.float32)
        check(self.lib.ps_engine_last_routing(self.h, ids.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p)))
        return ids, w

    def fine_tune_predictor(self, predictor, hidden_lbh, steps: int = 1, lr: float = 1e-3, layers=None):
        """Online LLaPor fine_tune (predictor.cpp:654-663) on the last step's observations:
        net l learns (hidden, routing) of layer l-1 -> routing of layer l. hidden_lbh:
        the step's gating inputs [L,B,H] (host). The engine's next step uses the
        updated nets (their GPU copies refresh before the next forward)."""
        L = self.spec.num_layers
        B = hidden_lbh.shape[1]
        ids, w = self.last_routing(B)
        k = self.spec.top_k
        for l in (layers or range(1, L)):
            hid = np.ascontiguousarray(hidden_lbh[l - 1], np.float64)
            gp = np.ascontiguousarray(w[l - 1], np.float64)
            ap, a = np.ascontiguousarray(ids[l - 1]), np.ascontiguousarray(ids[l])
            check(self.lib.ps_llapor_fine_tune(predictor, l, B, hid.ctypes.data_as(C.c_void_p),
                                               ap.ctypes.data_as(C.c_void_p), k, gp.ctypes.data_as(C.c_void_p),
                                               a.ctypes.data_as(C.c_void_p), k, steps, lr))

    def set_lookahead(self, lookahead: int, steal_late: bool = False):
        check(self.lib.ps_engine_set_lookahead(self.h, lookahead, int(bool(steal_late))))

    def set_cost(self, t_io, t_g, t_attn, beta, startup):
        """Replace the PreSched cost parameters (ps_engine_set_cost)."""
        check(self.lib.ps_engine_set_cost(self.h, C.byref(capi.CostParams(t_io, t_g, t_attn, beta, startup, 0))))

    def reset_stats(self):
        check(self.lib.ps_engine_reset_stats(self.h))

    def close(self):
        if getattr(self, "h", None):
            check(self.lib.ps_engine_destroy(self.h))
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
