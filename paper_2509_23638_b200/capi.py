"""ctypes binding of the C ABI in include/ps_api.h (libprescope_b200.so).

Plumbing only: the product is the C++/CUDA library. The loader fails loudly when the
library is missing — there is no Python or CPU fallback for any GPU entry point.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib

_HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = _HERE / "libprescope_b200.so"

PS_OK, PS_EINVAL, PS_ERANGE, PS_ERUNTIME, PS_ECUDA, PS_ENCCL = range(6)
PS_POLICY_PRESCHED, PS_POLICY_GREEDY, PS_POLICY_ONDEMAND, PS_POLICY_FIXED, PS_POLICY_ORACLE = range(5)
PS_LOC_RESIDENT, PS_LOC_INFLIGHT, PS_LOC_HOST = range(3)
PS_MAX_GROUP = 256


class PsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[ps_status={status}] {msg}")
        self.status = status


class ModelSpec(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("experts_per_layer", C.c_int32), ("top_k", C.c_int32),
                ("hidden_dim", C.c_int32), ("expert_bytes", C.c_uint64), ("group_begin_middle", C.c_int32),
                ("group_begin_output", C.c_int32)]


class GroupGen(C.Structure):
    _fields_ = [("rho", C.c_double), ("kappa", C.c_double), ("zipf_s", C.c_double)]


class TraceGenConfig(C.Structure):
    _fields_ = [("input", GroupGen), ("middle", GroupGen), ("output", GroupGen), ("noise_scale", C.c_double)]


class CostParams(C.Structure):
    _fields_ = [("t_io", C.c_int64), ("t_g", C.c_int64), ("t_attn", C.c_int64), ("beta", C.c_double),
                ("startup", C.c_int64), ("alpha", C.c_int64)]


class ExpertLoad(C.Structure):
    _fields_ = [("expert", C.c_int32), ("layer", C.c_int32), ("tokens", C.c_int32), ("location", C.c_int32)]


class HitStats(C.Structure):
    _fields_ = [("r_hit", C.c_double), ("r_miss", C.c_double), ("window", C.c_int32)]


class LayerInputs(C.Structure):
    _fields_ = [("e_cur", C.POINTER(ExpertLoad)), ("n_cur", C.c_int32),
                ("e_next", C.POINTER(ExpertLoad)), ("n_next", C.c_int32),
                ("e_next2", C.POINTER(ExpertLoad)), ("n_next2", C.c_int32),
                ("params", CostParams), ("stats", HitStats)]


class DecisionTrace(C.Structure):
    _fields_ = [("sweep_gpu", C.POINTER(C.c_int64)), ("sweep_cpu", C.POINTER(C.c_int64)), ("n_sweep", C.c_int32),
                ("t_g_at_split", C.c_int64), ("t_c_at_split", C.c_int64), ("t_gap", C.c_int64),
                ("f", C.c_double), ("f_int", C.c_int32), ("xi", C.c_double),
                ("widened_window", C.c_int32), ("all_gpu_fallback", C.c_int32)]


class LayerPlan(C.Structure):
    _fields_ = [("cpu_set", C.POINTER(ExpertLoad)), ("n_cpu", C.c_int32),
                ("ondemand_seq", C.POINTER(ExpertLoad)), ("n_ondemand", C.c_int32),
                ("prefetch_seq", C.POINTER(ExpertLoad)), ("n_prefetch", C.c_int32),
                ("prefetch_from_widened", C.c_int32), ("split_index", C.c_int32),
                ("issued_prefetches", C.c_int32), ("trace", DecisionTrace)]


class Policy(C.Structure):
    _fields_ = [("kind", C.c_int32), ("fixed_prefetch", C.c_int32)]


class PipelineInstance(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("experts", C.c_int32), ("truth", C.POINTER(C.c_int32)),
                ("predicted", C.POINTER(C.c_int32)), ("resident", C.POINTER(C.c_uint8)),
                ("groups", C.POINTER(C.c_int32))]


class TimelineEvent(C.Structure):
    _fields_ = [("t_start", C.c_int64), ("t_end", C.c_int64), ("resource", C.c_int32), ("kind", C.c_int32),
                ("layer", C.c_int32), ("expert", C.c_int32), ("tokens", C.c_int32)]


class Timeline(C.Structure):
    _fields_ = [("events", C.POINTER(TimelineEvent)), ("cap_events", C.c_int32), ("n_events", C.c_int32),
                ("layer_start", C.POINTER(C.c_int64)), ("layer_end", C.POINTER(C.c_int64)),
                ("makespan", C.c_int64), ("plan_summary", C.POINTER(C.c_int32))]


class SimOptions(C.Structure):
    _fields_ = [("cpu_slots", C.c_int32), ("prefetch_slots", C.c_int32), ("initial_hit_rate", C.c_double),
                ("hit_window", C.c_int32)]


class Metrics(C.Structure):
    _fields_ = [("makespan", C.c_int64), ("decode_latency", C.c_int64), ("throughput_tokens_per_s", C.c_double),
                ("io_busy_fraction", C.c_double), ("gpu_idle_fraction", C.c_double)]


class ExpertGroup(C.Structure):
    _fields_ = [("n", C.c_int32), ("experts", C.c_int32 * PS_MAX_GROUP), ("slabs", C.c_void_p * PS_MAX_GROUP)]


class CacheConfig(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("experts", C.c_int32), ("expert_bytes", C.c_uint64),
                ("host_slabs", C.POINTER(C.c_void_p)), ("resident", C.POINTER(C.c_int32)), ("n_resident", C.c_int32),
                ("budget_bytes", C.c_uint64), ("n_slots", C.c_int32), ("device", C.c_int32)]


class CacheStats(C.Structure):
    _fields_ = [("prefetches", C.c_int64), ("ondemand_loads", C.c_int64), ("prefetches_cancelled", C.c_int64),
                ("slot_hits", C.c_int64), ("resident_hits", C.c_int64)]


class EngineConfig(C.Structure):
    _fields_ = [("spec", ModelSpec), ("gen", TraceGenConfig), ("weight_seed", C.c_uint64),
                ("budget_bytes", C.c_uint64), ("resident", C.POINTER(C.c_int32)), ("n_resident", C.c_int32),
                ("max_batch", C.c_int32), ("prefetch_slots", C.c_int32), ("policy", Policy),
                ("cost", CostParams), ("predictor", C.c_void_p), ("device", C.c_int32),
                ("host_pinned", C.c_int32), ("ep", C.c_void_p), ("n_shared", C.c_int32),
                ("host_threads", C.c_int32), ("compress_host", C.c_int32), ("predictor_kind", C.c_int32),
                ("stats_ranking", C.POINTER(C.c_int32)), ("expert_weights", C.POINTER(C.c_void_p)),
                ("lookahead", C.c_int32), ("steal_late", C.c_int32)]


class EngineStats(C.Structure):
    _fields_ = [("steps", C.c_int64), ("layers", C.c_int64), ("ondemand_loads", C.c_int64),
                ("prefetches_committed", C.c_int64), ("prefetches_cancelled", C.c_int64),
                ("prefetch_hits", C.c_int64), ("resident_hits", C.c_int64), ("h2d_bytes", C.c_double),
                ("h2d_busy_ms", C.c_double), ("compute_wait_ms", C.c_double), ("step_ms_total", C.c_double),
                ("ffn_ms_total", C.c_double), ("ffn_bytes_total", C.c_double),
                ("route_phase_ms_total", C.c_double), ("combine_ms_total", C.c_double),
                ("ffn_flops_total", C.c_double), ("tc_launches", C.c_int64), ("ffn_launches", C.c_int64),
                ("kernel_launches", C.c_int64),
                ("cost", CostParams), ("cpu_experts", C.c_int64), ("cpu_ms_total", C.c_double),
                ("cpu_bytes_total", C.c_double), ("z_decodes", C.c_int64), ("h2d_expert_bytes", C.c_double),
                ("lookahead_prefetches", C.c_int64), ("stolen_prefetches", C.c_int64),
                ("calibration_fit", C.c_int64), ("prefetches_used", C.c_int64),
                ("cpu_read_bytes", C.c_double), ("host_head_ms_total", C.c_double),
                ("host_tail_ms_total", C.c_double)]


PLAN_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(LayerInputs), C.c_int, C.POINTER(LayerPlan))

_P = C.c_void_p
_SIGS = {
    "ps_last_error": (C.c_char_p, []),
    "ps_version": (C.c_char_p, []),
    "ps_spec_validate": (C.c_int, [C.POINTER(ModelSpec)]),
    "ps_spec_group_of": (C.c_int, [C.POINTER(ModelSpec), C.c_int, C.POINTER(C.c_int)]),
    "ps_spec_preset": (C.c_int, [C.c_char_p, C.POINTER(ModelSpec)]),
    "ps_desk_scale": (C.c_int, [C.POINTER(ModelSpec), C.c_int, C.c_int, C.c_int, C.POINTER(ModelSpec)]),
    "ps_spec_ffn_dim": (C.c_int, [C.POINTER(ModelSpec), C.POINTER(C.c_int)]),
    "ps_topk_indices": (C.c_int, [_P, C.c_int, C.c_int, _P]),
    "ps_routing_map": (C.c_int, [C.POINTER(ModelSpec), C.c_int]),
    "ps_trace_inputs": (C.c_int, [C.POINTER(TraceGenConfig), C.POINTER(ModelSpec), C.c_int, C.c_uint64,
                                  _P, _P, _P, _P]),
    "ps_to_ticks": (C.c_int64, [C.c_double]),
    "ps_cost_params_validate": (C.c_int, [C.POINTER(CostParams)]),
    "ps_hit_stats_record": (C.c_int, [C.POINTER(HitStats), C.c_int]),
    "ps_cpu_cost": (C.c_int, [C.c_int, C.POINTER(CostParams), C.POINTER(C.c_int64)]),
    "ps_overlap_prefetch_count": (C.c_int, [C.c_int64, C.POINTER(CostParams), C.POINTER(C.c_double),
                                            C.POINTER(C.c_int)]),
    "ps_prefetch_gain": (C.c_double, [C.POINTER(HitStats), C.c_double, C.c_int, C.POINTER(CostParams)]),
    "ps_fit_cost_params": (C.c_int, [_P, _P, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                     C.POINTER(C.c_double)]),
    "ps_policy_parse": (C.c_int, [C.c_char_p, C.POINTER(Policy)]),
    "ps_policy_name": (C.c_int, [Policy, C.c_char_p, C.c_int]),
    "ps_layer_inputs_validate": (C.c_int, [C.POINTER(LayerInputs)]),
    "ps_presched_plan": (C.c_int, [C.POINTER(LayerInputs), Policy, C.POINTER(LayerPlan)]),
    "ps_simulate_pipeline": (C.c_int, [C.POINTER(PipelineInstance), Policy, PLAN_FN, _P, C.POINTER(CostParams),
                                       C.POINTER(SimOptions), C.POINTER(Timeline)]),
    "ps_verify_timeline": (C.c_int, [C.POINTER(TimelineEvent), C.c_int, C.POINTER(PipelineInstance),
                                     C.POINTER(CostParams), C.POINTER(C.c_int), C.c_char_p, C.c_int]),
    "ps_compute_metrics": (C.c_int, [C.POINTER(TimelineEvent), C.c_int, _P, _P, C.c_int, C.c_int64, C.c_int,
                                     C.POINTER(Metrics), _P, _P]),
    "ps_plan_residency": (C.c_int, [_P, C.c_int, C.c_int, C.c_uint64, C.c_uint64, _P, C.POINTER(C.c_int)]),
    "ps_route_topk": (C.c_int, [_P, _P, _P, _P, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                _P, _P, _P, _P, _P, _P]),
    "ps_route_permute": (C.c_int, [_P, _P, _P, _P, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                   _P, _P, _P, _P, _P, _P, _P, _P]),
    "ps_permute": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, _P, _P, _P, _P, C.c_int, _P, _P]),
    "ps_combine": (C.c_int, [_P, C.c_int, _P, _P, _P, C.c_int, C.c_int, C.c_int, C.c_int, _P, _P]),
    "ps_fnv1a64": (C.c_uint64, [_P, C.c_size_t]),
    "ps_trace_read": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "ps_trace_shape": (C.c_int, [_P, C.POINTER(ModelSpec), C.POINTER(C.c_int32), C.POINTER(C.c_uint64),
                                 C.POINTER(C.c_uint64)]),
    "ps_trace_arrays": (C.c_int, [_P, _P, _P, _P, _P]),
    "ps_trace_free": (C.c_int, [_P]),
    "ps_trace_write": (C.c_int, [C.c_char_p, C.POINTER(ModelSpec), C.c_int, C.c_uint64, _P, _P, _P, _P]),
    "ps_host_lane_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "ps_host_lane_destroy": (C.c_int, [_P]),
    "ps_host_lane_threads": (C.c_int, [_P]),
    "ps_host_lane_isa": (C.c_int, [_P]),
    "ps_host_lane_reads_z": (C.c_int, [_P]),
    "ps_host_lane_bind_caller": (C.c_int, [_P]),
    "ps_host_expert_ffn": (C.c_int, [_P, _P, C.c_int, C.c_int, _P, C.c_int, _P]),
    "ps_host_expert_ffn_batch": (C.c_int, [_P, C.c_int, _P, _P, _P, C.c_int, C.c_int, _P, _P]),
    "ps_host_expert_ffn_batch_tiled": (C.c_int, [_P, C.c_int, _P, _P, _P, C.c_int, C.c_int, _P, _P]),
    "ps_host_slab_tile": (C.c_int, [_P, C.c_int, C.c_int]),
    "ps_host_slab_untile": (C.c_int, [_P, C.c_int, C.c_int]),
    "ps_zslab_encode_tiled": (C.c_int, [_P, C.c_int, C.c_int, _P, C.c_uint64, C.POINTER(C.c_uint64), C.c_int]),
    "ps_host_expert_ffn_batch_z": (C.c_int, [_P, C.c_int, _P, _P, _P, C.c_int, C.c_int, _P, _P]),
    "ps_rows_from_host": (C.c_int, [_P, C.c_int64, _P, C.c_int, C.c_int64, _P]),
    "ps_rows_from_host_ranges": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, _P, C.c_int, C.c_int64, _P]),
    "ps_cast_bf16": (C.c_int, [_P, C.c_int64, _P, _P]),
    "ps_engine_decode_step_routed": (C.c_int, [_P, _P, _P, _P, C.c_int, _P]),
    "ps_zslab_bound": (C.c_uint64, [C.c_uint64]),
    "ps_zslab_encode": (C.c_int, [_P, C.c_uint64, _P, C.c_uint64, C.POINTER(C.c_uint64), C.c_int]),
    "ps_zslab_info": (C.c_int, [_P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "ps_zslab_decode": (C.c_int, [_P, _P, _P, _P]),
    "ps_export_timeline": (C.c_int, [_P, C.c_int, C.c_int64, C.c_char_p, C.c_int, C.POINTER(C.c_int)]),
    "ps_append_shared": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, _P, _P, _P, _P]),
    "ps_expert_ffn": (C.c_int, [C.POINTER(ExpertGroup), _P, _P, _P, C.c_int, _P, C.c_int, C.c_int, _P, _P,
                                C.c_int, C.c_int, _P]),
    "ps_expert_ffn_zslab": (C.c_int, [C.POINTER(ExpertGroup), _P, _P, _P, _P, C.c_int, _P, C.c_int, C.c_int, _P,
                                      _P, C.c_int, C.c_int, _P]),
    "ps_ffn_down_splits": (C.c_int, [C.c_int, C.c_int]),
    "ps_set_prefill_kernel": (C.c_int, [C.c_int]),
    "ps_expert_ffn_prefill": (C.c_int, [C.POINTER(ExpertGroup), _P, _P, _P, C.c_int, C.c_int, C.c_int, _P, _P,
                                        _P]),
    "ps_expert_ffn_prefill_dev": (C.c_int, [C.POINTER(ExpertGroup), _P, _P, C.c_int, C.c_int, C.c_int, _P, _P, _P]),
    "ps_init_expert_slab": (C.c_int, [_P, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int, _P]),
    "ps_init_expert_slab_host": (C.c_int, [_P, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int]),
    "ps_llapor_load": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(ModelSpec)]),
    "ps_llapor_random": (C.c_int, [C.POINTER(ModelSpec), C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64,
                                   C.POINTER(C.c_void_p)]),
    "ps_llapor_free": (C.c_int, [_P]),
    "ps_llapor_save": (C.c_int, [_P, C.c_char_p]),
    "ps_llapor_fine_tune": (C.c_int, [_P, C.c_int, C.c_int, _P, _P, C.c_int, _P, _P, C.c_int, C.c_int, C.c_double]),
    "ps_llapor_scratch_bytes": (C.c_size_t, [_P, C.c_int]),
    "ps_llapor_forward": (C.c_int, [_P, C.c_int, _P, _P, C.c_int, _P, C.c_int, C.c_int, _P, _P, _P, _P, _P]),
    "ps_ep_local_experts": (C.c_int, [C.c_int, C.c_int, C.c_int]),
    "ps_ep_remap_ids": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, _P, _P]),
    "ps_ep_recv_plan": (C.c_int, [_P, C.c_int, C.c_int, _P, _P, _P]),
    "ps_ep_pack_counts": (C.c_int, [_P, _P, C.c_int, C.c_int, _P, _P]),
    "ps_ep_unique_id": (C.c_int, [C.c_char_p, C.c_int]),
    "ps_ep_comm_create": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "ps_ep_comm_destroy": (C.c_int, [_P]),
    "ps_ep_loopback_create": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "ps_ep_comm_rank": (C.c_int, [_P]),
    "ps_ep_comm_world": (C.c_int, [_P]),
    "ps_ep_all_to_all": (C.c_int, [_P, _P, _P, _P, _P, _P]),
    "ps_gather_rows": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, _P, _P]),
    "ps_engine_create": (C.c_int, [C.POINTER(EngineConfig), C.POINTER(C.c_void_p)]),
    "ps_engine_destroy": (C.c_int, [_P]),
    "ps_engine_set_router": (C.c_int, [_P, _P]),
    "ps_engine_decode_step": (C.c_int, [_P, _P, _P, C.c_int, _P, _P]),
    "ps_engine_decode_step_host": (C.c_int, [_P, _P, _P, C.c_int, _P, _P]),
    "ps_cache_create": (C.c_int, [C.POINTER(CacheConfig), C.POINTER(C.c_void_p)]),
    "ps_cache_destroy": (C.c_int, [_P]),
    "ps_cache_prefetch": (C.c_int, [_P, C.c_int, C.c_int]),
    "ps_cache_ondemand": (C.c_int, [_P, C.c_int, C.c_int]),
    "ps_cache_acquire": (C.c_int, [_P, C.c_int, C.c_int, _P, C.POINTER(C.c_void_p)]),
    "ps_cache_release": (C.c_int, [_P, C.c_int, C.c_int, _P]),
    "ps_cache_cancel_prefetches": (C.c_int, [_P, C.POINTER(C.c_int)]),
    "ps_cache_sync": (C.c_int, [_P]),
    "ps_cache_get_stats": (C.c_int, [_P, C.POINTER(CacheStats)]),
    "ps_engine_step_begin": (C.c_int, [_P, C.c_int]),
    "ps_engine_set_lookahead": (C.c_int, [_P, C.c_int, C.c_int]),
    "ps_engine_last_routing": (C.c_int, [_P, _P, _P]),
    "ps_engine_layer_forward": (C.c_int, [_P, C.c_int, _P, _P, _P, _P, _P]),
    "ps_engine_step_end": (C.c_int, [_P]),
    "ps_engine_get_stats": (C.c_int, [_P, C.POINTER(EngineStats)]),
    "ps_engine_reset_stats": (C.c_int, [_P]),
    "ps_engine_last_timeline": (C.c_int, [_P, C.POINTER(Timeline), _P, _P]),
    "ps_engine_calibrate": (C.c_int, [_P, C.POINTER(CostParams)]),
    "ps_engine_set_cost": (C.c_int, [_P, C.POINTER(CostParams)]),
    "ps_engine_last_predictions": (C.c_int, [_P, _P]),
    "ps_verify_timeline_ex": (C.c_int, [C.POINTER(TimelineEvent), C.c_int, C.POINTER(PipelineInstance),
                                        C.POINTER(CostParams), C.c_int, C.POINTER(C.c_int), C.c_char_p, C.c_int]),
}

_lib = None


def load(path: os.PathLike | str | None = None) -> C.CDLL:
    """Load libprescope_b200.so; raises if it was not built (no fallback)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = pathlib.Path(path) if path else LIB_PATH
    if not p.exists():
        raise RuntimeError(f"{p} is missing: run __graft_entry__.build() (no CPU/Python fallback exists)")
    lib = C.CDLL(str(p), mode=C.RTLD_GLOBAL)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def check(status: int) -> None:
    if status != PS_OK:
        raise PsError(status, load().ps_last_error().decode(errors="replace"))


def declared_symbols(header: os.PathLike | str | None = None) -> list[str]:
    """Function names declared in include/ps_api.h."""
    import re
    h = pathlib.Path(header) if header else _HERE.parent / "include" / "ps_api.h"
    text = h.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    text = re.sub(r"typedef[^;]*;", "", text)  # function-pointer typedefs are not exports
    return sorted(set(re.findall(r"\b(ps_[a-z0-9_]+)\s*\(", text)))
