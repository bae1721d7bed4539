"""ctypes binding of the C-ABI in include/semwarm_b200.h (libsemwarm_b200.so, built in-tree).

There is no fallback: if the shared library is missing or fails to load, every entry point
raises. The structures below mirror the header field-for-field.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
# SW_LIB_PATH: load another in-tree build of the same library (A/B timing of two builds)
LIB_PATH = os.environ.get("SW_LIB_PATH") or os.path.join(PKG, "libsemwarm_b200.so")

SW_OK = 0
SW_EINVAL = -1
SW_ERUNTIME = -2
SW_ECUDA = -3
SW_ENOMEM = -4
SW_WARN_UNKNOWN_ID = 1

SW_FLAG_EXACT_ONLY = 0x1
SW_FLAG_TC_ALWAYS = 0x2
SW_FLAG_GROW = 0x4

SW_GROUP_TRANSPORT_AUTO = 0
SW_GROUP_TRANSPORT_NCCL = 1
SW_GROUP_TRANSPORT_COPY = 2

SW_CHOICE_AMBIGUOUS_DRAW = 0x1
SW_CHOICE_NONFINITE_PHI = 0x2
SW_CHOICE_INCOMPLETE = 0x4
SW_CHOICE_AMBIGUOUS_ARM = 0x8

POLICY = {"exploit": 0, "explore": 1, "rule": 2, "fixed": 3}
HIT_RECORD_BYTES = 128


class SwConfig(C.Structure):
    _fields_ = [("dim", C.c_int32), ("rows_per_entry", C.c_int32), ("max_entries", C.c_int64),
                ("latent_c", C.c_int32), ("latent_t_max", C.c_int32), ("latent_f", C.c_int32),
                ("max_batch", C.c_int32), ("latent_slots", C.c_int64), ("latent_fps", C.c_double),
                ("flags", C.c_uint32), ("reserved", C.c_int32)]


class SwSelectorConfig(C.Structure):
    _fields_ = [("top_k", C.c_int32), ("reserved", C.c_int32), ("temperature", C.c_double),
                ("quality_threshold", C.c_double)]


class SwPolicy(C.Structure):
    _fields_ = [("kind", C.c_int32), ("fixed_arm", C.c_int32),
                ("rule_similarity_threshold", C.c_double), ("rule_skip_fraction", C.c_double)]


class SwcmConfig(C.Structure):
    _fields_ = [("capacity", C.c_uint64), ("decay_per_hour", C.c_double),
                ("grace_hours", C.c_double), ("quality_floor", C.c_double),
                ("pyramid_delta", C.c_double), ("embedding_seed", C.c_uint64),
                ("refine_regenerations", C.c_int32), ("refine_attempt_cap", C.c_int32),
                ("refine_window", C.c_int32), ("reserved", C.c_int32),
                ("refine_skip_threshold", C.c_double), ("latent_capacity", C.c_int64)]


class SwrWorkload(C.Structure):
    _fields_ = [("n_prompts", C.c_int64), ("cluster_count", C.c_int32), ("dim", C.c_int32),
                ("near_duplicate_rate", C.c_double), ("cluster_perturbation", C.c_double),
                ("duplicate_perturbation", C.c_double), ("duration_lo_s", C.c_double),
                ("duration_hi_s", C.c_double), ("arrival_rate_hz", C.c_double),
                ("total_steps", C.c_int32), ("reserved", C.c_int32)]


class SwrConfig(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("selector", SwSelectorConfig), ("policy", SwPolicy),
                ("q_max", C.c_double), ("penalty_slope", C.c_double), ("noise_scale", C.c_double),
                ("skip_headroom", C.c_double), ("step_time_s_per_10s", C.c_double),
                ("alpha", C.c_double), ("latent_rate", C.c_int32),
                ("default_total_steps", C.c_int32), ("refinement_enabled", C.c_int32),
                ("batch", C.c_int32)]


class SwrStats(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("total_s", "lookup_s", "mutation_s", "maintenance_s")] + \
               [(n, C.c_int64) for n in ("batches", "lookups", "admits", "evictions",
                                          "refinements", "reuses")] + \
               [(n, C.c_double) for n in ("total_nfe_s", "baseline_nfe_s", "speedup",
                                           "mean_quality", "mean_reward", "hit_rate",
                                           "mean_latency_s", "median_latency_s", "p95_latency_s")]


OUTCOME_DTYPE = np.dtype([("request_id", "<u8"), ("cache_hit", "<i4"), ("arm_index", "<i4"),
                          ("steps_skipped", "<i4"), ("fallback", "<i4"), ("entry_id", "<u8"),
                          ("admitted_entry_id", "<u8"), ("quality", "<f8"), ("nfe_cost_s", "<f8"),
                          ("sim_latency_s", "<f8"), ("skip_fraction", "<f8"),
                          ("reference_similarity", "<f8")])
assert OUTCOME_DTYPE.itemsize == 80


REGEN_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int32, C.c_double, C.c_uint64,
                       C.POINTER(C.c_float), C.POINTER(C.c_double), C.POINTER(C.c_float),
                       C.POINTER(C.c_int32))


# numpy mirrors of the array-of-struct types
SEGMENT_DTYPE = np.dtype([("level", "<i4"), ("reserved", "<i4"), ("start_s", "<f8"),
                          ("length_s", "<f8")])
HIT_DTYPE = np.dtype([("entry_id", "<u8"), ("level", "<i4"), ("reserved", "<i4"),
                      ("start_s", "<f8"), ("length_s", "<f8"), ("similarity", "<f8")])
REQUEST_DTYPE = np.dtype([("id", "<u8"), ("duration_s", "<f8"), ("total_steps", "<i4"),
                          ("reserved", "<i4")])
CHOICE_DTYPE = np.dtype([("hit", "<i4"), ("arm", "<i4"), ("steps_skipped", "<i4"),
                         ("n_hits", "<i4"), ("entry_id", "<u8"), ("level", "<i4"),
                         ("row", "<i4"), ("start_s", "<f8"), ("length_s", "<f8"),
                         ("similarity", "<f8"), ("skip_fraction", "<f8"), ("pick", "<i4"),
                         ("flags", "<u4"), ("t_out", "<i4"), ("owner", "<i4"), ("slot", "<i8")])
assert SEGMENT_DTYPE.itemsize == 24 and HIT_DTYPE.itemsize == 40
assert REQUEST_DTYPE.itemsize == 24 and CHOICE_DTYPE.itemsize == 88

_lib = None


class SemwarmError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def lib() -> C.CDLL:
    """Load libsemwarm_b200.so (raises if it was not built — there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} not found: the CUDA extension is not built (run __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, u64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
    sig = {
        "sw_version": ([], C.c_int),
        "sw_last_error": ([], C.c_char_p),
        "sw_ctx_create": ([C.POINTER(SwConfig), C.c_int, C.POINTER(vp)], C.c_int),
        "sw_ctx_destroy": ([vp], C.c_int),
        "sw_set_negative": ([vp, vp], C.c_int),
        "sw_set_gater": ([vp, vp, vp, i32, f64], C.c_int),
        "sw_set_schedule": ([vp, vp, i32], C.c_int),
        "sw_arena_insert": ([vp, u64, i32, vp, vp, vp, i32], C.c_int),
        "sw_arena_insert_batch": ([vp, i64, vp, vp, vp, vp, vp, vp, vp, i32], C.c_int),
        "sw_arena_remove": ([vp, u64], C.c_int),
        "sw_arena_replace": ([vp, u64, i32, vp, vp, vp, i32], C.c_int),
        "sw_arena_entry_count": ([vp], i64),
        "sw_arena_contains": ([vp, u64], C.c_int),
        "sw_arena_fill_synthetic": ([vp, i64, u64, u64, f64], C.c_int),
        "sw_arena_read_rows": ([vp, u64, vp, i32], C.c_int),
        "sw_search": ([vp, vp, i32, i32, vp, vp, vp], C.c_int),
        "sw_search_host": ([vp, vp, i32, i32, vp, vp], C.c_int),
        "sw_plan": ([vp, vp, vp, i32, u64, C.POINTER(SwSelectorConfig), C.POINTER(SwPolicy),
                     vp, vp], C.c_int),
        "sw_align_noise": ([vp, vp, vp, i32, vp, u64, vp, i32, vp], C.c_int),
        "sw_warmstart": ([vp, vp, vp, i32, u64, C.POINTER(SwSelectorConfig),
                          C.POINTER(SwPolicy), vp, u64, vp, vp, i32, vp], C.c_int),
        "sw_warmstart_host": ([vp, vp, vp, i32, u64, C.POINTER(SwSelectorConfig),
                               C.POINTER(SwPolicy), u64, vp, vp, i32, vp], C.c_int),
        "sw_warmstart_async": ([vp, vp, vp, i32, u64, C.POINTER(SwSelectorConfig),
                                C.POINTER(SwPolicy), vp, u64, vp, vp, i32, vp], C.c_int),
        "sw_join": ([vp, vp], C.c_int),
        "sw_local_topk_async": ([vp, vp, i32, i32, i32, vp, vp, vp], C.c_int),
        "sw_async_stream": ([vp, C.POINTER(vp)], C.c_int),
        "sw_warmstart_host_submit": ([vp, vp, vp, i32, u64, C.POINTER(SwSelectorConfig),
                                      C.POINTER(SwPolicy), u64, vp, vp, i32, vp,
                                      C.POINTER(C.c_int64)], C.c_int),
        "sw_warmstart_host_wait": ([vp, C.c_int64], C.c_int),
        "sw_local_topk": ([vp, vp, i32, i32, i32, vp, vp, vp], C.c_int),
        "sw_merge_select": ([vp, vp, vp, i32, vp, vp, i32, i32, u64,
                             C.POINTER(SwSelectorConfig), C.POINTER(SwPolicy), vp, vp], C.c_int),
        "sw_align_noise_owned": ([vp, vp, vp, i32, i32, vp, u64, vp, i32, vp], C.c_int),
        "sw_ivf_config": ([vp, vp, vp, vp, vp, vp], C.c_int),
        "sw_gater_load_swmb": ([vp, C.c_char_p, f64], C.c_int),
        "sw_gater_save_swmb": ([vp, C.c_char_p], C.c_int),
        "swcm_save_snapshot": ([vp, C.c_char_p], C.c_int),
        "swcm_load_snapshot": ([vp, C.c_char_p], C.c_int),
        "sw_group_create": ([C.POINTER(SwConfig), i32, vp, i32, C.POINTER(vp)], C.c_int),
        "sw_group_destroy": ([vp], C.c_int),
        "sw_group_info": ([vp, vp, vp], C.c_int),
        "sw_group_shard": ([vp, i32, C.POINTER(vp)], C.c_int),
        "sw_group_owner": ([vp, u64], i32),
        "sw_group_insert": ([vp, u64, i32, vp, vp, vp, i32], C.c_int),
        "sw_group_remove": ([vp, u64], C.c_int),
        "sw_group_set_negative": ([vp, vp], C.c_int),
        "sw_group_set_gater": ([vp, vp, vp, i32, f64], C.c_int),
        "sw_group_warmstart_host": ([vp, vp, vp, i32, u64, C.POINTER(SwSelectorConfig),
                                     C.POINTER(SwPolicy), u64, vp, vp, i32], C.c_int),
        "sw_group_shard_choices": ([vp, i32, i32, vp], C.c_int),
        "sw_score_select_host": ([vp, i32, vp, vp, vp, f64, C.POINTER(SwSelectorConfig), u64,
                                  vp, vp], C.c_int),
        "sw_gater_host": ([vp, vp, vp, vp, i32, i32, vp, vp], C.c_int),
        "sw_last_launch_info": ([vp, vp, vp, vp], C.c_int),
        "sw_profile_enable": ([vp, i32], C.c_int),
        "sw_debug_query_stats": ([vp, i32, vp], C.c_int),
        "swcm_create": ([vp, i32, C.POINTER(SwcmConfig), C.POINTER(vp)], C.c_int),
        "swcm_destroy": ([vp], C.c_int),
        "swcm_admit": ([vp, vp, f64, vp, f64, f64, vp, i32, C.POINTER(u64)], C.c_int),
        "swcm_last_evicted": ([vp, vp, i32], C.c_int),
        "swcm_record_reuse": ([vp, u64, i32, f64, f64, f64], C.c_int),
        "swcm_evict_if_full": ([vp, f64, vp, i32], C.c_int),
        "swcm_refinement_candidates": ([vp, vp, i32], C.c_int),
        "swcm_refine": ([vp, u64, u64, REGEN_FN, vp, C.POINTER(i32)], C.c_int),
        "swcm_importance": ([vp, u64, f64, C.POINTER(f64)], C.c_int),
        "swcm_size": ([vp], C.c_int),
        "swcm_ids": ([vp, vp, i32], C.c_int),
        "swcm_check_consistent": ([vp], C.c_int),
        "sw_profile_reset": ([vp], C.c_int),
        "sw_ivf_configure": ([vp, i32, i32, u64, u64], C.c_int),
        "sw_ivf_set_nprobe": ([vp, i32], C.c_int),
        "sw_ivf_rebuild": ([vp], C.c_int),
        "sw_ivf_info": ([vp, C.POINTER(i32), C.POINTER(u64), C.POINTER(u64)], C.c_int),
        "sw_ivf_centroids": ([vp, vp, i32], C.c_int),
        "sw_ivf_set_centroids": ([vp, vp, i32], C.c_int),
        "sw_ivf_entry_lists": ([vp, u64, vp, i32], C.c_int),
        "sw_swix_load": ([vp, C.c_char_p], C.c_int),
        "sw_ctx_info": ([vp, vp, vp, vp, vp, vp, vp], C.c_int),
        "sw_set_align_mode": ([vp, i32, i32, i32], C.c_int),
        "swb_create": ([vp, i32, i32, u64, C.POINTER(SwSelectorConfig), C.POINTER(SwPolicy), u64,
                        i32, i32, C.POINTER(vp)], C.c_int),
        "swb_destroy": ([vp], C.c_int),
        "swb_load_test": ([vp, vp, vp, i32, i32, i32, u64, vp, vp, vp, vp], C.c_int),
        "swb_submit": ([vp, vp, vp, vp, vp], C.c_int),
        "swb_stats": ([vp, C.POINTER(i64), C.POINTER(i64)], C.c_int),
        "sw_time_stretch": ([vp, vp, vp, i32, i32, vp, i32, i32, vp, i64, vp, vp, vp, vp],
                            C.c_int),
        "sw_swix_save": ([vp, C.c_char_p], C.c_int),
        "sw_swem_read": ([C.c_char_p, vp, i64, C.POINTER(i32), C.POINTER(i32)], i64),
        "sw_profile_read": ([vp, i32, C.POINTER(C.c_double), C.POINTER(C.c_int64)], C.c_int),
        "sw_overflow_stats": ([vp, C.POINTER(C.c_int64)], C.c_int),
        "sw_arena_capacity": ([vp], C.c_int64),
        "sw_arena_reserve": ([vp, i64], C.c_int),
        "sw_arena_row_count": ([vp], C.c_int64),
        "sw_arena_export": ([vp, i64, i64, vp, vp, vp, vp], C.c_int64),
        "sw_index_check_consistent": ([vp], C.c_int),
        "sw_ivf_set_rebuild_interval": ([vp, u64], C.c_int),
        "sw_ivf_build": ([vp, i64, vp, vp, vp, vp], C.c_int),
        "sw_search_host_ex": ([vp, vp, i32, i32, i32, vp, vp], C.c_int),
        "sw_score_candidates_host": ([vp, i32, i32, vp, vp, vp, f64, vp, vp], C.c_int),
        "sw_select_host": ([vp, i32, vp, vp, f64, f64, f64, vp, vp], C.c_int),
        "sw_choice_rows": ([vp, vp, i32, vp, vp], C.c_int),
        "sw_negative_embedding": ([i32, vp], C.c_int),
        "swr_synth_workload": ([C.POINTER(SwrWorkload), u64, vp, vp, vp, vp], C.c_int),
        "swr_replay": ([vp, vp, C.POINTER(SwrConfig), i64, vp, vp, vp, vp, vp,
                        C.POINTER(SwrStats)], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


EXPORTED = [
    "sw_version", "sw_last_error", "sw_ctx_create", "sw_ctx_destroy", "sw_set_negative",
    "sw_set_gater", "sw_set_schedule", "sw_arena_insert", "sw_arena_insert_batch",
    "sw_arena_remove", "sw_arena_replace", "sw_arena_entry_count", "sw_arena_contains",
    "sw_arena_fill_synthetic", "sw_arena_read_rows", "sw_search", "sw_search_host", "sw_plan",
    "sw_align_noise", "sw_warmstart", "sw_warmstart_host",
    "sw_warmstart_host_submit", "sw_warmstart_host_wait", "sw_warmstart_async", "sw_join",
    "sw_local_topk_async", "sw_async_stream",
    "sw_ivf_config", "sw_gater_load_swmb", "sw_gater_save_swmb", "swcm_save_snapshot",
    "swcm_load_snapshot",
    "sw_local_topk", "sw_merge_select", "sw_group_create", "sw_group_destroy", "sw_group_info",
    "sw_group_shard", "sw_group_owner", "sw_group_insert", "sw_group_remove",
    "sw_group_set_negative", "sw_group_set_gater", "sw_group_warmstart_host",
    "sw_group_shard_choices",
    "sw_align_noise_owned", "sw_score_select_host", "sw_gater_host", "sw_last_launch_info",
    "sw_profile_enable", "sw_profile_reset", "sw_profile_read", "sw_debug_query_stats",
    "sw_overflow_stats", "sw_arena_capacity", "sw_arena_reserve", "sw_arena_row_count",
    "sw_arena_export", "sw_index_check_consistent", "sw_ivf_set_rebuild_interval", "sw_ivf_build",
    "sw_search_host_ex", "sw_score_candidates_host", "sw_select_host", "sw_choice_rows",
    "sw_negative_embedding", "swr_synth_workload", "swr_replay",
    "swcm_create", "swcm_destroy", "swcm_admit", "swcm_last_evicted", "swcm_record_reuse",
    "swcm_evict_if_full", "swcm_refinement_candidates", "swcm_refine", "swcm_importance",
    "swcm_size", "swcm_ids", "swcm_check_consistent", "sw_ivf_configure", "sw_ivf_set_nprobe",
    "sw_ivf_rebuild", "sw_ivf_info", "sw_ivf_centroids", "sw_ivf_set_centroids",
    "sw_ivf_entry_lists", "sw_swix_load", "sw_swix_save", "sw_swem_read", "sw_time_stretch",
    "sw_ctx_info", "sw_set_align_mode", "swb_create", "swb_destroy", "swb_submit", "swb_stats",
    "swb_load_test",
]
STAGES = ["prep", "score_tc", "finish", "select", "align", "merge", "align_geom"]


def check(rc: int, what: str = "") -> int:
    if rc < 0:
        msg = lib().sw_last_error().decode(errors="replace")
        if rc == SW_EINVAL:
            raise ValueError(f"{what}: {msg}")
        raise SemwarmError(rc, f"{what}: {msg}")
    return rc


def ptr(a) -> int:
    """Raw pointer of a numpy array or a torch tensor (host or device)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return a.ctypes.data
    return a.data_ptr()  # torch.Tensor
