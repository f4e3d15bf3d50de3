"""ctypes binding of libdbsp_b200.so (the C ABI in include/dbsp_b200.h).

The library is loaded from the package directory only (built in-tree by
build.py).  There is no fallback: if the shared object is missing the import
of any compute entry point raises, loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libdbsp_b200.so"

u32, u64, i32, i64, f64, f32 = C.c_uint32, C.c_uint64, C.c_int32, C.c_int64, C.c_double, C.c_float
P = C.POINTER


class MaskSetT(C.Structure):
    _fields_ = [("heads", P(P(u64))), ("num_heads", u32), ("num_q_blocks", u32),
                ("num_kv_blocks", u32), ("block_size", u32)]


class StrategyT(C.Structure):
    _fields_ = [("ulysses", u32), ("ring", u32)]


class PlanT(C.Structure):
    _fields_ = [("head_assignment", P(u32)), ("q_assignment", P(u32)), ("kv_assignment", P(u32))]


class PlannerConfigT(C.Structure):
    _fields_ = [("reuse_threshold", f64), ("exchange_reward", f64)]


class PlanOutcomeT(C.Structure):
    _fields_ = [("head_replanned", i32), ("rho_pre", f64), ("rho_post", f64)]


class GeneratorSpecT(C.Structure):
    _fields_ = [("num_heads", u32), ("num_q_blocks", u32), ("num_kv_blocks", u32),
                ("block_size", u32), ("pattern", u32), ("min_density", f64),
                ("max_density", f64), ("skew", f64), ("seed", u64)]


class ExchangeT(C.Structure):
    _fields_ = [("q_blocks_moved", u64), ("kv_blocks_moved", u64), ("token_payload", u64)]


class ProfileT(C.Structure):
    _fields_ = [("num_all2all", u32), ("all2all_degrees", P(u32)), ("all2all_offsets", P(u32)),
                ("all2all_x", P(f64)), ("all2all_y", P(f64)),
                ("num_p2p", u32), ("p2p_degrees", P(u32)), ("p2p_offsets", P(u32)),
                ("p2p_x", P(f64)), ("p2p_y", P(f64)),
                ("dense_attn_seconds", f64), ("launch_seconds", f64), ("exchange_overlap", f64),
                ("replan_seconds", f64), ("bytes_per_token_per_head", f64)]


class LatencyT(C.Structure):
    _fields_ = [("all2all_s", f64), ("attn_compute_s", f64), ("ring_p2p_exposed_s", f64),
                ("imbalance_penalty_s", f64), ("exchange_s", f64), ("replan_s", f64),
                ("total_s", f64)]


class CallInputsT(C.Structure):
    _fields_ = [("heads", u32), ("q_blocks", u32), ("kv_blocks", u32), ("block_size", u32),
                ("strategy", StrategyT), ("density", f64), ("rho", f64),
                ("exchange", ExchangeT), ("charge_replan", i32)]


class ProfileSampleT(C.Structure):
    _fields_ = [("primitive", u32), ("degree", u32), ("x", f64), ("seconds", f64)]


class FitOptionsT(C.Structure):
    _fields_ = [("exchange_overlap", f64), ("replan_seconds", f64),
                ("bytes_per_token_per_head", f64)]


class ProfileStorageT(C.Structure):
    _fields_ = [("all2all_degrees", P(u32)), ("all2all_offsets", P(u32)), ("all2all_x", P(f64)),
                ("all2all_y", P(f64)), ("p2p_degrees", P(u32)), ("p2p_offsets", P(u32)),
                ("p2p_x", P(f64)), ("p2p_y", P(f64))]


class PredictionT(C.Structure):
    _fields_ = [("strategy", StrategyT), ("outcome", PlanOutcomeT), ("latency", LatencyT)]


class LocalViewT(C.Structure):
    _fields_ = [("num_heads", u32), ("head_ids", P(u32)), ("num_q_blocks", u32),
                ("q_block_ids", P(u32)), ("num_kv_blocks", u32), ("kv_block_ids", P(u32)),
                ("kv_tokens_global", u32)]


class AttnArgsT(C.Structure):
    _fields_ = [("q", C.c_void_p), ("k", C.c_void_p), ("v", C.c_void_p), ("o", C.c_void_p),
                ("lse", C.c_void_p), ("o_accum", C.c_void_p), ("lse_accum", C.c_void_p),
                ("q_tokens", u32), ("kv_tokens", u32), ("heads", u32), ("head_dim", u32),
                ("softmax_scale", f32), ("accumulate", u32), ("finalize", u32)]


class QkvArgsT(C.Structure):
    _fields_ = [("x", C.c_void_p), ("w", C.c_void_p), ("bias", C.c_void_p), ("out", C.c_void_p),
                ("tokens", u32), ("hidden", u32), ("heads", u32), ("head_dim", u32)]


class QkvScatterT(C.Structure):
    _fields_ = [("q_peers", C.c_void_p), ("k_peers", C.c_void_p), ("v_peers", C.c_void_p),
                ("block_map", C.c_void_p), ("head_map", C.c_void_p), ("heads_of", C.c_void_p), ("ring", u32)]


class OutScatterT(C.Structure):
    _fields_ = [("out_peers", C.c_void_p), ("q_block_map", C.c_void_p), ("head_map", C.c_void_p),
                ("out_heads", C.c_uint32)]


# name -> (restype, argtypes)
_SIGS = {
    "dbsp_last_error": (C.c_char_p, []),
    "dbsp_version": (C.c_char_p, []),
    "dbsp_mix_seed": (u64, [u64, u64, u64]),
    "dbsp_generate_mask_set": (C.c_int, [P(GeneratorSpecT), P(u64)]),
    "dbsp_perturb_mask_set": (C.c_int, [P(MaskSetT), f64, u64, P(u64)]),
    "dbsp_total_blocks": (C.c_int, [P(MaskSetT), P(u64)]),
    "dbsp_blocks_per_head": (C.c_int, [P(MaskSetT), P(u64)]),
    "dbsp_density": (C.c_int, [P(MaskSetT), P(f64)]),
    "dbsp_save_mask_set": (C.c_int, [P(MaskSetT), C.c_char_p]),
    "dbsp_load_mask_set_header": (C.c_int, [C.c_char_p, P(u32), P(u32), P(u32), P(u32)]),
    "dbsp_load_mask_set": (C.c_int, [C.c_char_p, P(u64)]),
    "dbsp_enumerate_strategies": (C.c_int, [u32, P(StrategyT), P(u32)]),
    "dbsp_validate_plan": (C.c_int, [P(MaskSetT), StrategyT, P(PlanT)]),
    "dbsp_default_plan": (C.c_int, [P(MaskSetT), StrategyT, P(PlanT)]),
    "dbsp_workload_table": (C.c_int, [P(MaskSetT), StrategyT, P(PlanT), P(u64), P(u32)]),
    "dbsp_imbalance_ratio": (C.c_int, [P(u64), u32, u32, P(f64)]),
    "dbsp_exchange_volume": (C.c_int, [P(MaskSetT), StrategyT, P(PlanT), P(ExchangeT)]),
    "dbsp_summed_grid": (C.c_int, [P(MaskSetT), P(u64)]),
    "dbsp_head_level_imbalance": (C.c_int, [P(u64), P(u32), u32, u32, P(f64)]),
    "dbsp_partition_heads": (C.c_int, [P(MaskSetT), u32, P(u32)]),
    "dbsp_partition_blocks": (C.c_int, [P(MaskSetT), u32, f64, P(u32), P(u32)]),
    "dbsp_biased_greedy": (C.c_int, [P(u64), u32, u32, f64, P(u32)]),
    "dbsp_plan_dual": (C.c_int, [P(MaskSetT), StrategyT, P(PlannerConfigT), P(PlanT), P(PlanT),
                                 P(PlanOutcomeT)]),
    "dbsp_brute_force_heads": (C.c_int, [P(MaskSetT), u32, P(u32)]),
    "dbsp_brute_force_blocks": (C.c_int, [P(u64), u32, u32, u32, P(u32), P(u32), P(f64)]),
    "dbsp_fit_profile": (C.c_int, [P(ProfileSampleT), u32, P(FitOptionsT), P(ProfileStorageT),
                                   P(ProfileT)]),
    "dbsp_pwl_eval": (C.c_int, [P(f64), P(f64), u32, f64, P(f64)]),
    "dbsp_predict_from_inputs": (C.c_int, [P(CallInputsT), P(ProfileT), P(LatencyT)]),
    "dbsp_predict_latency": (C.c_int, [P(MaskSetT), StrategyT, P(PlanT), P(ProfileT), i32,
                                       P(LatencyT)]),
    "dbsp_selector_create": (C.c_int, [u32, P(C.c_void_p)]),
    "dbsp_selector_destroy": (None, [C.c_void_p]),
    "dbsp_selector_stored": (C.c_int, [C.c_void_p, i64, P(i32), P(StrategyT), P(u32), P(PlanT)]),
    "dbsp_selector_store": (C.c_int, [C.c_void_p, i64, StrategyT, P(PlanT), P(u32)]),
    "dbsp_predict_all": (C.c_int, [P(MaskSetT), P(ProfileT), u32, P(PlannerConfigT),
                                   P(StrategyT), P(PlanT), u32, P(PredictionT), P(PlanT), P(u32)]),
    "dbsp_select": (C.c_int, [C.c_void_p, i64, P(MaskSetT), P(ProfileT), P(PlannerConfigT),
                              P(StrategyT), P(PlanT), P(PlanOutcomeT), P(LatencyT)]),
    "dbsp_select_two_phase": (C.c_int, [C.c_void_p, i64, P(MaskSetT), P(ProfileT), P(PlannerConfigT),
                                        P(StrategyT), P(PlanT), P(PlanOutcomeT), P(LatencyT)]),
    "dbsp_select_device": (C.c_int, [C.c_void_p, i64, C.c_void_p, u32, u32, u32, u32, P(ProfileT),
                                     P(PlannerConfigT), P(StrategyT), P(PlanT), P(PlanOutcomeT), P(LatencyT),
                                     C.c_void_p]),
    "dbsp_qkv_project": (C.c_int, [P(QkvArgsT), C.c_void_p, C.c_void_p]),
    "dbsp_nccl_unique_id": (C.c_int, [C.c_void_p, u32]),
    "dbsp_sp_context_create": (C.c_int, [u32, u32, C.c_void_p, P(C.c_void_p)]),
    "dbsp_sp_context_destroy": (None, [C.c_void_p]),
    "dbsp_sp_attention": (C.c_int, [C.c_void_p, P(MaskSetT), StrategyT, P(PlanT), C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p, u32, u32, C.c_void_p]),
    "dbsp_sp_set_timing": (C.c_int, [C.c_void_p, i32]),
    "dbsp_sp_period_ms": (C.c_int, [C.c_void_p, P(C.c_float), u32, P(u32)]),
    "dbsp_sp_synchronize": (C.c_int, [C.c_void_p, C.c_void_p, u32]),
    "dbsp_sp_attention_simulated": (C.c_int, [P(MaskSetT), StrategyT, P(PlanT), C.c_void_p, C.c_void_p,
                                              C.c_void_p, C.c_void_p, u32, u32, C.c_void_p]),
    "dbsp_schedule_create": (C.c_int, [P(C.c_void_p)]),
    "dbsp_schedule_destroy": (None, [C.c_void_p]),
    "dbsp_schedule_build": (C.c_int, [C.c_void_p, P(MaskSetT), P(LocalViewT), i32]),
    "dbsp_schedule_stats": (C.c_int, [C.c_void_p, P(u64), P(u64), P(u64)]),
    "dbsp_schedule_layout": (C.c_int, [C.c_void_p, P(u32)]),
    "dbsp_schedule_build_device": (C.c_int, [C.c_void_p, C.c_void_p, u32, u32, u32, P(LocalViewT), i32,
                                             C.c_void_p]),
    "dbsp_schedule_download": (C.c_int, [C.c_void_p, C.c_void_p, P(u32), u64]),
    "dbsp_schedule_upload": (C.c_int, [C.c_void_p, C.c_void_p]),
    "dbsp_schedule_upload_bytes": (C.c_int, [C.c_void_p, P(u64)]),
    "dbsp_attention_launch": (C.c_int, [C.c_void_p, P(AttnArgsT), C.c_void_p]),
    "dbsp_attention_launch_scatter": (C.c_int, [C.c_void_p, P(AttnArgsT), P(OutScatterT), C.c_void_p]),
    "dbsp_sparse_attention": (C.c_int, [P(MaskSetT), P(AttnArgsT), C.c_void_p]),
    "dbsp_launch_count": (u64, []),
    "dbsp_accum_init": (C.c_int, [C.c_void_p, C.c_void_p, u32, u32, u32, C.c_void_p]),
    "dbsp_copy_2d": (C.c_int, [C.c_void_p, u64, C.c_void_p, u64, u64, u64, i32, C.c_void_p]),
    "dbsp_mask_stats_device": (C.c_int, [C.c_void_p, u32, u32, u32, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def lib() -> C.CDLL:
    """Load the in-tree shared library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: run `python -m paper_2511_23113_b200.build` "
                "(or __graft_entry__.build()) first; there is no fallback path")
        handle = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib
