"""ctypes binding of the in-tree C-ABI library (include/disco_b200.h).

The product path has no fallback: if the library is missing or fails to load,
importing the package raises.  Build it with ``python -m
paper_2209_12769_b200.build`` (or ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FO_LIB_PATH") or os.path.join(HERE, "_build", "libdiscob200.so")

FO_OK, FO_CYCLE, FO_MISSING_COST, FO_NEGATIVE_DURATION, FO_DIM_MISMATCH = 0, 1, 2, 3, 4
FO_INVALID_ARG, FO_CUDA_ERROR, FO_UNSUPPORTED = 5, 6, 7
FO_PROVIDER_PROFILE, FO_PROVIDER_HW_ORACLE = 0, 1
FO_EST_INVALID, FO_EST_NONE, FO_EST_ANALYTIC, FO_EST_LINEAR, FO_EST_MESSAGE_PASSING = -2, -1, 0, 1, 2
FO_PREC_FP32, FO_PREC_FP64 = 0, 1

P = C.POINTER
vp = C.c_void_p


class GraphDesc(C.Structure):
    _fields_ = [("n_ops", C.c_int32), ("n_edges", C.c_int32), ("n_allreduces", C.c_int32),
                ("op_kind", P(C.c_int32)), ("op_out_bytes", P(C.c_int64)), ("op_profile_us", P(C.c_double)),
                ("op_compute_us", P(C.c_double)), ("edge_src", P(C.c_int32)), ("edge_dst", P(C.c_int32)),
                ("edge_bytes", P(C.c_int64)), ("ar_producer", P(C.c_int32)), ("ar_bytes", P(C.c_int64))]


class CostModel(C.Structure):
    _fields_ = [("provider", C.c_int32), ("variant", C.c_int32), ("comm_C", C.c_double), ("comm_D", C.c_double),
                ("launch_us", C.c_double), ("mem_us_per_byte", C.c_double), ("layers", C.c_int32),
                ("hidden", C.c_int32), ("feat_dim", C.c_int32), ("op_vocab_slot", P(C.c_int32)),
                ("params", P(C.c_double)), ("n_params", C.c_int64), ("norm_mean", P(C.c_double)),
                ("norm_std", P(C.c_double)), ("out_scale", C.c_double), ("hw_noise", C.c_double),
                ("hw_key_prefix", C.c_char_p), ("hw_key_prefix_len", C.c_int32), ("op_key_bytes", C.c_char_p),
                ("op_key_off", P(C.c_int64))]


class SearchCfg(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_int32), ("max_unchanged", C.c_int32),
                ("methods_mask", C.c_int32), ("precision", C.c_int32), ("n_threads", C.c_int32)]


class TraceRec(C.Structure):
    _fields_ = [("step", C.c_int32), ("method", C.c_int32), ("cost_us", C.c_double), ("best_cost_us", C.c_double),
                ("queue_len", C.c_int32), ("enqueued", C.c_int32)]


# (name, restype, argtypes) -- every symbol include/disco_b200.h declares
SIGNATURES = [
    ("fo_graph_create", C.c_int, [P(GraphDesc), C.c_int32, P(vp)]),
    ("fo_graph_destroy", C.c_int, [vp]),
    ("fo_graph_set_cost_model", C.c_int, [vp, P(CostModel)]),
    ("fo_batch_best", C.c_int, [vp, vp, C.c_int32, C.c_int64, vp, vp]),
    ("fo_pairs_best", C.c_int, [vp, C.c_int32, vp, vp]),
    ("fo_memo_clear", C.c_int, [vp, vp]),
    ("fo_predict_features", C.c_int, [vp, C.c_int32, vp, vp, vp, vp, C.c_int32, vp, vp, C.c_int32, vp]),
    ("fo_memo_enable", C.c_int, [vp, C.c_int32]),
    ("fo_score", C.c_int, [vp, vp, vp, vp, C.c_int32, C.c_int32, C.c_int32, vp, vp, vp]),
    ("fo_score_host", C.c_int, [vp, vp, vp, vp, C.c_int32, C.c_int32, C.c_int32, vp, vp]),
    ("fo_score_i16", C.c_int, [vp, vp, vp, vp, C.c_int32, C.c_int32, C.c_int32, vp, vp, vp]),
    ("fo_score_host_i16", C.c_int, [vp, vp, vp, vp, C.c_int32, C.c_int32, C.c_int32, vp, vp]),
    ("fo_simulate", C.c_int, [vp, vp, vp, vp, C.c_int32, C.c_int32, vp, vp, vp, vp, P(C.c_int32), vp, vp, vp,
                              P(C.c_int32), P(C.c_double), P(C.c_int32)]),
    ("fo_node_durations", C.c_int, [vp, vp, vp, vp, C.c_int32, C.c_int32, vp, P(C.c_int32), P(C.c_int32)]),
    ("fo_make_candidates", C.c_int, [vp, vp, vp, vp, vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, vp, vp, vp,
                                     P(C.c_int32)]),
    ("fo_random_apply", C.c_int, [vp, vp, vp, vp, C.c_int32, C.c_int32, vp, P(C.c_int32)]),
    ("fo_expand_all", C.c_int, [vp, vp, vp, vp, C.c_int32, vp, vp, vp, P(C.c_int32)]),
    ("fo_state_hash", C.c_int, [vp, vp, vp, vp, C.c_int32, vp]),
    ("fo_topo_order", C.c_int, [vp, vp, vp, vp, vp, P(C.c_int32)]),
    ("fo_greedy_postorder", C.c_int, [vp, vp, vp, vp, vp, vp, vp]),
    ("fo_rewrite_pairs", C.c_int, [vp, vp, vp, vp, C.c_int32, vp, C.c_int32, P(C.c_int32)]),
    ("fo_rewrite_apply", C.c_int, [vp, vp, vp, vp, C.c_int32, C.c_int32, C.c_int32, P(C.c_int32)]),
    ("fo_set_parent", C.c_int, [vp, vp, vp, vp]),
    ("fo_set_phase_stop", C.c_int, [vp, C.c_int32]),
    ("fo_set_delta_mode", C.c_int, [vp, C.c_int32]),
    ("fo_inc_stats", C.c_int, [vp, C.c_int32, vp]),
    ("fo_set_estimator_arith", C.c_int, [vp, C.c_int32]),
    ("fo_make_candidates_delta", C.c_int, [vp, vp, vp, vp, vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, vp, vp,
                                           C.c_int64]),
    ("fo_score_delta", C.c_int, [vp, vp, vp, C.c_int32, C.c_int32, vp, vp, vp]),
    ("fo_score_delta_host", C.c_int, [vp, vp, vp, C.c_int32, C.c_int32, vp, vp]),
    ("fo_score_delta_slot", C.c_int, [vp, C.c_int32, vp, vp, C.c_int32, C.c_int32, C.c_int32, vp, vp, vp]),
    ("fo_score_delta_submit", C.c_int, [vp, vp, vp, C.c_int32, C.c_int32, C.c_int32, vp, vp, P(C.c_int64)]),
    ("fo_score_wait", C.c_int, [vp, C.c_int64]),
    ("fo_threshold_ar", C.c_int, [vp, vp, vp, vp, C.c_int64, vp, C.c_int32, vp, vp, vp]),
    ("fo_search_create", C.c_int, [vp, P(SearchCfg), vp, C.c_int32, vp, vp, vp, P(vp)]),
    ("fo_search_round", C.c_int, [vp, P(C.c_int32), vp]),
    ("fo_search_start", C.c_int, [vp, vp]),
    ("fo_search_run", C.c_int, [vp, C.c_int64, P(C.c_int32)]),
    ("fo_search_run_cb", C.c_int, [vp, C.c_int64, vp, vp, P(C.c_int32)]),
    ("fo_xchg_unique_id", C.c_int, [vp]),
    ("fo_xchg_create", C.c_int, [vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, P(vp)]),
    ("fo_xchg_attach", C.c_int, [vp, vp, C.c_int64, C.c_int32]),
    ("fo_xchg_finish", C.c_int, [vp]),
    ("fo_xchg_history", C.c_int, [vp, vp, C.c_int64, P(C.c_int64)]),
    ("fo_xchg_destroy", C.c_int, [vp]),
    ("fo_search_result", C.c_int, [vp, C.c_int32, P(C.c_double), vp, vp, vp, vp, P(TraceRec), C.c_int64]),
    ("fo_search_timing", C.c_int, [vp, P(C.c_double), P(C.c_double), P(C.c_int64)]),
    ("fo_search_rounds", C.c_int, [vp, P(C.c_int64)]),
    ("fo_score_geometry", C.c_int, [vp, C.c_int32, C.c_int32, vp]),
    ("fo_search_destroy", C.c_int, [vp]),
    ("fo_last_error", C.c_char_p, []),
    ("fo_kernel_launches", C.c_int64, []),
]

_lib = None


def lib():
    """The loaded library; raises (never falls back) when it is unavailable."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -m paper_2209_12769_b200.build)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    msg = lib().fo_last_error()
    return msg.decode() if msg else ""


SUBMIT_SLOTS = 4  # fo_score_delta_submit: batches in flight (fo_graph::kSubmitSlots)

# fo_round_fn: int32 (void *ctx, int64 round, int32 active, const double *best, int32 R)
ROUND_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_int64, C.c_int32, C.POINTER(C.c_double), C.c_int32)


def ptr(a):
    """Raw address of a numpy array or torch tensor (plain pointer hand-off)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


def tptr(a, ct):
    return a.ctypes.data_as(P(ct))
