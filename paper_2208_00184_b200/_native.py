"""ctypes signatures of the context / resident-pipeline / synthesis entry points of
libdagplace_b200.so (include/dagplace_b200.h)."""
from __future__ import annotations

import ctypes as C

from ._abi import CommC, DevicesC, GraphC, PipelineCfgC

I64P = C.POINTER(C.c_int64)
I32P = C.POINTER(C.c_int32)

# every symbol the header declares (checked by tests/test_abi_exports.py)
HEADER_SYMBOLS = [
    "dp_last_error_message", "dp_last_error_code", "dp_ctx_create", "dp_ctx_destroy",
    "dp_ctx_set_stream", "dp_ctx_synchronize", "dp_ctx_launch_count", "dp_ctx_enable_stage_timing",
    "dp_ctx_stage_count", "dp_ctx_stage_name", "dp_ctx_stage_ms", "dp_ctx_stage_bytes", "dp_ctx_peel_stats",
    "dp_comm_time", "dp_ccr", "dp_validate", "dp_violation_list_free", "dp_require_valid",
    "dp_graph_index", "dp_compute_levels", "dp_topo_order", "dp_is_valid_topo_order",
    "dp_merge_is_safe", "dp_optimal_breakpoints", "dp_cluster_map_free", "dp_build_coarse_graph",
    "dp_graph_out_free", "dp_contract_colocation_groups", "dp_contraction_free", "dp_fuse",
    "dp_fusion_result_free", "dp_order_place", "dp_adjusting_placement", "dp_expand_placement",
    "dp_placement_result_free", "dp_simulate", "dp_sim_report_free", "dp_simulate_candidates",
    "dp_brute_force_optimal", "dp_pipeline", "dp_pipeline_batch", "dp_pipeline_result_free",
    "dp_resident_create", "dp_resident_generate", "dp_resident_generate_batch", "dp_resident_fetch", "dp_resident_destroy", "dp_gen_layered",
    "dp_gen_candidates", "dp_gen_gnmt", "dp_gen_bert",
    "dp_graph_from_json", "dp_devices_from_json",
    "dp_fit_node_models", "dp_node_models_free", "dp_estimate_graph", "dp_fit_comm_model",
    "dp_deviation_report", "dp_deviation_free",
]


def declare(lib: C.CDLL) -> None:
    lib.dp_last_error_message.restype = C.c_char_p
    lib.dp_last_error_code.restype = C.c_int32
    lib.dp_ctx_create.restype = C.c_int
    lib.dp_ctx_create.argtypes = [C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]
    lib.dp_ctx_destroy.restype = None
    lib.dp_ctx_destroy.argtypes = [C.c_void_p]
    lib.dp_ctx_set_stream.argtypes = [C.c_void_p, C.c_void_p]
    lib.dp_ctx_synchronize.argtypes = [C.c_void_p]
    lib.dp_ctx_launch_count.restype = C.c_int64
    lib.dp_ctx_launch_count.argtypes = [C.c_void_p]
    lib.dp_ctx_enable_stage_timing.argtypes = [C.c_void_p, C.c_int32]
    lib.dp_ctx_stage_count.restype = C.c_int32
    lib.dp_ctx_stage_count.argtypes = [C.c_void_p]
    lib.dp_ctx_stage_name.restype = C.c_char_p
    lib.dp_ctx_stage_name.argtypes = [C.c_void_p, C.c_int32]
    lib.dp_ctx_stage_ms.restype = C.c_double
    lib.dp_ctx_stage_ms.argtypes = [C.c_void_p, C.c_int32]
    lib.dp_ctx_stage_bytes.restype = C.c_double
    lib.dp_ctx_peel_stats.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
    lib.dp_ctx_stage_bytes.argtypes = [C.c_void_p, C.c_int32]
    lib.dp_resident_create.restype = C.c_int
    lib.dp_resident_create.argtypes = [C.c_void_p, C.POINTER(GraphC), C.POINTER(DevicesC), CommC,
                                       C.POINTER(PipelineCfgC), C.POINTER(C.c_void_p)]
    lib.dp_resident_generate.restype = C.c_int
    lib.dp_resident_generate.argtypes = [C.c_void_p]
    lib.dp_resident_generate_batch.restype = C.c_int
    lib.dp_resident_generate_batch.argtypes = [C.POINTER(C.c_void_p), C.c_int32]
    lib.dp_resident_fetch.restype = C.c_int
    lib.dp_resident_fetch.argtypes = [C.c_void_p, I32P, I32P, I64P, I64P]
    lib.dp_resident_destroy.restype = None
    lib.dp_resident_destroy.argtypes = [C.c_void_p]
    lib.dp_gen_layered.restype = C.c_int
    lib.dp_gen_layered.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_uint64,
                                   I64P, I64P, I64P, I64P, I64P, I64P, I64P]
    _declare_gen(lib)


def _declare_gen(lib):
    lib.dp_gen_gnmt.restype = C.c_int
    lib.dp_gen_gnmt.argtypes = [C.c_int64, C.c_int64, C.c_uint64] + [I64P] * 7
    lib.dp_gen_bert.restype = C.c_int
    lib.dp_gen_bert.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_uint64] + [I64P] * 7
    lib.dp_gen_candidates.restype = C.c_int
    lib.dp_gen_candidates.argtypes = [C.POINTER(C.c_uint8), C.c_int64, C.c_int32, C.c_int64, C.c_int64,
                                      C.POINTER(C.c_uint8)]


def stage_times(lib: C.CDLL, ctx) -> list:
    out = []
    for i in range(lib.dp_ctx_stage_count(ctx)):
        out.append((lib.dp_ctx_stage_name(ctx, i).decode(), lib.dp_ctx_stage_ms(ctx, i),
                    lib.dp_ctx_stage_bytes(ctx, i)))
    return out
