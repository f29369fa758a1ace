"""ctypes binding of include/dbag.h (the product C-ABI, libdbag.so).

Loads the in-tree libdbag.so and fails loudly when it is missing: there is no
CPU fallback anywhere in the product path."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DBAG_LIB") or os.path.join(HERE, "libdbag.so")

DPTR = C.POINTER(C.c_double)
I32P = C.POINTER(C.c_int32)
I64P = C.POINTER(C.c_int64)


class ProblemView(C.Structure):
    _fields_ = [("num_cameras", C.c_int32), ("num_points", C.c_int32), ("num_obs", C.c_int64),
                ("obs_cam", I32P), ("obs_pt", I32P), ("obs_uv", DPTR), ("cam_pose", DPTR),
                ("cam_f", DPTR), ("points", DPTR)]


class ParamView(C.Structure):
    _fields_ = [("num_cameras", C.c_int32), ("num_points", C.c_int32), ("cam_pose", DPTR),
                ("cam_f", DPTR), ("points", DPTR)]


class Options(C.Structure):
    _fields_ = [("rho_x", C.c_double), ("rho_y", C.c_double), ("max_iters", C.c_int32),
                ("primal_tol", C.c_double), ("stop_on_primal", C.c_int32), ("loss", C.c_int32),
                ("huber_delta", C.c_double), ("inner_max_iters", C.c_int32),
                ("grad_tol", C.c_double), ("step_tol", C.c_double), ("lbfgs_memory", C.c_int32),
                ("armijo_c", C.c_double), ("backtrack", C.c_double),
                ("max_line_search", C.c_int32), ("eps_depth", C.c_double),
                ("workers", C.c_int32), ("points_per_block", C.c_int32),
                ("cameras_per_block", C.c_int32), ("device", C.c_int32),
                ("numerics", C.c_int32)]


class IterationRecord(C.Structure):
    _fields_ = [("iter", C.c_int32), ("mean_reproj_err", C.c_double),
                ("max_primal_x", C.c_double), ("max_primal_y", C.c_double),
                ("camera_mse", C.c_double), ("point_mse", C.c_double), ("wall_ms", C.c_double),
                ("comm_floats", C.c_int64), ("max_dual_x", C.c_double),
                ("max_dual_y", C.c_double), ("sum_reproj_err", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class RoundStats(C.Structure):
    _fields_ = [("n_jacobian", C.c_uint64), ("n_trial", C.c_uint64), ("n_accept", C.c_uint64),
                ("n_direction", C.c_uint64), ("n_pairs_used", C.c_uint64),
                ("ms_local", C.c_double), ("ms_camera", C.c_double), ("ms_point", C.c_double),
                ("ms_final", C.c_double), ("n_model_flops", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class SceneInfo(C.Structure):
    _fields_ = [("config", C.c_int32), ("seed", C.c_uint64), ("scale", C.c_double),
                ("num_cameras", C.c_int32), ("num_points", C.c_int32), ("num_obs", C.c_int64),
                ("sigma_pixel", C.c_double), ("outlier_frac", C.c_double),
                ("sigma_init", C.c_double)]


class LmOptions(C.Structure):
    _fields_ = [("max_iters", C.c_int32), ("error_stop", C.c_double), ("lambda_init", C.c_double),
                ("lambda_max", C.c_double), ("lambda_up", C.c_double),
                ("lambda_down", C.c_double), ("use_schur", C.c_int32), ("eps_depth", C.c_double),
                ("device", C.c_int32)]


class ShardInfo(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("cam_begin", C.c_int32),
                ("cam_end", C.c_int32), ("local_obs", C.c_int64), ("local_points", C.c_int32),
                ("boundary_points", C.c_int32), ("boundary_copies", C.c_int64),
                ("send_count", C.c_int64), ("recv_count", C.c_int64), ("comm_floats", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


H = C.c_void_p
I8P = C.POINTER(C.c_int8)
U8P = C.POINTER(C.c_uint8)

# name -> (restype, argtypes); every symbol declared in include/dbag.h
SIGNATURES = {
    "dbag_abi_version": (C.c_int32, []),
    "dbag_last_error": (C.c_char_p, []),
    "dbag_last_error_info": (None, [I32P, I32P, DPTR, I64P]),
    "dbag_options_default": (None, [C.POINTER(Options)]),
    "dbag_create": (C.c_int, [C.POINTER(ProblemView), C.POINTER(ParamView), C.POINTER(Options),
                              C.POINTER(H)]),
    "dbag_destroy": (None, [H]),
    "dbag_local_update": (C.c_int, [H, C.c_int64]),
    "dbag_local_update_all": (C.c_int, [H]),
    "dbag_consensus_update": (C.c_int, [H]),
    "dbag_dual_update": (C.c_int, [H]),
    "dbag_set_reference": (C.c_int, [H, C.POINTER(ParamView)]),
    "dbag_iterate": (C.c_int, [H, C.c_int32, C.POINTER(IterationRecord)]),
    "dbag_run": (C.c_int, [H, C.c_int32, C.POINTER(IterationRecord), C.c_int64, I64P]),
    "dbag_get_consensus": (C.c_int, [H, DPTR, DPTR, DPTR]),
    "dbag_set_consensus": (C.c_int, [H, DPTR, DPTR]),
    "dbag_get_copies": (C.c_int, [H, DPTR, DPTR, DPTR, DPTR]),
    "dbag_set_copies": (C.c_int, [H, DPTR, DPTR, DPTR, DPTR]),
    "dbag_iteration": (C.c_int32, [H]),
    "dbag_num_blocks": (C.c_int64, [H]),
    "dbag_get_block_order": (C.c_int, [H, I32P]),
    "dbag_num_copies": (C.c_int, [H, I64P, I64P]),
    "dbag_lm_options_default": (None, [C.POINTER(LmOptions)]),
    "dbag_lm_create": (C.c_int, [C.POINTER(ProblemView), C.POINTER(ParamView),
                                 C.POINTER(LmOptions), C.POINTER(H)]),
    "dbag_lm_solve": (C.c_int, [H, C.c_int32, C.POINTER(ParamView), C.POINTER(IterationRecord),
                                C.c_int64, I64P, I32P, I32P]),
    "dbag_lm_compute_step": (C.c_int, [H, C.c_double, C.c_int32, DPTR, DPTR]),
    "dbag_lm_get_state": (C.c_int, [H, DPTR, DPTR]),
    "dbag_lm_destroy": (None, [H]),
    "dbag_rms_reprojection_error": (C.c_int, [H, DPTR]),
    "dbag_align_similarity": (C.c_int, [C.POINTER(ParamView), C.POINTER(ParamView), C.c_int32,
                                        DPTR, DPTR]),
    "dbag_get_blocks": (C.c_int, [H, I64P, I64P, I32P, I64P, I32P, I32P, I32P]),
    "dbag_partition": (C.c_int, [C.POINTER(ProblemView), C.c_int32, C.c_int32, C.POINTER(H),
                                 I64P, I64P, I64P, I64P]),
    "dbag_partition_fetch": (C.c_int, [H, I64P, I32P, I64P, I32P, I64P, I32P, I32P, I32P]),
    "dbag_partition_destroy": (None, [H]),
    "dbag_max_primal": (C.c_int, [H, DPTR, DPTR]),
    "dbag_dual_sums": (C.c_int, [H, DPTR, DPTR]),
    "dbag_block_objective": (C.c_int, [H, C.c_int64, DPTR]),
    "dbag_ops_per_iteration": (C.c_int64, [H]),
    "dbag_comm_floats": (C.c_int64, [H]),
    "dbag_mean_reprojection_error": (C.c_int, [H, DPTR]),
    "dbag_total_squared_error": (C.c_int, [H, DPTR]),
    "dbag_enqueue_round": (C.c_int, [H]),
    "dbag_reset": (C.c_int, [H]),
    "dbag_stream": (C.c_void_p, [H]),
    "dbag_synchronize": (C.c_int, [H]),
    "dbag_set_profiling": (C.c_int, [H, C.c_int32]),
    "dbag_get_round_stats": (C.c_int, [H, C.POINTER(RoundStats)]),
    "dbag_reset_stats": (C.c_int, [H]),
    "dbag_measure_fp64_peak": (C.c_int, [C.c_int32, DPTR]),
    "dbag_selftest_division": (C.c_int, [C.c_int32, C.c_int64, C.c_uint64, I64P]),
    "dbag_partition_cameras": (C.c_int, [C.c_int32, I64P, C.c_int32, I32P]),
    "dbag_shard_plan_create": (C.c_int, [C.POINTER(ProblemView), C.c_int32, C.c_int32,
                                         C.POINTER(H), C.POINTER(ShardInfo)]),
    "dbag_shard_plan_get_info": (None, [H, C.POINTER(ShardInfo)]),
    "dbag_shard_plan_arrays": (C.c_int, [H, I32P, I64P, I32P, I32P, I8P, I64P, I64P, I64P]),
    "dbag_shard_plan_exchange": (C.c_int, [H, I64P, I64P]),
    "dbag_shard_plan_destroy": (None, [H]),
    "dbag_create_sharded": (C.c_int, [C.POINTER(ProblemView), C.POINTER(ParamView),
                                      C.POINTER(Options), C.c_int32, C.c_int32, C.POINTER(H)]),
    "dbag_nccl_unique_id": (C.c_int, [U8P]),
    "dbag_attach_nccl": (C.c_int, [H, U8P]),
    "dbag_round_phase": (C.c_int, [H, C.c_int32, C.POINTER(IterationRecord)]),
    "dbag_exchange_copy": (C.c_int, [H, H, C.c_int32]),
    "dbag_parse_problem_text": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(H), I32P, I32P, I64P]),
    "dbag_bal_fetch": (C.c_int, [H, I32P, I32P, DPTR, DPTR, DPTR, DPTR]),
    "dbag_bal_destroy": (None, [H]),
    "dbag_serialize_problem_text": (C.c_int, [C.POINTER(ProblemView), C.POINTER(ParamView),
                                              C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "dbag_metrics_csv": (C.c_int, [C.POINTER(IterationRecord), C.c_int64, C.c_char_p, C.c_size_t,
                                   C.POINTER(C.c_size_t)]),
    "dbag_io_last_error": (C.c_char_p, [I32P]),
    "dbag_scene_generate": (C.c_int, [C.c_int32, C.c_uint64, C.c_double, C.POINTER(H),
                                      C.POINTER(SceneInfo)]),
    "dbag_scene_fetch": (C.c_int, [H, I32P, I32P, DPTR, DPTR, DPTR, DPTR, DPTR, DPTR]),
    "dbag_scene_destroy": (None, [H]),
}

_lib = None


def load(build_if_missing=True):
    """Load libdbag.so (building it in-tree when absent and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if not build_if_missing:
            raise ImportError(f"libdbag.so missing at {LIB_PATH}; run __graft_entry__.build()")
        from . import build as _b
        _b.build()
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is None and os.environ.get("DBAG_LIB"):
            continue  # an older A/B build (tools/build_variants.py) may lack newer entry points
        if fn is None:
            raise ImportError(f"{LIB_PATH} does not export {name}")
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
