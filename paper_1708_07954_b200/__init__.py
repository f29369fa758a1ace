"""B200-native D-ADMM bundle-adjustment core (arXiv 1708.07954, data-parallel
hot path): CUDA kernels for sm_100a behind the C-ABI in include/dbag.h, with a
host mirror of the reference AdmmSolver API (admm.py)."""
from .admm import (AdmmOptions, AdmmSolver, AdmmState, DepthBelowGuard, DeviceError,  # noqa
                   DuplicateObservation, Error, IndexOutOfRange, InnerOptions, LossKind,
                   ParamState, Problem, Scene, SingularSystem, SizeMismatch, Unsupported,
                   ValidationError, generate_config_scene, run_admm, ParseError,
                   parse_problem_text, serialize_problem_text, metrics_csv,
                   LocalBlock, partition, communication_cost, align_similarity,
                   LmOptions, LmResult, solve_lm, lm_compute_step)
from ._capi import load as load_library  # noqa: F401

__all__ = ["AdmmOptions", "AdmmSolver", "AdmmState", "ParamState", "Problem", "LossKind",
           "InnerOptions", "run_admm", "generate_config_scene", "load_library", "LocalBlock",
           "partition", "communication_cost", "align_similarity", "LmOptions", "LmResult", "solve_lm",
           "lm_compute_step"]
