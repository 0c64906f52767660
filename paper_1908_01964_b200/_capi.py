"""ctypes binding of include/rcscm_gpu.h (librcscm_gpu.so, built in-tree).

The product path has no CPU fallback: if the CUDA library is missing or fails
to load, importing this module raises immediately.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RCSCM_GPU_LIB") or os.path.join(_HERE, "librcscm_gpu.so")  # env: A/B builds

RCSCM_OK = 0
RCSCM_INVALID_INPUT = 2
RCSCM_NUMERICAL = 3
RCSCM_CUDA_ERROR = 4
RCSCM_UNSUPPORTED = 5

RCSCM_C128 = 0
RCSCM_C64 = 1

STAGE_SETUP = 1
STAGE_PRECOMPUTE = 2
STAGE_ACCEL = 4
STAGE_NAIVE = 8
STAGE_WIENER = 16
STAGE_RESET = 32

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64


class GpuConfig(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("precision", ctypes.c_int), ("stream", ctypes.c_void_p),
                ("devices", ctypes.POINTER(ctypes.c_int)), ("num_devices", ctypes.c_int)]


class CInputs(ctypes.Structure):
    _fields_ = [
        ("num_bins", ctypes.c_int64),
        ("frames", ctypes.c_int64),
        ("mics", ctypes.c_int),
        ("n_h", ctypes.c_int),
        ("a", _dp),
        ("R_prime", _dp),
        ("R_prime_pinv", _dp),
        ("b", _dp),
    ]


class CParams(ctypes.Structure):
    _fields_ = [("r_h", _dp), ("r_u", _dp), ("lambda_", _dp)]


class CHyper(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_double), ("beta", ctypes.c_double)]


class COpts(ctypes.Structure):
    _fields_ = [
        ("iters", ctypes.c_int),
        ("compute_objective", ctypes.c_int),
        ("record_trajectory", ctypes.c_int),
        ("rel_obj_tol", ctypes.c_double),
        ("threads", ctypes.c_int),
        ("eps_var", ctypes.c_double),
        ("gamma_fault", ctypes.c_double),
    ]


class CResult(ctypes.Structure):
    _fields_ = [
        ("objective", _dp),
        ("n_objective", _ip),
        ("iter_seconds", _dp),
        ("n_iters", _ip),
        ("traj_r_h", _dp),
        ("traj_r_u", _dp),
        ("traj_lambda", _dp),
    ]


class CExtractOpts(ctypes.Structure):
    _fields_ = [
        ("sample_rate", ctypes.c_double),
        ("win_ms", ctypes.c_double),
        ("hop_ms", ctypes.c_double),
        ("nmf_bases", ctypes.c_int),
        ("ilrma_iters", ctypes.c_int),
        ("seed", ctypes.c_uint64),
        ("target_index", ctypes.c_int),
        ("backend", ctypes.c_int),
        ("iters", ctypes.c_int),
        ("alpha", ctypes.c_double),
        ("beta", ctypes.c_double),
        ("eps_var", ctypes.c_double),
        ("rel_obj_tol", ctypes.c_double),
        ("compute_objective", ctypes.c_int),
        ("samples_layout", ctypes.c_int),
    ]


class CExtractResult(ctypes.Structure):
    _fields_ = [
        ("target_index", ctypes.c_int),
        ("n_iters", ctypes.c_int),
        ("bins", ctypes.c_int64),
        ("frames", ctypes.c_int64),
        ("objective", _dp),
        ("n_objective", ctypes.c_int),
        ("iter_seconds", _dp),
    ]


# Every symbol include/rcscm_gpu.h declares, with its ctypes signature.
SIGNATURES = {
    "rcscm_gpu_create": (ctypes.c_int, [ctypes.POINTER(GpuConfig), ctypes.POINTER(_vp)]),
    "rcscm_gpu_destroy": (None, [_vp]),
    "rcscm_gpu_last_error": (ctypes.c_char_p, []),
    "rcscm_gpu_launch_count": (ctypes.c_int64, [_vp]),
    "rcscm_gpu_build_noise_scm": (ctypes.c_int, [_vp, _i64, _i64, ctypes.c_int, _dp, _dp, _dp, ctypes.c_int,
                                                 ctypes.c_double, _dp, _dp, _dp, _dp]),
    "rcscm_gpu_init_params": (ctypes.c_int, [_vp, ctypes.POINTER(CInputs), ctypes.c_int, _dp, _dp, _dp, _dp, _dp,
                                             ctypes.POINTER(CParams)]),
    "rcscm_gpu_map_objective": (ctypes.c_int, [_vp, ctypes.POINTER(CInputs), ctypes.POINTER(CParams),
                                               ctypes.POINTER(CHyper), _dp, _dp]),
    "rcscm_gpu_run_naive": (ctypes.c_int, [_vp, ctypes.POINTER(CInputs), ctypes.POINTER(CParams),
                                           ctypes.POINTER(CHyper), _dp, ctypes.POINTER(COpts),
                                           ctypes.POINTER(CParams), ctypes.POINTER(CResult)]),
    "rcscm_gpu_stft_shape": (ctypes.c_int, [ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                            ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                            ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]),
    "rcscm_gpu_stft_analyze": (ctypes.c_int, [_vp, _dp, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                                              ctypes.c_double, ctypes.c_double, _dp]),
    "rcscm_gpu_stft_synthesize": (ctypes.c_int, [_vp, _dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                                 ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                                 ctypes.c_double, ctypes.c_double, _dp]),
    "rcscm_gpu_extract": (ctypes.c_int, [_vp, ctypes.POINTER(CExtractOpts), _dp, ctypes.c_int64, ctypes.c_int, _dp,
                                         _dp, ctypes.POINTER(CExtractResult)]),
    "rcscm_gpu_sphere": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, _dp, _dp, _dp]),
    "rcscm_gpu_run_ilrma": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, ctypes.c_uint64, _dp, _dp, _dp, _dp, _dp]),
    "rcscm_gpu_run_algorithm1": (ctypes.c_int, [_vp, ctypes.POINTER(CInputs), ctypes.POINTER(CParams),
                                                ctypes.POINTER(CHyper), _dp, ctypes.POINTER(COpts),
                                                ctypes.POINTER(CParams), ctypes.POINTER(CResult)]),
    "rcscm_gpu_run_algorithm2": (ctypes.c_int, [_vp, ctypes.POINTER(CInputs), ctypes.POINTER(CParams),
                                                ctypes.POINTER(CHyper), _dp, ctypes.POINTER(COpts),
                                                ctypes.POINTER(CParams), ctypes.POINTER(CResult)]),
    "rcscm_gpu_run_accel": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.POINTER(CInputs), ctypes.POINTER(CParams),
                                           ctypes.POINTER(CHyper), _dp, ctypes.POINTER(COpts),
                                           ctypes.POINTER(CParams), ctypes.POINTER(CResult)]),
    "rcscm_gpu_build_inputs": (ctypes.c_int, [_vp, _i64, _i64, ctypes.c_int, _dp, _dp, _dp, ctypes.c_int,
                                              ctypes.c_double, ctypes.c_int, _dp, _dp, _dp, _dp, _dp, _dp,
                                              ctypes.POINTER(CParams)]),
    "rcscm_gpu_extract_target": (ctypes.c_int, [_vp, ctypes.POINTER(CInputs), ctypes.POINTER(CParams), _dp, _dp,
                                                _dp]),
    "rcscm_gpu_extract_noise": (ctypes.c_int, [_vp, ctypes.POINTER(CInputs), ctypes.POINTER(CParams), _dp, _dp]),
    "rcscm_gpu_session_load": (ctypes.c_int, [_vp, _i64, _i64, _i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp,
                                              _dp, _dp, _dp, _dp]),
    "rcscm_gpu_session_run": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(CHyper),
                                             ctypes.c_double]),
    "rcscm_gpu_session_fetch": (ctypes.c_int, [_vp, _dp, _dp, _dp, _dp, _dp, ctypes.c_int]),
    "rcscm_gpu_session_check": (ctypes.c_int, [_vp]),
    "rcscm_gpu_stream": (_vp, [_vp]),
    "rcscm_gpu_probe_fp64": (ctypes.c_int, [_vp, _dp, _dp]),
    "rcscm_gpu_probe_fp32": (ctypes.c_int, [_vp, _dp, _dp]),
}

_lib = None


def load():
    """Load librcscm_gpu.so (raises OSError if it is absent: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OSError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                          "(there is no CPU fallback for the product path)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib
