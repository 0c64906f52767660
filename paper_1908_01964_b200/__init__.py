"""B200-native (sm_100a) hot path of rank-constrained SCM estimation (arXiv 1908.01964).

The numerics live in librcscm_gpu.so (CUDA kernels + C ABI, include/rcscm_gpu.h);
this package is the Python mirror of the reference's entry points over it.
"""
from .api import (  # noqa: F401
    CudaError,
    ExtractionResult,
    GpuContext,
    Hyperparams,
    InvalidInputError,
    NumericalError,
    RcscmInputs,
    RcscmParams,
    SolverOptions,
    SolverResult,
    UnsupportedError,
    build_noise_scm,
    default_context,
    extract_noise,
    extract_target,
    init_params,
    map_objective,
    run_algorithm1,
    run_algorithm2,
    run_naive,
)
from . import records, synth  # noqa: F401
