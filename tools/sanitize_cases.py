"""Small GPU cases for compute-sanitizer (racecheck / synccheck / memcheck): the
cluster K2 at every cluster size (2, 4, 8, 16 CTAs; st.async + mbarrier
exchange), the single-CTA K2, the fused Wiener epilogue, the pipelined
run_algorithm2 (chunks on copy / compute / D2H streams), the naive rule,
Algorithm 1, and the cmd_extract chain (STFT, ILRMA, solver, Wiener, ISTFT).
Tiny shapes: the sanitizers serialise and instrument every access.

usage: compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402  (inputs only: make_verify_instance)
from paper_1908_01964_b200 import GpuContext, Hyperparams, SolverOptions, synth  # noqa: E402
import paper_1908_01964_b200._capi as C  # noqa: E402

h = Hyperparams()
gpu = GpuContext(0)


def cluster(cl):
    os.environ["RCSCM_ACCEL_CL"] = str(cl)
    inp, p, X = O.make_verify_instance(3, 96 * cl, 2, 5 + cl)
    gpu.run_algorithm2(inp, p, h, X, SolverOptions(iters=4))
    del os.environ["RCSCM_ACCEL_CL"]


def session_fused(cfg, J):
    X, W, A, T, V = synth.stack(synth.make_config(cfg, utterances=2, I=4, J=J))
    gpu.session_load(X, W, A, T, V, 0)
    gpu.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
    gpu.session_run(C.STAGE_RESET | C.STAGE_PRECOMPUTE | C.STAGE_ACCEL | C.STAGE_WIENER, 3)
    gpu.session_check()


def pipelined():
    os.environ["RCSCM_PIPELINE_CHUNKS"] = "3"
    inp, p, X = O.make_verify_instance(300, 32, 4, 3)
    gpu.run_algorithm2(inp, p, h, X, SolverOptions(iters=3))
    del os.environ["RCSCM_PIPELINE_CHUNKS"]


def naive_accel1():
    inp, p, X = O.make_verify_instance(5, 40, 3, 9)
    gpu.run_naive(inp, p, h, X, SolverOptions(iters=3))
    gpu.run_algorithm1(inp, p, h, X, SolverOptions(iters=3))
    gpu.run_algorithm2(inp, p, h, X, SolverOptions(iters=3, compute_objective=True, record_trajectory=True))


def extract():
    rng = np.random.default_rng(0)
    samples = rng.standard_normal((2, 4000))
    gpu.extract(samples, 16000.0, nmf_bases=2, ilrma_iters=2, iters=3)


CASES = {"cluster2": lambda: cluster(2), "cluster4": lambda: cluster(4), "cluster8": lambda: cluster(8),
         "cluster16": lambda: cluster(16), "single": lambda: session_fused(3, 64),
         "fused_c4": lambda: session_fused(4, 512), "pipelined": pipelined, "naive_accel1": naive_accel1,
         "extract": extract}

if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
        print("case", name, "ok", flush=True)
    gpu.close()
