"""Parity table against the binary128 ground truth (oracle/truth.cpp).

For every case of tests/truth_cases.py: one iteration of Algorithm 2 and of the
naive rule from params0, evaluated by the double oracle (the reference's
arithmetic) and by the GPU (C ABI), each compared elementwise with the binary128
truth. Prints a markdown table (max relative error per field, the r_u error in
units of eps * S, and how many slots exceed 1e-9) -- DESIGN.md section 5 and
profiles/r02/parity_truth.md carry its output. Needs a GPU unless --cpu.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from truth_cases import CASES, NAIVE_CASES, bound_units, case_id, field_errors, instance  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cpu", action="store_true", help="oracle rows only")
a = ap.parse_args()

from oracle import oracle as O  # noqa: E402

O.build()
gpu = None
if not a.cpu:
    from paper_1908_01964_b200 import GpuContext, Hyperparams, SolverOptions

    gpu = GpuContext(0)

print("| rule | case | slots | impl | r_h max rel | r_u max rel | lambda max rel | slots r_u > 1e-9 "
      "| max err / (eps B): r_h, r_u, lambda | slots gpu err > max(1e-9, oracle err) |")
print("|---|---|---|---|---|---|---|---|---|---|")
for rule, cases in (("accel2", CASES), ("naive", NAIVE_CASES)):
    for c in cases:
        u, inp, p0 = instance(O, *c)
        if rule == "accel2":
            tr, B = O.truth_accel_one_iter(inp, p0, u.X)
            o = O.run("accel2_binparallel", inp, p0, u.X, O.SolverOptions(iters=1, threads=8)).params
        else:
            tr, B = O.truth_naive_one_iter(inp, p0, u.X)
            o = O.run("naive", inp, p0, u.X, O.SolverOptions(iters=1)).params
        rows = [("oracle", o)]
        if gpu is not None:
            fn = gpu.run_algorithm2 if rule == "accel2" else gpu.run_naive
            rows.append(("gpu", fn(inp, p0, Hyperparams(), u.X, SolverOptions(iters=1)).params))
        eo = field_errors(o, tr)
        for name, p in rows:
            e = field_errors(p, tr)
            bu = bound_units(p, tr, B)
            worse = "-" if name == "oracle" else ", ".join(
                str(int((e[f] > np.maximum(1e-9, eo[f])).sum())) for f in ("r_h", "r_u", "lambda"))
            print(f"| {rule} | {case_id(c)} | {u.X.shape[0] * u.X.shape[1]} | {name} | {e['r_h'].max():.2e} | "
                  f"{e['r_u'].max():.2e} | {e['lambda'].max():.2e} | {int((e['r_u'] > 1e-9).sum())} | "
                  f"{bu['r_h'].max():.2f}, {bu['r_u'].max():.2f}, {bu['lambda'].max():.2f} | {worse} |", flush=True)
