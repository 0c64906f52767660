"""complex64-mode output error vs the complex128 oracle on shrunk configs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_1908_01964_b200 import GpuContext, Hyperparams, SolverOptions, synth
g64 = GpuContext(0, precision="c64")
for cfg, I, J, it in [(0, 64, 320, 100), (1, 64, 640, 100), (4, 16, 4096, 100), (2, 4, 20000, 50)]:
    u = synth.make_config(cfg, 1, I=I, J=J)[0]
    inp = O.build_noise_scm(u.W, u.A, u.X, 0); p0 = O.init_params(inp, u.T, u.V, u.W, u.A, u.X)
    g = g64.run_algorithm2(inp, p0, Hyperparams(), u.X, SolverOptions(iters=it)).params
    o = O.run("accel2", inp, p0, u.X, O.SolverOptions(iters=it)).params
    gd = g64.extract_target(inp, g, u.X).dry; _, od = O.extract_target(inp, o, u.X)
    r = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
    print(f"cfg{cfg} I={I} J={J} iters={it}: dry rel-L2 {r(gd, od):.2e}  r_h {r(g.r_h, o.r_h):.2e}  r_u {r(g.r_u, o.r_u):.2e}  lambda {r(g.lam, o.lam):.2e}")
