"""One device extract (reference test configuration) for a launch-list profile."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_1908_01964_b200 import GpuContext
from test_extract import _mixture
x = _mixture(4, 139200, 1)
ctx = GpuContext(0)
g = ctx.extract(x, 16000.0, nmf_bases=10, ilrma_iters=50, seed=1, iters=100)
print("target_index", g["target_index"], "iters", g["n_iters"])
