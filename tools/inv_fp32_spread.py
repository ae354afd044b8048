"""Measure how far a correct fp32-accumulating evaluation of the bf16-emulating
deformation network moves one Gauss-Newton step (Eq. (10)) from the fp64
emulating oracle: the network of tests/test_gpu_inversion.py evaluated with every
matmul accumulated sequentially in fp32 (products exact: bf16 x bf16), in several
summation orders.  DESIGN.md reading #37 quotes its output.

    python tools/inv_fp32_spread.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from tests.inv_util import fp32_spread, inversion_scene  # noqa: E402

if __name__ == "__main__":
    sc, gnet, _ = inversion_scene()
    for ns in (64, 50, 256):
        spread, gap = fp32_spread(sc, gnet, sc.x, sc.z0.astype(np.float64), ns, orders=8, per_order=True)
        print(f"n_sample {ns}: emulate-vs-exact {gap:.3f} of the step; fp32 orders: "
              + " ".join(f"{s:.4f}" for s in spread))
