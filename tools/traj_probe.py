"""Trajectory divergence GPU vs oracle for the parity scenes over K substeps
(diagnostic for choosing trajectory-test bars).

    python tools/traj_probe.py [K]
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402


def main(K):
    import scenes
    import paper_2310_17790_b200 as nsf
    from oracle import mpm
    from tests.parity_util import rel_err
    from tests.test_gpu_parity import small_scenes
    for name, sc in small_scenes().items():
        if name in ("dense_cluster",):
            continue
        sim = nsf.Simulator(sc.cfg)
        sim.load_scene(sc)
        sim.substep(K)
        sim.sync()
        g = sim.read()
        sim.close()
        P = mpm.params_from_config(sc.cfg)
        ref = mpm.run({"x": sc.x, "v": sc.v, "C": sc.C, "F": sc.F, "tau": mpm.initial_tau(sc.F, P)}, P, K)
        ex = rel_err(g["x"], ref["x"])
        disp = rel_err(g["x"] - sc.x, ref["x"] - sc.x)
        dv = rel_err(g["v"], ref["v"])
        print(f"{name:12s} K={K} x {ex:.2e} disp {disp:.2e} v {dv:.2e}")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 100)
