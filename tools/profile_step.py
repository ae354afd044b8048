"""Run a few C3 substeps (no timing) -- the command profiled under ncu.

    python tools/profile_step.py [--config C3] [--substeps 4] [--warmup 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--substeps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=2)
    a = ap.parse_args()
    import torch
    import scenes
    import paper_2310_17790_b200 as nsf
    sc = {"C1": scenes.c1, "C2": scenes.c2, "C3": scenes.c3, "C4": scenes.c4, "C5": scenes.c5}[a.config]()
    sim = nsf.Simulator(sc.cfg)
    sim.load_scene(sc)
    sim.substep(a.warmup)
    sim.sync()
    sim.substep(a.substeps)
    sim.sync()
    st = sim.read(nsf.NSF_FIELD_X)
    assert np.all(np.isfinite(st["x"]))
    sim.close()
    print("ok", a.config, sc.n)


if __name__ == "__main__":
    main()
