"""Small end-to-end runs of the hot path for the bounds-checked library build.

    NSF_MPM_LIB=paper_2310_17790_b200/libnsf_mpm_checked.so python tools/checked_run.py c1_spin
(tests/test_gpu_checked.py runs it).  compute-sanitizer is closed on the GPU pool
(runs under it left GPUs needing a reset), so memory safety is checked by the
library's own device asserts (NSF_CHECK, csrc/params.cuh) on these scenes:
c1_spin (fused full-order path, 40 substeps: crosses a re-binning), dense_cluster
(~90 particles per cell: several staged rounds, >1 segment per block, scatter-list
overflow), c5_small (reduced path: tcgen05 MLP + P2G epilogue, reduced G2P,
re-binning), det (deterministic fixed-point path), gradw (split pipeline), sparse
(the sparse fused variant).  Prints one line per scene; a failed check traps the
kernel and the next call raises NSF_ERR_CUDA.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2310_17790_b200 as nsf  # noqa: E402
import scenes  # noqa: E402


def dense_cluster():
    sc = scenes.block_scene("dense", 32, (12, 12, 12), (18, 18, 18), scenes.FIXED_COROTATED, 16,
                            vnoise=0.3, Fnoise=0.01, Cnoise=1.0)
    rng = np.random.default_rng(16)
    n = 20000
    sc.x = rng.uniform(12.0 / 32, 18.0 / 32, size=(n, 3)).astype(np.float32)
    sc.v = (rng.normal(size=(n, 3)) * 0.3).astype(np.float32)
    sc.C = (rng.normal(size=(n, 3, 3)) * 1.0).astype(np.float32)
    sc.F = (np.eye(3) + rng.normal(size=(n, 3, 3)) * 0.01).astype(np.float32)
    return sc


def run(name, steps):
    if name == "c1_spin":
        sc = scenes.c1_spin()
    elif name == "dense_cluster":
        sc = dense_cluster()
    elif name == "c5_small":
        sc = scenes.c5_small(n_scenes=3, per_scene=300)
    elif name == "det":
        sc = scenes.c1_spin()
        sc.cfg.deterministic = 1
    elif name == "sparse":
        os.environ["NSF_FUSED_VARIANT"] = "sparse"
        sc = scenes.c1_spin()
    elif name == "gradw":
        sc = scenes.block_scene("FCg", 32, (9, 6, 10), (20, 15, 19), scenes.FIXED_COROTATED, 14,
                                keep=3333, vnoise=0.3, Fnoise=0.02, Cnoise=3.0, force_mode=scenes.FORCE_GRADW)
    else:
        raise SystemExit(f"unknown scene {name}")
    sim = nsf.Simulator(sc.cfg)
    sim.load_scene(sc)
    sim.substep(steps)
    sim.sync()
    mask = nsf.NSF_FIELD_X | nsf.NSF_FIELD_V | nsf.NSF_FIELD_C
    s = sim.read(mask)
    sim.close()
    print(f"{name}: {steps} substeps ok, |x| = {np.linalg.norm(s['x']):.6f}")


if __name__ == "__main__":
    names = sys.argv[1:] or ["c1_spin", "dense_cluster", "c5_small"]
    steps = int(os.environ.get("SAN_STEPS", "40"))
    for n in names:
        run(n, steps)
