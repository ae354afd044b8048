"""Far particles and the grid-update modes of the fused kernel:
the grid update visits the segments' halo (every block in the
27-block neighbourhood of a non-empty segment) plus the blocks a "far" particle
-- one whose stencil left that neighbourhood -- flagged; with the update in the
kernel after a grid-wide barrier (barrier) or with three rotating grids (rot)
the touched lists alone decide.

Scene: an elastic block plus isolated "bullets" flying at 100 m/s (0.64 cells
per substep), which leave their re-binning blocks by more than 4 cells after a
few substeps and so exercise the far fix-up on most substeps before and after
the re-binning at substep 32.  Every mode's trajectory must equal the
separate-pass trajectory to fp32 reduction-order noise, and all the oracle's.
"""
import numpy as np
import pytest

import scenes
from tests.parity_util import BAR_STEP, BAR_TRAJ, compare, gpu_state, oracle_step, single_step_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nsf():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2310_17790_b200 as m
    return m


def bullet_scene(seed=71):
    sc = scenes.block_scene("far", 64, (36, 8, 36), (52, 24, 52), scenes.FIXED_COROTATED, seed, keep=6000,
                            vnoise=0.3, Fnoise=0.01, Cnoise=0.5)
    rng = np.random.default_rng(seed)
    # 24 bullets on a lattice 8 cells apart (no shared stencil node), moving +x at 100 m/s
    g = np.array([[i, j, k] for i in range(2) for j in range(3) for k in range(4)], np.float64)
    xb = (np.array([6.0, 30.0, 8.0]) + 8.0 * g + rng.uniform(0.3, 0.7, g.shape)) / 64.0
    vb = np.tile([100.0, 0.0, 0.0], (len(xb), 1))
    n0 = sc.n
    sc.x = np.concatenate([sc.x, xb.astype(np.float32)])
    sc.v = np.concatenate([sc.v, vb.astype(np.float32)])
    sc.C = np.concatenate([sc.C, np.zeros((len(xb), 3, 3), np.float32)])
    sc.F = np.concatenate([sc.F, np.tile(np.eye(3, dtype=np.float32), (len(xb), 1, 1))])
    sc.cfg.gravity = (0.0, 0.0, 0.0)
    return sc, np.arange(n0, sc.n)


def _run(nsf, sc, gu, steps, monkeypatch):
    monkeypatch.setenv("NSF_FUSED_GU", gu)
    sim = nsf.Simulator(sc.cfg)
    sim.load_scene(sc)
    try:
        s0 = gpu_state(sim)
        sim.substep(steps)
        sim.sync()
        return s0, gpu_state(sim)
    finally:
        sim.close()


@pytest.mark.parametrize("gu", ["kernel", "barrier", "rot"])
def test_far_particles_match_separate_pass_and_oracle(nsf, gu, monkeypatch):
    sc, bullets = bullet_scene()
    steps = 40   # crosses the re-binning after substep 32
    s0, a = _run(nsf, sc, gu, steps, monkeypatch)
    _, b = _run(nsf, sc, "kernel", steps, monkeypatch)
    # the bullets really left their blocks' neighbourhoods (> 4 cells)
    assert np.min(a["x"][bullets, 0] - sc.x[bullets, 0]) * 64 > 20
    # vs the separate pass: the same arithmetic, only the reduction order differs
    errs = compare(a, b, sc.cfg)
    assert all(e <= BAR_STEP for e in errs.values()), errs
    assert np.max(np.abs(a["x"][bullets] - b["x"][bullets])) < 1e-6
    # and the oracle's trajectory
    ref = {k: s0[k] for k in ("x", "v", "C", "F", "tau")}   # the loaded fp32 state (tau^0: reading #9)
    for k in range(steps):
        ref = oracle_step(ref, sc.cfg, k)
    e = np.linalg.norm(a["x"] - ref["x"]) / np.linalg.norm(ref["x"])
    assert e <= BAR_TRAJ, e
    assert np.max(np.abs(a["x"][bullets] - ref["x"][bullets])) < 1e-5
