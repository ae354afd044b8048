"""GPU edge cases of the substep (reading #21, #25 in DESIGN.md):

* inverted (det F < 0) and nearly singular F (sigma_3 < 1e-4) driven through the
  fused G2P2G kernel, whose fast constitutive paths (polar iteration, eigen-free
  log strain) must fall back to the rotation-safe SVD -- single-substep parity
  with the fp64 oracle at the 1e-5 bar, with the grid update both in the fused
  kernel and as its own pass;
* nsf_mpm_inverted_count equal to the number of particles whose F_E the oracle
  leaves with det <= 0;
* a NaN injected into one particle is reported as NSF_ERR_NONFINITE with that
  particle's load index, and a particle thrown out of the safe region as
  NSF_ERR_OUT_OF_DOMAIN with its index (full-order and reduced paths).
"""
import numpy as np
import pytest

import scenes
from tests.parity_util import BAR_STEP, single_step_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nsf():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2310_17790_b200 as m
    return m


def _rot(rng, n):
    """n random rotations (det +1) from QR of Gaussian matrices."""
    A = rng.normal(size=(n, 3, 3))
    Q, R = np.linalg.qr(A)
    Q = Q * np.sign(np.diagonal(R, axis1=1, axis2=2))[:, None, :]
    Q[np.linalg.det(Q) < 0, :, 0] *= -1.0
    return Q


def edge_scene(model, seed):
    """A block of particles where 15% have an inverted F (singular values 1.3, 1.0,
    -0.7: the reflection is well separated, so the rotation-safe SVD is unique) and
    10% a nearly singular one (1.2, 0.9, 5e-5); the rest is I + noise."""
    sc = scenes.block_scene("edge", 32, (9, 4, 9), (21, 14, 21), model, seed, keep=6000,
                            vnoise=0.2, Fnoise=0.02, Cnoise=1.0)
    rng = np.random.default_rng(seed)
    n = sc.n
    idx = rng.permutation(n)
    inv, sing = idx[: int(0.15 * n)], idx[int(0.15 * n): int(0.25 * n)]
    F = sc.F.astype(np.float64)
    for sel, sig in ((inv, (1.3, 1.0, -0.7)), (sing, (1.2, 0.9, 5e-5))):
        U, V = _rot(rng, len(sel)), _rot(rng, len(sel))
        F[sel] = U @ np.diag(sig) @ np.transpose(V, (0, 2, 1))
    sc.F = F.astype(np.float32)
    return sc, inv


MODELS = {"FC": scenes.FIXED_COROTATED, "DP": scenes.DRUCKER_PRAGER, "VM": scenes.VON_MISES}


@pytest.mark.parametrize("gu", ["rot", "kernel", "barrier"])
@pytest.mark.parametrize("model", list(MODELS))
def test_inverted_and_degenerate_F(nsf, model, gu, monkeypatch):
    monkeypatch.setenv("NSF_FUSED_GU", gu)
    sc, inv = edge_scene(MODELS[model], 31 + list(MODELS).index(model))
    sim = nsf.Simulator(sc.cfg)
    sim.load_scene(sc)
    try:
        errs, s1, ref = single_step_parity(sim, sc.cfg, 0)
        assert all(e <= BAR_STEP for e in errs.values()), errs
        # the count of inverted updates is the oracle's count of det F_E <= 0
        det_ref = np.linalg.det(ref["F"])
        # no sign decision within fp32 rounding (|det| error ~ 1e-7 sigma_1 sigma_2; the nearly
        # singular ones keep det ~ 5e-5)
        assert np.min(np.abs(det_ref)) > 1e-5
        assert sim.inverted_count() == int(np.sum(det_ref <= 0.0))
        if model == "FC":   # F_E = F_trial: the inverted particles stay inverted
            assert int(np.sum(det_ref <= 0.0)) == len(inv)
    finally:
        sim.close()


def _expect(nsf, sim, status, index):
    with pytest.raises(nsf.NsfError) as e:
        sim.sync()
    assert e.value.status == status, str(e.value)
    assert f"particle {index} (load order)" in str(e.value), str(e.value)


def test_nonfinite_input_rejected_at_load(nsf):
    """A NaN in a particle's F (or a tau(F) that overflows) is rejected by the load
    with NSF_ERR_NONFINITE and that particle's index; the handle stays unloaded."""
    sc = scenes.c1_spin()
    bad = 1234
    sc.F = sc.F.copy()
    sc.F[bad, 1, 1] = np.nan
    sim = nsf.Simulator(sc.cfg)
    with pytest.raises(nsf.NsfError) as e:
        sim.load_scene(sc)
    assert e.value.status == nsf.NSF_ERR_NONFINITE and f"particle {bad} (load order)" in str(e.value)
    with pytest.raises(nsf.NsfError) as e:     # nothing loaded
        sim.substep(1)
    assert e.value.status == nsf.NSF_ERR_BAD_STATE
    sc.F[bad] = np.eye(3) * 1e6                # finite, but lambda (J - 1) J overflows fp32
    with pytest.raises(nsf.NsfError) as e:
        sim.load_scene(sc)
    assert e.value.status == nsf.NSF_ERR_NONFINITE and f"particle {bad} (load order)" in str(e.value)
    sim.close()


def test_reduced_nonfinite_during_substep_reports_load_index(nsf):
    """A point whose network input overflows the MLP gets tau = inf/NaN inside the
    substep (device side); the reduced G2P flags it with its load index.  Points are
    sparse (300 per 64^3 grid), so the bad point shares no stencil node with another."""
    sc = scenes.c5_small(n_scenes=3, per_scene=300)
    # a point of scene 1 whose stencil shares no node with any other point's
    # (stencil bases >= 3 cells apart on some axis)
    a, b = int(sc.scene_offsets[1]), int(sc.scene_offsets[2])
    base = np.floor(sc.x[a:b].astype(np.float64) * sc.cfg.grid_res - 0.5).astype(np.int64)
    cheb = np.max(np.abs(base[:, None, :] - base[None, :, :]), axis=2)
    np.fill_diagonal(cheb, 1 << 20)
    bad = a + int(np.flatnonzero(cheb.min(axis=1) >= 3)[0])
    sc.X_ref = sc.X_ref.copy()
    sc.X_ref[bad] = np.nan       # the network input: tau = NaN inside the substep
    sim = nsf.Simulator(sc.cfg)
    sim.load_scene(sc)
    sim.substep(1)
    _expect(nsf, sim, nsf.NSF_ERR_NONFINITE, bad)
    sim.close()


def test_out_of_domain_reports_load_index(nsf):
    sc = scenes.c1_spin()
    # an isolated particle (cell 6.4 on each axis, away from the body in cells
    # [12, 20) and from the walls) moving 0.2 = 6.4 cells per substep, inserted at 777
    bad = 777
    sc.x = np.insert(sc.x, bad, (0.2, 0.2, 0.2), axis=0)
    sc.v = np.insert(sc.v, bad, (0.0, -2.0e3, 0.0), axis=0)
    sc.C = np.insert(sc.C, bad, np.zeros((3, 3)), axis=0)
    sc.F = np.insert(sc.F, bad, np.eye(3), axis=0)
    sim = nsf.Simulator(sc.cfg)
    sim.load_scene(sc)
    sim.substep(1)
    _expect(nsf, sim, nsf.NSF_ERR_OUT_OF_DOMAIN, bad)
    sim.close()
