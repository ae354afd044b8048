"""GPU parity of network inference and of the sample /
integration particle sets (lines 265-269) against oracle/inference.py.

Bars: x and C as the MLP (1e-3 relative L2 against the bf16-emulating oracle,
reading #20); v = (g(z_n) - g(z_prev)) / dt is a difference of two bf16
networks, so it is compared at a latent step |z_n - z_prev| ~ 0.5 where the
difference is well above the bf16 rounding noise (bar 2e-2), and must be exactly
0 when z_prev = z_n.  The integration set is unique except for points whose
stencil decision flips within the network's rounding noise: every point where
GPU and oracle disagree must lie within 1e-4 of a cell boundary (oracle x), and
there may be at most 2 such points per scene."""
import numpy as np
import pytest
from scipy.spatial import cKDTree

import scenes
from oracle.inference import field, infer_state, integration_set, ordered_points
from tests.parity_util import rel_err

pytestmark = pytest.mark.gpu
BAR_MLP = 1e-3
BAR_V = 2e-2


@pytest.fixture(scope="module")
def nsf():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2310_17790_b200 as m
    return m


def setup(nsf, n_scenes=3, per_scene=300, g=None):
    sc = scenes.c5_small(n_scenes=n_scenes, per_scene=per_scene)
    sc.dz = np.zeros_like(sc.dz)          # z_n = z0 at every step
    g, l = g or scenes.deformation_field(), scenes.affine_field()
    sim = nsf.Simulator(sc.cfg)
    sim.load_scene(sc)
    sim.load_deformation_field(g)
    sim.load_affine_field(l)
    return sc, g, l, sim


def test_infer_state_parity(nsf):
    sc, g, l, sim = setup(nsf)
    try:
        rng = np.random.default_rng(41)
        z_prev = (sc.z0 + 0.5 * rng.normal(size=sc.z0.shape)).astype(np.float32)
        sim.infer_state(z_prev)
        st = sim.read(nsf.NSF_FIELD_X | nsf.NSF_FIELD_V | nsf.NSF_FIELD_C)
        dt = sc.cfg.dt
        for s in range(sc.cfg.n_scenes):
            a, b = sc.scene_offsets[s], sc.scene_offsets[s + 1]
            x, v, C = infer_state(sc.X_ref[a:b], sc.z0[s], z_prev[s], g, l, dt, mode="emulate")
            assert rel_err(st["x"][a:b], x) <= BAR_MLP
            assert rel_err(st["C"][a:b], C) <= BAR_MLP
            assert rel_err(st["v"][a:b], v) <= BAR_V
        # z_prev = z_n (step 0, no z_prev): at rest, exactly
        sim.infer_state(None)
        assert np.all(sim.read(nsf.NSF_FIELD_V)["v"] == 0.0)
        # the state drives the next substep
        sim.infer_state(z_prev)
        sim.substep(2)
        sim.sync()
        assert np.all(np.isfinite(sim.read(nsf.NSF_FIELD_X)["x"]))
    finally:
        sim.close()


def _near_boundary(x, dx, eps=1e-4):
    t = x / dx - 0.5
    return np.any(np.abs(t - np.round(t)) * dx < eps, axis=-1)


def test_integration_set_parity(nsf):
    n_ref, n_sample = 5000, 16
    # a near-identity stand-in g: the body is not collapsed, N is a proper subset (~10%)
    sc, g, l, sim = setup(nsf, g=scenes.deformation_field_near_identity())
    try:
        X_all = scenes.reference_body(n_ref=n_ref).astype(np.float32)
        rng = np.random.default_rng(42)
        ns = sc.cfg.n_scenes
        sidx = np.stack([rng.choice(n_ref, n_sample, replace=False) for _ in range(ns)]).astype(np.int32)
        counts = sim.build_integration_set(X_all, sidx)
        x_new = sim.read(nsf.NSF_FIELD_X)["x"]
        assert x_new.shape[0] == counts.sum()
        off = np.concatenate([[0], np.cumsum(counts)])
        N_grid = (sc.cfg.grid_res,) * 3
        for s in range(ns):
            x_all = field(X_all, sc.z0[s], g, "emulate")
            N_o, I_o = integration_set(X_all, sidx[s], sc.z0[s], g, N_grid, sc.cfg.dx, mode="emulate")
            xs = x_new[off[s]:off[s + 1]]
            # S first, in the given order
            assert rel_err(xs[:n_sample], x_all[sidx[s]]) <= BAR_MLP
            # the GPU's members, identified by their positions
            d, idx = cKDTree(x_all).query(xs)
            assert np.all(d < 1e-3), (s, float(d.max()))
            assert len(xs) < n_ref, "N should be a proper subset"
            gpu_set = set(idx.tolist())
            assert len(gpu_set) == len(idx)
            diff = gpu_set ^ set(N_o.tolist())
            assert len(diff) <= 2, (s, len(diff))
            for p in diff:
                assert _near_boundary(x_all[p], sc.cfg.dx), (s, p)
            # N \ S in increasing index order
            rest = idx[n_sample:]
            assert np.all(np.diff(rest) > 0)
            assert np.array_equal(ordered_points(N_o, sidx[s])[:n_sample], sidx[s])
        # the new points step and invert (S = the first n_sample points)
        sim.substep(1)
        z = sim.invert_latents(n_sample, 1)
        assert np.all(np.isfinite(z))
    finally:
        sim.close()


def test_inference_requires_networks(nsf):
    sc = scenes.c5_small(n_scenes=2, per_scene=50)
    sim = nsf.Simulator(sc.cfg)
    sim.load_scene(sc)
    try:
        with pytest.raises(nsf.NsfError):
            sim.infer_state(None)
        sim.load_deformation_field(scenes.deformation_field())
        with pytest.raises(nsf.NsfError):
            sim.infer_state(None)
        sim.load_affine_field(scenes.affine_field())
        sim.infer_state(None)
        X = scenes.reference_body(n_ref=100).astype(np.float32)
        with pytest.raises(nsf.NsfError):      # repeated sample index
            sim.build_integration_set(X, np.zeros((2, 3), np.int32))
        with pytest.raises(nsf.NsfError):      # out of range
            sim.build_integration_set(X, np.full((2, 3), 100, np.int32))
    finally:
        sim.close()
