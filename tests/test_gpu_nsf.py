"""GPU parity for the reduced-order variant (§5.1-5.2, BASELINE.json
config 5): the neural stress field MLP vs the oracle's bf16-emulating fp64 MLP
(bar 1e-3, reading #20), and the reduced substep (MPM on the sampled points
with tau from the MLP, no F / SVD) vs the oracle from the same state, fed the
GPU's own tau (bar 1e-5 per field)."""
import numpy as np
import pytest

import scenes
import oracle
from oracle import mpm
from oracle.mlp import nsf_stress
from tests.parity_util import rel_err, BAR_STEP

pytestmark = pytest.mark.gpu
BAR_MLP = 1e-3


@pytest.fixture(scope="module")
def nsf():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2310_17790_b200 as m
    return m


def make(nsf, sc):
    sim = nsf.Simulator(sc.cfg)
    sim.load_scene(sc)
    return sim


@pytest.mark.parametrize("m", [1, 127, 128, 1000, 4099])
def test_eval_stress_field_vs_oracle(nsf, m):
    sc = scenes.c5_small(n_scenes=2, per_scene=64)
    sim = make(nsf, sc)
    rng = np.random.default_rng(m)
    pts = rng.uniform(0.2, 0.8, size=(m, 3)).astype(np.float32)
    z = rng.normal(size=6).astype(np.float32)
    got = nsf.nsf_mpm_eval_stress_field(sim.h, z, pts)
    sim.close()
    ref = nsf_stress(pts, z, sc.mlp, sc.cfg.stress_scale, "emulate")
    exact = nsf_stress(pts, z, sc.mlp, sc.cfg.stress_scale, "exact")
    assert rel_err(got, ref) <= BAR_MLP
    assert rel_err(got, exact) <= 2e-2          # report-level: bf16 rounding points


def test_eval_stress_field_device_io(nsf):
    import torch
    sc = scenes.c5_small(n_scenes=1, per_scene=64)
    sim = make(nsf, sc)
    pts = torch.rand(300, 3, device="cuda") * 0.5 + 0.25
    z = torch.randn(6, device="cuda")
    got = nsf.nsf_mpm_eval_stress_field(sim.h, z, pts)
    host = nsf.nsf_mpm_eval_stress_field(sim.h, z.cpu().numpy(), pts.cpu().numpy())
    sim.close()
    assert np.array_equal(got.cpu().numpy(), host)


def _reduced_parity(nsf, sc, steps_before):
    sim = make(nsf, sc)
    P = mpm.params_from_config(sc.cfg)
    if steps_before:
        sim.substep(steps_before)
    s0 = sim.read(nsf.NSF_FIELD_X | nsf.NSF_FIELD_V | nsf.NSF_FIELD_C)
    sim.substep(1)
    sim.sync()
    s1 = sim.read(nsf.NSF_FIELD_X | nsf.NSF_FIELD_V | nsf.NSF_FIELD_C | nsf.NSF_FIELD_TAU)
    sim.close()
    k = steps_before
    # the MLP part: tau used in substep k vs the oracle MLP at z(k)
    ref_tau = np.concatenate([
        nsf_stress(sc.X_ref[a:b], sc.z0[s].astype(np.float64) + k * sc.dz[s].astype(np.float64), sc.mlp,
                   sc.cfg.stress_scale, "emulate")
        for s, (a, b) in enumerate(zip(sc.scene_offsets[:-1], sc.scene_offsets[1:]))])
    e_tau = rel_err(s1["tau"], ref_tau)
    # the MPM part with the GPU's own tau (identical state)
    ref = oracle.reduced_substep({"x": s0["x"], "v": s0["v"], "C": s0["C"]}, P, sc.scene_offsets, sc.X_ref,
                                 sc.mlp, sc.cfg.stress_scale, sc.z0, sc.dz, step=k, tau_override=s1["tau"])
    g = float(np.linalg.norm(sc.cfg.gravity))
    vmax = float(np.max(np.linalg.norm(ref["v"], axis=1)))
    errs = {"x": rel_err(s1["x"], ref["x"]), "v": rel_err(s1["v"], ref["v"], g * sc.cfg.dt),
            "C": rel_err(s1["C"], ref["C"], vmax * sc.cfg.grid_res)}
    return e_tau, errs


@pytest.mark.parametrize("transfer", [0, 2])
@pytest.mark.parametrize("steps_before", [0, 5])
def test_reduced_substep_parity_small(nsf, steps_before, transfer):
    """transfer 2: RPIC (reading #38) in the reduced G2P."""
    sc = scenes.c5_small(n_scenes=3, per_scene=300)
    sc.cfg.transfer = transfer
    if transfer:   # non-zero C so that the skew projection matters
        sc.C = (np.random.default_rng(5).normal(size=sc.C.shape) * 2.0).astype(np.float32)
    e_tau, errs = _reduced_parity(nsf, sc, steps_before)
    assert e_tau <= BAR_MLP, e_tau
    assert all(e <= BAR_STEP for e in errs.values()), errs


def test_reduced_substep_parity_ragged_scenes(nsf):
    """Scenes of different sizes (incl. an empty one) on one handle."""
    sc = scenes.c5_small(n_scenes=4, per_scene=200)
    keep = np.concatenate([np.arange(0, 200), np.arange(200, 200 + 37), np.arange(400, 400), np.arange(600, 800)])
    off = np.array([0, 200, 237, 237, 437], np.int64)
    sc.x, sc.v, sc.C, sc.F = sc.x[keep], sc.v[keep], sc.C[keep], sc.F[keep]
    sc.X_ref = sc.X_ref[keep]
    sc.scene_offsets = off
    e_tau, errs = _reduced_parity(nsf, sc, 2)
    assert e_tau <= BAR_MLP, e_tau
    assert all(e <= BAR_STEP for e in errs.values()), errs


def test_reduced_full_size_sampled(nsf):
    """BASELINE.json config 5 at full size (256 scenes x 2,048 points), in the launch
    configuration bench.py uses: one substep, sampled scenes checked against the
    oracle (the MPM part is exact per scene, so a scene is a valid sample)."""
    sc = scenes.c5()
    sim = make(nsf, sc)
    P = mpm.params_from_config(sc.cfg)
    sim.substep(3)
    s0 = sim.read(nsf.NSF_FIELD_X | nsf.NSF_FIELD_V | nsf.NSF_FIELD_C)
    sim.substep(1)
    sim.sync()
    s1 = sim.read(nsf.NSF_FIELD_X | nsf.NSF_FIELD_V | nsf.NSF_FIELD_C | nsf.NSF_FIELD_TAU)
    sim.close()
    for s in (0, 97, 255):
        a, b = int(sc.scene_offsets[s]), int(sc.scene_offsets[s + 1])
        z = sc.z0[s].astype(np.float64) + 3 * sc.dz[s].astype(np.float64)
        ref_tau = nsf_stress(sc.X_ref[a:b], z, sc.mlp, sc.cfg.stress_scale, "emulate")
        assert rel_err(s1["tau"][a:b], ref_tau) <= BAR_MLP
        ref = oracle.reduced_substep({"x": s0["x"][a:b], "v": s0["v"][a:b], "C": s0["C"][a:b]}, P,
                                     np.array([0, b - a]), sc.X_ref[a:b], sc.mlp, sc.cfg.stress_scale,
                                     sc.z0[s:s + 1], sc.dz[s:s + 1], step=3, tau_override=s1["tau"][a:b])
        assert rel_err(s1["x"][a:b], ref["x"]) <= BAR_STEP
        assert rel_err(s1["v"][a:b], ref["v"], 9.8 * sc.cfg.dt) <= BAR_STEP
        vmax = float(np.max(np.linalg.norm(ref["v"], axis=1)))
        assert rel_err(s1["C"][a:b], ref["C"], vmax * sc.cfg.grid_res) <= BAR_STEP


def test_reduced_zero_network_free_fall(nsf):
    sc = scenes.c5_small(n_scenes=2, per_scene=100)
    for w in sc.mlp["W_bits"]:
        w[...] = 0
    for b in sc.mlp["b"]:
        b[...] = 0
    sim = make(nsf, sc)
    K = 20
    sim.substep(K)
    st = sim.read(nsf.NSF_FIELD_X | nsf.NSF_FIELD_V)
    sim.close()
    g, dt = sc.cfg.gravity[1], sc.cfg.dt
    assert np.allclose(st["v"][:, 1], K * dt * g, atol=1e-5)
    assert np.allclose(st["x"][:, 1], sc.x[:, 1] + dt ** 2 * g * K * (K + 1) / 2, atol=1e-6)
