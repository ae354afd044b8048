"""The reduced model's composed online loop on the GPU (§5):
per latent step n, nsf_mpm_rom_step does (1) sample / integration particles and
network inference at z_n (lines 251-254, 265-269), (2) one MPM substep on N
(lines 255-256), (3) the network inversion of Eq. (10) (lines 257-263).

Five loop steps, each checked against the oracle running the same three steps
from the GPU's own latents (z_n, z_{n-1}) -- teacher forcing, so every step is
judged at the f1 / f2 bars instead of compounding the inversion's intrinsic
sensitivity (DESIGN reading #37):
  * |N_s| equal to the oracle's integration set up to 2 stencil-boundary points;
  * the sample particles' positions after the substep within 1e-3 (relative L2)
    of the oracle's inference + reduced substep on its own N;
  * z_{n+1} reduces the Eq. (10) objective (targets: the GPU's sample positions)
    by the oracle Gauss-Newton step's reduction to within 1e-2 of that reduction,
    or to within the excess that fp32-accumulated evaluations of the same network
    reach, plus a quarter of the objective the oracle's step leaves (reading #37:
    that remainder is the bf16 evaluation noise of g, which two bf16
    implementations of g do not share).
"""
import numpy as np
import pytest

import oracle
import scenes
from oracle import mpm
from oracle.inference import infer_state, integration_set, ordered_points
from oracle.inversion import g_with_tangents
from tests.inv_util import fp32_objective_spread
from tests.parity_util import rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nsf():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2310_17790_b200 as m
    return m


def test_rom_loop_five_steps(nsf):
    n_ref, n_sample, iters, steps = 5000, 64, 2, 5
    sc = scenes.c5_small(n_scenes=3, per_scene=300)
    sc.dz = np.zeros_like(sc.dz)
    ns, r = sc.cfg.n_scenes, sc.z0.shape[1]
    g, l = scenes.deformation_field_near_identity(), scenes.affine_field()
    X_all = scenes.reference_body(n_ref=n_ref).astype(np.float32)
    rng = np.random.default_rng(43)
    sidx = np.stack([rng.choice(n_ref, n_sample, replace=False) for _ in range(ns)]).astype(np.int32)
    P = mpm.params_from_config(sc.cfg)
    grid = (sc.cfg.grid_res,) * 3
    sim = nsf.Simulator(sc.cfg)
    sim.load_scene(sc)
    sim.load_deformation_field(g)
    sim.load_affine_field(l)
    z_n = sc.z0.astype(np.float64)
    # the latent was moving: z_{-1} = z_0 - 0.05 u (|u| = 1 per scene), so the sample
    # particles carry a velocity and the inversion has a real step to take
    u = rng.normal(size=z_n.shape)
    z_prev = (z_n - 0.05 * u / np.linalg.norm(u, axis=1, keepdims=True)).astype(np.float32).astype(np.float64)
    moved = 0.0
    try:
        for step in range(steps):
            z_next, counts = sim.rom_step(X_all, sidx, iters, z_prev=z_prev if step == 0 else None)
            x_gpu = sim.read(nsf.NSF_FIELD_X)["x"]
            off = np.concatenate([[0], np.cumsum(counts)])
            for s in range(ns):
                N_o, _ = integration_set(X_all, sidx[s], z_n[s], g, grid, sc.cfg.dx, mode="emulate")
                assert abs(int(counts[s]) - len(N_o)) <= 2, (step, s, int(counts[s]), len(N_o))
                order = ordered_points(N_o, sidx[s])
                x, v, C = infer_state(X_all[order], z_n[s], z_prev[s], g, l, sc.cfg.dt, mode="emulate")
                out = oracle.reduced_substep({"x": x, "v": v, "C": C}, P, np.array([0, len(order)]), X_all[order],
                                             sc.mlp, sc.cfg.stress_scale, z_n[s][None], np.zeros((1, r)), step=0)
                xs_gpu = x_gpu[off[s]:off[s] + n_sample].astype(np.float64)
                assert rel_err(xs_gpu, out["x"][:n_sample]) <= 1e-3, (step, s)
                # inversion from z_n with the GPU's sample positions as targets
                XS = X_all[sidx[s]]
                zo, f0, fo, spread = fp32_objective_spread(XS, xs_gpu, z_n[s], g, iters)
                fg = float(np.sum((g_with_tangents(XS, z_next[s].astype(np.float64), g, "emulate")[0]
                                   - xs_gpu) ** 2))
                # reading #37: within 1e-2 of the oracle step's reduction or the excess an
                # fp32-accumulated evaluation reaches, plus a quarter of the floor the
                # oracle's step leaves: there the residual is the bf16 evaluation noise of
                # g, and two bf16 implementations of g differ by ~15% of it
                assert fg - fo <= max(1e-2 * (f0 - fo), spread) + 0.25 * fo, (step, s, f0, fo, fg, spread)
                assert fo < 0.5 * f0 and fg < 0.5 * f0, (step, s, f0, fo, fg)   # a real step, both sides
            moved += float(np.linalg.norm(z_next - z_n))
            z_prev, z_n = z_n, z_next.astype(np.float64)
        assert moved > 0.0          # the latents did evolve
    finally:
        sim.close()
