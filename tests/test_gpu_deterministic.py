"""Deterministic mode (nsf_material.deterministic = 1): P2G reduced in 64-bit
fixed point, so a substep does not depend on the order in which particles are
reduced.  Checks: parity with the oracle (same 1e-5 bar as the default mode),
and bitwise-identical results when the same particles are loaded in a shuffled
order (a different storage order, hence a different reduction order)."""
import copy

import numpy as np
import pytest

import scenes
from oracle import mpm
from tests.parity_util import BAR_STEP, gpu_state, single_step_parity
from tests.test_gpu_parity import small_scenes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nsf():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2310_17790_b200 as m
    return m


def det(sc):
    sc = copy.deepcopy(sc)
    sc.cfg.deterministic = 1
    return sc


@pytest.mark.parametrize("name", ["C1spin", "FC_ragged", "DP", "VM", "VM_gradw", "FC_rpic", "HB"])
def test_deterministic_parity(nsf, name):
    sc = det(small_scenes()[name])
    sim = nsf.Simulator(sc.cfg)
    sim.load_scene(sc)
    sim.substep(3)
    errs, _, _ = single_step_parity(sim, sc.cfg, 3)
    sim.close()
    assert all(e <= BAR_STEP for e in errs.values()), errs


def _run(nsf, sc, order, k):
    s = copy.deepcopy(sc)
    s.x, s.v, s.C, s.F = s.x[order], s.v[order], s.C[order], s.F[order]
    sim = nsf.Simulator(s.cfg)
    sim.load_scene(s)
    sim.substep(k)
    sim.sync()
    out = sim.read()
    sim.close()
    inv = np.empty_like(order)
    inv[order] = np.arange(len(order))
    return {f: np.asarray(a)[inv] for f, a in out.items()}


@pytest.mark.parametrize("name", ["FC_ragged", "VM"])
def test_bitwise_independent_of_particle_order(nsf, name):
    sc = det(small_scenes()[name])
    n = sc.n
    a = _run(nsf, sc, np.arange(n), 40)
    b = _run(nsf, sc, np.random.default_rng(5).permutation(n), 40)
    for f in a:
        assert np.array_equal(a[f].view(np.uint32), b[f].view(np.uint32)), f


def test_deterministic_reduced(nsf):
    """The reduced model in deterministic mode: repeatable bit for bit and within
    the reduced-substep parity bar of the default mode's oracle check."""
    import oracle
    sc = scenes.c5_small(n_scenes=2, per_scene=300)
    sc.cfg.deterministic = 1
    outs = []
    for _ in range(2):
        sim = nsf.Simulator(sc.cfg)
        sim.load_scene(sc)
        r0 = sim.read(nsf.NSF_FIELD_X | nsf.NSF_FIELD_V | nsf.NSF_FIELD_C)
        sim.substep(1)
        sim.sync()
        r1 = sim.read(nsf.NSF_FIELD_X | nsf.NSF_FIELD_V | nsf.NSF_FIELD_C | nsf.NSF_FIELD_TAU)
        sim.close()
        outs.append(r1)
    for f in outs[0]:
        assert np.array_equal(outs[0][f].view(np.uint32), outs[1][f].view(np.uint32)), f
    P = mpm.params_from_config(sc.cfg)
    ref = oracle.reduced_substep(r0, P, sc.scene_offsets, sc.X_ref, sc.mlp, sc.cfg.stress_scale, sc.z0, sc.dz,
                                 step=0, tau_override=outs[0]["tau"])
    e = np.linalg.norm(outs[0]["x"] - ref["x"]) / np.linalg.norm(ref["x"])
    assert e <= BAR_STEP, e


def test_two_scenes_equal_one_scene_bitwise(nsf):
    """Full-order model with n_scenes = 2 (block keys carry the scene): two copies
    of a scene on one handle reproduce the single-scene run bit for bit
    (deterministic mode), each copy on its own grid."""
    base = det(small_scenes()["FC_ragged"])
    one = _run(nsf, base, np.arange(base.n), 20)
    two = copy.deepcopy(base)
    two.cfg.n_scenes = 2
    two.x = np.concatenate([base.x, base.x])
    two.v = np.concatenate([base.v, base.v])
    two.C = np.concatenate([base.C, base.C])
    two.F = np.concatenate([base.F, base.F])
    two.scene_offsets = np.array([0, base.n, 2 * base.n], np.int64)
    both = _run(nsf, two, np.arange(two.n), 20)
    for f in one:
        for s in range(2):
            part = both[f][s * base.n:(s + 1) * base.n]
            assert np.array_equal(part.view(np.uint32), one[f].view(np.uint32)), (f, s)


def test_two_scenes_fused_parity(nsf):
    """The fused (default) pipeline with two scenes: each scene matches the oracle
    of its own particles."""
    from tests.parity_util import compare, voigt_to_mat
    base = small_scenes()["VM"]
    two = copy.deepcopy(base)
    two.cfg.n_scenes = 2
    rng = np.random.default_rng(3)
    keep = np.sort(rng.choice(base.n, base.n // 2, replace=False))
    two.x = np.concatenate([base.x, base.x[keep]])
    two.v = np.concatenate([base.v, -base.v[keep]])
    two.C = np.concatenate([base.C, base.C[keep]])
    two.F = np.concatenate([base.F, base.F[keep]])
    two.scene_offsets = np.array([0, base.n, base.n + len(keep)], np.int64)
    sim = nsf.Simulator(two.cfg)
    sim.load_scene(two)
    sim.substep(5)
    s0 = gpu_state(sim)
    sim.substep(1)
    sim.sync()
    s1 = gpu_state(sim)
    sim.close()
    P = mpm.params_from_config(base.cfg)
    for a, b in zip(two.scene_offsets[:-1], two.scene_offsets[1:]):
        ref = mpm.substep({k: s0[k][a:b] for k in ("x", "v", "C", "F", "tau")}, P, 5)
        got = {k: s1[k][a:b] for k in ("x", "v", "C", "F", "tau")}
        errs = compare(got, ref, base.cfg)
        assert all(e <= BAR_STEP for e in errs.values()), errs
