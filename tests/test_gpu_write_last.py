"""v, C and tau are stored only by the last substep of a nsf_mpm_substep(n) call
(inside the fused kernel they only feed the next P2G, PAPER.md
P:173-180, and nothing can read them before the call returns).

A 40-substep call (38 substeps that keep v, C, tau in registers, across the
re-binning at substep 32 and its gathering substep, then one that stores them)
must leave the same state as 40 one-substep calls and as the same call with
NSF_WRITE_EVERY=1, to fp32 reduction-order noise; and the stored v, C, tau must be
those of the stored x, F: one more substep from the read-back state matches the
oracle advancing that state (bar 1e-5) -- stale v, C or tau would not, since the
GPU's next substep uses its grid sums and the oracle the fields read.
"""
import numpy as np
import pytest

import scenes
from tests.parity_util import BAR_STEP, compare, gpu_state, single_step_parity

pytestmark = pytest.mark.gpu

STEPS = 40
NOISE_BAR = 1e-3   # BAR_TRAJ: 40 substeps of fp32 atomics in a different order (as tests/test_gpu_far.py)


@pytest.fixture(scope="module")
def nsf():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2310_17790_b200 as m
    return m


def _scene(model):
    # a block falling at 2 m/s with velocity / C / F noise: every particle changes every substep.
    # von Mises: 1,000 segments of 512 particles (the 3-CTA/SM instantiation with the separate
    # grid-update pass, as C3); the others: 216 segments (2 CTAs/SM, grid update after a barrier)
    if model == scenes.VON_MISES:
        return scenes.block_scene("wl", 128, (44, 40, 44), (84, 80, 84), model, 91, v0=(0.0, -2.0, 0.0),
                                  vnoise=0.3, Fnoise=0.01, Cnoise=0.5)
    return scenes.block_scene("wl", 64, (20, 12, 20), (44, 36, 44), model, 91, keep=60000, v0=(0.0, -2.0, 0.0),
                              vnoise=0.3, Fnoise=0.01, Cnoise=0.5)


def _run(nsf, sc, calls, monkeypatch, write_every=False):
    if write_every:
        monkeypatch.setenv("NSF_WRITE_EVERY", "1")
    else:
        monkeypatch.delenv("NSF_WRITE_EVERY", raising=False)
    sim = nsf.Simulator(sc.cfg)
    sim.load_scene(sc)
    for n in calls:
        sim.substep(n)
    sim.sync()
    return sim


@pytest.mark.parametrize("model", [scenes.FIXED_COROTATED, scenes.VON_MISES, scenes.DRUCKER_PRAGER])
def test_one_call_equals_single_substep_calls(nsf, model, monkeypatch):
    sc = _scene(model)
    sims = {"one call": _run(nsf, sc, [STEPS], monkeypatch),
            "single calls": _run(nsf, sc, [1] * STEPS, monkeypatch),
            "write every": _run(nsf, sc, [STEPS], monkeypatch, write_every=True)}
    try:
        st = {k: gpu_state(s) for k, s in sims.items()}
        for k in ("single calls", "write every"):
            err = compare(st["one call"], st[k], sc.cfg)
            assert max(err.values()) <= NOISE_BAR, (k, err)
        # the stored v, C, tau belong to the stored x, F
        monkeypatch.delenv("NSF_WRITE_EVERY", raising=False)
        err, _, _ = single_step_parity(sims["one call"], sc.cfg, STEPS)
        assert max(err.values()) <= BAR_STEP, err
    finally:
        for s in sims.values():
            s.close()


def test_two_calls_read_between(nsf, monkeypatch):
    """A read between two multi-substep calls sees a complete state, and does not disturb the run."""
    sc = _scene(scenes.VON_MISES)
    a = _run(nsf, sc, [17], monkeypatch)
    b = _run(nsf, sc, [1] * 17, monkeypatch)
    try:
        err = compare(gpu_state(a), gpu_state(b), sc.cfg)
        assert max(err.values()) <= NOISE_BAR, err
        a.substep(23)
        b.substep(23)
        a.sync()
        b.sync()
        err = compare(gpu_state(a), gpu_state(b), sc.cfg)
        assert max(err.values()) <= NOISE_BAR, err
        assert np.isfinite(gpu_state(a)["tau"]).all()
    finally:
        a.close()
        b.close()
