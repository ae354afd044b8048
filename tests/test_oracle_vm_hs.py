"""Pins for the von Mises hardening / softening / damage update of the oracle
(DESIGN readings #30-#32), CPU only.

What pins it (none of these re-call the function under test to make the
expected value):
  - xi = theta = 0 reduces to the perfect-plasticity map, itself pinned by
    test_oracle_constitutive.py (yield surface, idempotence, worked examples);
  - a traceless log strain eps = diag(2c, -c, -c) has |eps_hat| = c sqrt(6), so
    delta_gamma and the hardened / softened yield stress are closed forms;
  - ||eps - proj(eps)||_F = delta_gamma (the radial return moves eps by
    delta_gamma along a unit direction), so softening removes theta delta_gamma;
  - the returned state lies on the yield surface of tau_Y^n (||dev tau|| = tau_Y^n,
    Hencky elasticity), and with hardening a repeated update is elastic;
  - damage: tau_Y reaches 0 -> zero stress, tau_Y stays 0, no return map.
"""
import numpy as np

from oracle.constitutive import (lame, return_map_von_mises, return_map_von_mises_hs,
                                 elastoplastic_update_vm_hs, svd_rotation_safe, tau_hencky)
from oracle import mpm
import scenes

MU, LAM, _ = lame(1e6, 0.3)


def _sigma_traceless(c):
    return np.exp(np.array([[2 * c, -c, -c]]))


def test_zero_coefficients_reduce_to_perfect_plasticity():
    rng = np.random.default_rng(1)
    s = np.exp(rng.normal(0.0, 0.05, (200, 3)))
    tY = 5e4
    Z, tY1, dmg = return_map_von_mises_hs(s, MU, np.full(200, tY), 0.0, 0.0)
    assert np.array_equal(Z, return_map_von_mises(s, MU, tY))
    assert np.all(tY1 == tY) and not dmg.any()


def test_hardening_closed_form():
    c, tY, xi = 0.04, 5e4, 0.3
    dg = c * np.sqrt(6.0) - tY / (2.0 * MU)          # |eps_hat| = c sqrt(6)
    assert dg > 0
    Z, tY1, dmg = return_map_von_mises_hs(_sigma_traceless(c), MU, np.array([tY]), xi, 0.0)
    assert tY1[0] == np.float64(tY1[0]) and abs(tY1[0] - (tY + 2.0 * MU * xi * dg)) <= 1e-9 * tY
    # the projected strain: eps - dg * eps_hat / |eps_hat|
    eps = np.array([2 * c, -c, -c])
    assert np.allclose(np.log(Z[0]), eps - dg * eps / (c * np.sqrt(6.0)), rtol=0, atol=1e-15)
    assert not dmg.any()


def test_softening_removes_theta_delta_gamma():
    rng = np.random.default_rng(2)
    s = np.exp(rng.normal(0.0, 0.04, (500, 3)))
    tY, theta = 2e4, 3e5
    Z, tY1, dmg = return_map_von_mises_hs(s, MU, np.full(500, tY), 0.0, theta)
    eps = np.log(s)
    eh = eps - eps.mean(axis=1, keepdims=True)
    dg = np.linalg.norm(eh, axis=1) - tY / (2.0 * MU)
    proj = dg > 0
    assert proj.sum() > 100 and (~proj).sum() > 50
    expect = np.where(proj, np.maximum(tY - theta * dg, 0.0), tY)
    assert np.allclose(tY1, expect, rtol=1e-12, atol=1e-9)
    # ||eps - log Z||_F equals delta_gamma where projected
    assert np.allclose(np.linalg.norm(eps - np.log(Z), axis=1)[proj], dg[proj], rtol=1e-12)
    assert np.array_equal(dmg, tY1 <= 0.0)


def test_returned_state_on_old_surface_and_hardened_repeat_is_elastic():
    rng = np.random.default_rng(3)
    n = 300
    F = np.eye(3) + rng.normal(0.0, 0.03, (n, 3, 3))
    tY = np.full(n, 1.5e4)
    FE, tau, tY1 = elastoplastic_update_vm_hs(F, MU, LAM, tY, 0.5, 0.0)
    dev = tau - np.trace(tau, axis1=1, axis2=2)[:, None, None] / 3.0 * np.eye(3)
    ndev = np.linalg.norm(dev, axis=(1, 2))
    plastic = tY1 > tY
    assert plastic.sum() > 50
    assert np.allclose(ndev[plastic], tY[plastic], rtol=1e-9)            # on the yield surface of tau_Y^n
    assert np.all(ndev[~plastic] <= tY[~plastic] * (1 + 1e-12))
    FE2, tau2, tY2 = elastoplastic_update_vm_hs(FE, MU, LAM, tY1, 0.5, 0.0)
    assert np.array_equal(tY2, tY1)                                       # inside the hardened surface
    assert np.allclose(FE2, FE, rtol=0, atol=1e-13)


def test_damage_zero_stress_and_persistent():
    c = 0.03
    s = _sigma_traceless(c)
    tY = 1e4
    dg = c * np.sqrt(6.0) - tY / (2.0 * MU)
    theta = 2.0 * tY / dg                                  # softening drives tau_Y below zero
    U = np.eye(3)[None]
    F = U * s[:, None, :]
    FE, tau, tY1 = elastoplastic_update_vm_hs(F, MU, LAM, np.array([tY]), 0.0, theta)
    assert tY1[0] == 0.0 and np.all(tau == 0.0)
    # damaged: no return map (F_E = F_trial), zero stress, tau_Y stays 0
    F2 = np.eye(3)[None] + 0.05
    FE2, tau2, tY2 = elastoplastic_update_vm_hs(F2, MU, LAM, tY1, 0.0, theta)
    assert np.allclose(FE2, F2, rtol=0, atol=1e-14) and np.all(tau2 == 0.0) and tY2[0] == 0.0
    # without softening a zero yield stress is perfect plasticity, not damage: the
    # deviatoric strain is returned entirely, the volumetric stress stays
    F3 = F * np.exp(0.01)
    FE3, tau3, tY3 = elastoplastic_update_vm_hs(F3, MU, LAM, np.array([0.0]), 0.2, 0.0)
    K = LAM + 2.0 * MU / 3.0
    assert np.allclose(tau3[0], 3.0 * 0.01 * K * np.eye(3), rtol=1e-9, atol=1e-6) and tY3[0] > 0.0


def test_elastic_update_keeps_yield_stress():
    rng = np.random.default_rng(4)
    F = np.eye(3) + rng.normal(0.0, 1e-4, (50, 3, 3))
    tY = np.full(50, 5e4)
    FE, tau, tY1 = elastoplastic_update_vm_hs(F, MU, LAM, tY, 0.4, 1e5)
    assert np.array_equal(tY1, tY)
    U, s, V = svd_rotation_safe(F)
    assert np.allclose(tau, tau_hencky(U, s, MU, LAM), rtol=1e-12, atol=1e-9)


def test_substep_carries_yield_stress():
    sc = scenes.block_scene("vmhs", 32, (12, 12, 12), (16, 16, 16), scenes.VON_MISES, 7,
                            Fnoise=0.02, yield_stress=1.5e4, hardening=0.3)
    P = mpm.params_from_config(sc.cfg)
    st = {"x": sc.x, "v": sc.v, "C": sc.C, "F": sc.F, "tau": mpm.initial_tau(sc.F, P)}
    out = mpm.substep(st, P, 0)
    assert out["tau_Y"].shape == (sc.n,)
    assert np.all(out["tau_Y"] >= 1.5e4) and np.any(out["tau_Y"] > 1.5e4)
    # same substep without the per-particle law: identical kinematics, perfect plasticity
    P0 = mpm.params_from_config(sc.cfg)
    P0.hardening = 0.0
    out0 = mpm.substep(st, P0, 0)
    assert np.array_equal(out0["x"], out["x"]) and "tau_Y" not in out0
    assert np.allclose(out0["F"], out["F"], rtol=0, atol=1e-15)   # hardening acts from the next update on
