"""Pins for oracle/constitutive.py against closed forms, worked examples,
energy finite differences and an independent library routine (CPU only)."""
import json
import os

import numpy as np
import pytest

import oracle
from oracle.constitutive import (lame, dp_alpha, svd_rotation_safe, tau_fixed_corotated,
                                 tau_hencky, return_map_drucker_prager,
                                 return_map_von_mises, elastoplastic_update)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def rand_rot(rng, n):
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    return np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
        np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
        np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1)], 1)


@pytest.mark.parametrize("ex", GOLD["lame"])
def test_lame_worked(ex):
    mu, lam, kappa = lame(ex["E"], ex["nu"])
    assert mu == pytest.approx(ex["mu"], rel=1e-15)
    if "lam" in ex:
        assert lam == pytest.approx(ex["lam"], rel=1e-15, abs=1e-300)
        assert kappa == pytest.approx(ex["kappa"], rel=1e-15)


def test_lame_domain():
    for E, nu in [(0.0, 0.3), (-1.0, 0.3), (1.0, 0.5), (1.0, -0.1)]:
        with pytest.raises(ValueError):
            lame(E, nu)


def test_dp_alpha_golden():
    ex = GOLD["drucker_prager_alpha"][0]
    assert dp_alpha(ex["phi_deg"]) == pytest.approx(ex["alpha"], rel=1e-14)


def test_svd_rotation_safe_vs_eigh():
    """Reconstruction, det U = det V = +1, and sigma^2 = eigenvalues of F^T F from an
    independent routine (symmetric eigensolver), including inverted F."""
    rng = np.random.default_rng(0)
    F = np.eye(3) + rng.normal(scale=0.7, size=(500, 3, 3))
    U, s, V = svd_rotation_safe(F)
    rec = np.einsum("nij,nj,nkj->nik", U, s, V)
    assert np.max(np.abs(rec - F)) < 1e-12
    assert np.allclose(np.linalg.det(U), 1.0) and np.allclose(np.linalg.det(V), 1.0)
    assert np.allclose(U @ np.swapaxes(U, 1, 2), np.eye(3), atol=1e-12)
    ev = np.linalg.eigh(np.swapaxes(F, 1, 2) @ F)[0][:, ::-1]
    assert np.allclose(np.sort(s ** 2, axis=1)[:, ::-1], ev, rtol=1e-10, atol=1e-12)
    neg = np.linalg.det(F) < 0
    assert neg.any()
    assert np.all(s[neg, 2] < 0) and np.all(s[~neg, 2] >= 0)


def test_svd_spec_examples():
    U, s, V = svd_rotation_safe(np.diag([-2.0, 1.0, 1.0])[None])
    assert np.allclose(np.abs(s), [2, 1, 1])
    assert s[0, 2] < 0 and np.isclose(np.linalg.det(U[0]), 1) and np.isclose(np.linalg.det(V[0]), 1)


@pytest.mark.parametrize("ex", GOLD["fixed_corotated"])
def test_fc_worked(ex):
    tau = tau_fixed_corotated(np.array(ex["F"], float)[None], ex["mu"], ex["lam"])[0]
    assert np.allclose(tau, ex["tau"], atol=1e-13)


def test_fc_rotation_invariance_and_equivariance():
    rng = np.random.default_rng(1)
    R = rand_rot(rng, 50)
    assert np.max(np.abs(tau_fixed_corotated(R, 3.0, 2.0))) < 1e-12
    F = np.eye(3) + 0.3 * rng.normal(size=(50, 3, 3))
    t1 = tau_fixed_corotated(R @ F, 3.0, 2.0)
    t2 = R @ tau_fixed_corotated(F, 3.0, 2.0) @ np.swapaxes(R, 1, 2)
    assert np.allclose(t1, t2, atol=1e-11)
    assert np.allclose(t1, np.swapaxes(t1, 1, 2), atol=1e-12)


def _fd_tau(psi, F, h=1e-6):
    """tau = dpsi/dF F^T by central differences."""
    P = np.zeros((3, 3))
    for i in range(3):
        for j in range(3):
            E = np.zeros((3, 3))
            E[i, j] = h
            P[i, j] = (psi(F + E) - psi(F - E)) / (2 * h)
    return P @ F.T


def test_fc_energy_fd():
    """PAPER.md 149: tau = (dpsi/dF) F^T with psi = mu |F - R|^2 + lam/2 (J-1)^2."""
    rng = np.random.default_rng(2)
    mu, lam = 1.7, 2.3

    def psi(F):
        U, s, Vt = np.linalg.svd(F)
        if np.linalg.det(U) * np.linalg.det(Vt) < 0:
            U[:, 2] *= -1
            s[2] *= -1
        R = U @ Vt
        return mu * np.sum((F - R) ** 2) + 0.5 * lam * (np.linalg.det(F) - 1) ** 2

    for _ in range(20):
        F = np.eye(3) + 0.3 * rng.normal(size=(3, 3))
        if np.linalg.det(F) < 0.2:
            continue
        assert np.allclose(tau_fixed_corotated(F[None], mu, lam)[0], _fd_tau(psi, F), atol=2e-7)


@pytest.mark.parametrize("ex", GOLD["hencky"])
def test_hencky_worked(ex):
    tau = tau_hencky(np.eye(3)[None], np.array(ex["sigma"])[None], ex["mu"], ex["lam"])[0]
    assert np.allclose(np.diag(tau), ex["tau_diag"], atol=1e-13)
    assert np.allclose(tau - np.diag(np.diag(tau)), 0)


def test_hencky_energy_fd():
    """tau = dpsi/dF F^T, psi = mu |log Sigma|^2 + lam/2 (sum log Sigma)^2; catches the
    U..V^T transposition in PAPER.md line 524 (reading #3)."""
    rng = np.random.default_rng(3)
    mu, lam = 1.3, 0.9

    def psi(F):
        s = np.linalg.svd(F, compute_uv=False)
        e = np.log(s)
        return mu * np.sum(e ** 2) + 0.5 * lam * np.sum(e) ** 2

    for _ in range(20):
        F = np.eye(3) + 0.3 * rng.normal(size=(3, 3))
        if np.linalg.det(F) < 0.2:
            continue
        U, s, V = svd_rotation_safe(F[None])
        assert np.allclose(tau_hencky(U, s, mu, lam)[0], _fd_tau(psi, F), atol=2e-7)


def _eps(Z):
    return np.log(Z)


def test_dp_branches_and_cone():
    rng = np.random.default_rng(4)
    mu, lam = lame(3.5e5, 0.3)[:2]
    alpha = dp_alpha(30.0)
    # expansion: tr eps > 0 -> Z = 1 (F_E = U V^T, stress free)
    s = np.array([[1.1, 1.05, 1.0]])
    assert np.allclose(return_map_drucker_prager(s, mu, lam, alpha), 1.0)
    # F = I -> I
    assert np.allclose(return_map_drucker_prager(np.ones((1, 3)), mu, lam, alpha), 1.0)
    # random compressive states: projected ones land on the cone; tr preserved
    s = np.exp(rng.normal(scale=0.05, size=(2000, 3)) - 0.02)
    Z = return_map_drucker_prager(s, mu, lam, alpha)
    e, eZ = np.log(s), _eps(Z)
    tr = e.sum(1)
    ehat = e - tr[:, None] / 3
    dg = np.linalg.norm(ehat, axis=1) + alpha * (3 * lam + 2 * mu) * tr / (2 * mu)
    proj = (tr <= 0) & (dg > 0)
    el = (tr <= 0) & (dg <= 0)
    assert proj.sum() > 100 and el.sum() > 10
    trZ = eZ.sum(1)
    ehZ = eZ - trZ[:, None] / 3
    cone = np.linalg.norm(ehZ, axis=1) + alpha * (3 * lam + 2 * mu) * trZ / (2 * mu)
    assert np.max(np.abs(cone[proj])) < 1e-14
    assert np.allclose(trZ[proj], tr[proj], atol=1e-15)
    assert np.array_equal(Z[el], s[el])
    # idempotent
    Z2 = return_map_drucker_prager(Z[~(tr > 0)], mu, lam, alpha)
    assert np.allclose(Z2, Z[~(tr > 0)], rtol=1e-13)


def test_dp_clamp_inverted():
    mu, lam = lame(1.0, 0.3)[:2]
    Z = return_map_drucker_prager(np.array([[0.5, 0.4, -0.3]]), mu, lam, dp_alpha(30))
    assert np.all(np.isfinite(Z))


def test_vm_return_on_yield_surface():
    rng = np.random.default_rng(5)
    E, nu, tY = 1e6, 0.3, 5e4
    mu, lam = lame(E, nu)[:2]
    s = np.exp(rng.normal(scale=0.1, size=(2000, 3)))
    Z = return_map_von_mises(s, mu, tY)
    U = np.broadcast_to(np.eye(3), (2000, 3, 3))
    tau = tau_hencky(U, Z, mu, lam)
    dev = tau - np.trace(tau, axis1=1, axis2=2)[:, None, None] / 3 * np.eye(3)
    nd = np.linalg.norm(dev, axis=(1, 2))
    tau0 = tau_hencky(U, s, mu, lam)
    dev0 = tau0 - np.trace(tau0, axis1=1, axis2=2)[:, None, None] / 3 * np.eye(3)
    inside = np.linalg.norm(dev0, axis=(1, 2)) <= tY
    assert inside.sum() > 50 and (~inside).sum() > 50
    assert np.allclose(nd[~inside], tY, rtol=1e-12)            # on the surface
    assert np.array_equal(Z[inside], s[inside])                 # unchanged inside
    assert np.allclose(np.log(Z).sum(1), np.log(s).sum(1), atol=1e-14)   # tr eps preserved
    assert np.allclose(return_map_von_mises(Z, mu, tY), Z, rtol=1e-13)   # idempotent
    # tau_Y = 0 -> deviatoric log strain vanishes
    Z0 = return_map_von_mises(s, mu, 0.0)
    e0 = np.log(Z0)
    assert np.allclose(e0 - e0.mean(1, keepdims=True), 0, atol=1e-15)


def test_vm_paper_denominator_misses_surface():
    """Reading #4: with |eps| in the denominator (as PAPER.md 542 prints) the return
    misses the yield surface; with |eps_hat| it lands on it.  Documents the choice."""
    mu, lam = lame(1e6, 0.3)[:2]
    tY = 5e4
    s = np.array([[1.3, 0.8, 0.95]])
    e = np.log(s)
    eh = e - e.mean()
    dg = np.linalg.norm(eh) - tY / (2 * mu)
    Zp = np.exp(e - dg * eh / np.linalg.norm(e))
    tau = tau_hencky(np.eye(3)[None], Zp, mu, lam)[0]
    dev = tau - np.trace(tau) / 3 * np.eye(3)
    assert abs(np.linalg.norm(dev) - tY) > 1.0   # 43.6 Pa off for this state
    Z = return_map_von_mises(s, mu, tY)
    tau = tau_hencky(np.eye(3)[None], Z, mu, lam)[0]
    assert np.isclose(np.linalg.norm(tau - np.trace(tau) / 3 * np.eye(3)), tY, rtol=1e-12)


def test_elastoplastic_update_models():
    rng = np.random.default_rng(6)
    F = np.eye(3) + 0.05 * rng.normal(size=(100, 3, 3))
    mu, lam = lame(1e6, 0.3)[:2]
    FE, tau = elastoplastic_update(F, 0, mu, lam)
    assert np.array_equal(FE, F)
    for model in (1, 2):
        FE, tau = elastoplastic_update(F, model, mu, lam, dp_alpha(30), 5e4)
        assert np.allclose(tau, np.swapaxes(tau, 1, 2), atol=1e-9)
        # elastic particles keep F
        U, s, V = svd_rotation_safe(F)
        Z = return_map_von_mises(s, mu, 5e4) if model == 2 else \
            return_map_drucker_prager(s, mu, lam, dp_alpha(30))
        same = np.all(Z == s, axis=1)
        assert np.allclose(FE[same], F[same], atol=1e-14)


def test_stvk_as_printed_is_elastic_hencky():
    """Model 4, the appendix's "StVK elasticity": no return map
    (F^E = F_trial even far beyond any yield surface), tau = dpsi/dF F^T with the Hencky
    energy psi = mu |log Sigma|^2 + lam/2 (sum log Sigma)^2 (U^T per reading #3), zero at
    F = I, and isotropic: tau(Q F) = Q tau(F) Q^T for a rotation Q."""
    from oracle.constitutive import elastoplastic_update
    rng = np.random.default_rng(11)
    mu, lam = 1.3, 0.9

    def psi(F):
        s = np.linalg.svd(F, compute_uv=False)
        e = np.log(s)
        return mu * np.sum(e ** 2) + 0.5 * lam * np.sum(e) ** 2

    FE, tau0 = elastoplastic_update(np.eye(3)[None], 4, mu, lam)
    assert np.allclose(tau0, 0.0, atol=1e-14)
    for _ in range(12):
        F = np.eye(3) + 0.4 * rng.normal(size=(3, 3))
        if np.linalg.det(F) < 0.2:
            continue
        FE, tau = elastoplastic_update(F[None], 4, mu, lam)
        assert np.array_equal(FE[0], F)
        assert np.allclose(tau[0], _fd_tau(psi, F), atol=2e-7)
        q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        if np.linalg.det(q) < 0:
            q[:, 0] *= -1
        _, tq = elastoplastic_update((q @ F)[None], 4, mu, lam)
        assert np.allclose(tq[0], q @ tau[0] @ q.T, atol=1e-12)


# ---------------------------------------------------------------------------
# Herschel-Bulkley (reading #39)
from oracle.constitutive import return_map_herschel_bulkley, tau_herschel_bulkley  # noqa: E402

HB_MU, HB_KAPPA, HB_SY, HB_DT = 3.0e4, 8.0e4, 2.0e3, 1.0e-4


def _hb_trials(rng, n, scale=0.3):
    return np.eye(3) + rng.normal(size=(n, 3, 3)) * scale


def _dev_norm(t):
    dev = t - (np.trace(t, axis1=1, axis2=2) / 3.0)[:, None, None] * np.eye(3)
    return np.linalg.norm(dev, axis=(1, 2)), dev


def test_hb_stress_is_energy_derivative():
    """tau = kappa/2 (J^2 - 1) I + mu dev(bbar) is (dpsi/dF) F^T of the compressible
    neo-Hookean energy psi = mu/2 (tr(bbar) - 3) + kappa/2 ((J^2 - 1)/2 - ln J)
    (central differences on random F with J > 0)."""
    rng = np.random.default_rng(21)
    F = _hb_trials(rng, 20, 0.2)
    F = F[np.linalg.det(F) > 0.2]
    mu, kappa = 1.3, 2.9

    def psi(G):
        J = np.linalg.det(G)
        b = G @ G.T
        return mu / 2 * (np.trace(b) * J ** (-2.0 / 3.0) - 3.0) + kappa / 2 * ((J * J - 1) / 2 - np.log(J))
    h = 1e-6
    for Fk, tk in zip(F, tau_herschel_bulkley(F, mu, kappa)):
        P = np.zeros((3, 3))
        for i in range(3):
            for j in range(3):
                E = np.zeros((3, 3))
                E[i, j] = h
                P[i, j] = (psi(Fk + E) - psi(Fk - E)) / (2 * h)
        assert np.allclose(P @ Fk.T, tk, rtol=1e-6, atol=1e-7)


def test_hb_inside_yield_and_infinite_viscosity_unchanged():
    rng = np.random.default_rng(22)
    F = _hb_trials(rng, 300, 0.002)                     # small strain: s < sqrt(2/3) sigma_Y
    st, _ = _dev_norm(tau_herschel_bulkley(F, HB_MU, HB_KAPPA))
    assert np.all(st < np.sqrt(2 / 3) * HB_SY)
    FE, _ = return_map_herschel_bulkley(F, HB_MU, HB_KAPPA, HB_SY, 0.0, HB_DT)
    assert np.array_equal(FE, F)
    F = _hb_trials(rng, 300)
    FE, _ = return_map_herschel_bulkley(F, HB_MU, HB_KAPPA, HB_SY, 1e30, HB_DT)   # eta -> infinity
    assert np.allclose(FE, F, rtol=0, atol=1e-12)


def test_hb_zero_viscosity_lands_on_yield_surface():
    """eta = 0: s = sqrt(2/3) sigma_Y exactly; the flow is isochoric (det F^E = det
    F_trial), keeps the deviator's direction and the rotation, and the map is
    idempotent."""
    rng = np.random.default_rng(23)
    F = _hb_trials(rng, 500)
    F[np.linalg.det(F) < 0, :, 0] *= -1.0                 # include only J > 0 here
    st, dev_t = _dev_norm(tau_herschel_bulkley(F, HB_MU, HB_KAPPA))
    plastic = st > np.sqrt(2 / 3) * HB_SY
    assert plastic.mean() > 0.9
    FE, tau = return_map_herschel_bulkley(F, HB_MU, HB_KAPPA, HB_SY, 0.0, HB_DT)
    sn, dev_n = _dev_norm(tau)
    assert np.allclose(sn[plastic], np.sqrt(2 / 3) * HB_SY, rtol=1e-10)
    assert np.allclose(np.linalg.det(FE), np.linalg.det(F), rtol=1e-12)
    cos = np.einsum("pij,pij->p", dev_n, dev_t) / (sn * st)
    assert np.allclose(cos[plastic], 1.0, atol=1e-12)
    # same rotation: F^E F_trial^-1 is symmetric positive definite (a pure stretch)
    Sx = FE @ np.linalg.inv(F)
    assert np.allclose(Sx, np.swapaxes(Sx, 1, 2), atol=1e-10)
    FE2, tau2 = return_map_herschel_bulkley(FE, HB_MU, HB_KAPPA, HB_SY, 0.0, HB_DT)
    assert np.allclose(FE2, FE, atol=1e-10) and np.allclose(tau2, tau, rtol=1e-9, atol=1e-6)


def test_hb_viscous_relaxation_magnitude():
    """0 < eta < inf: ||dev tau(F^E)|| = s - (s - sqrt(2/3) sigma_Y) / (1 + eta/(2 mu dt))
    (PAPER.md line 548), between the yield surface and the trial value."""
    rng = np.random.default_rng(24)
    F = _hb_trials(rng, 300)
    F[np.linalg.det(F) < 0, :, 0] *= -1.0
    eta = 2.0 * HB_MU * HB_DT * 1.5                      # relaxation factor 1 / 2.5
    st, _ = _dev_norm(tau_herschel_bulkley(F, HB_MU, HB_KAPPA))
    y = np.sqrt(2 / 3) * HB_SY
    _, tau = return_map_herschel_bulkley(F, HB_MU, HB_KAPPA, HB_SY, eta, HB_DT)
    sn, _ = _dev_norm(tau)
    p = st > y
    assert np.allclose(sn[p], st[p] - (st[p] - y) / 2.5, rtol=1e-10)
    assert np.all((sn[p] > y) & (sn[p] < st[p]))


def test_hb_rotation_equivariance():
    rng = np.random.default_rng(25)
    F = _hb_trials(rng, 100)
    A = rng.normal(size=(100, 3, 3))
    Q, R = np.linalg.qr(A)
    Q = Q * np.sign(np.diagonal(R, axis1=1, axis2=2))[:, None, :]
    Q[np.linalg.det(Q) < 0, :, 0] *= -1.0
    FE, tau = return_map_herschel_bulkley(F, HB_MU, HB_KAPPA, HB_SY, 0.3, HB_DT)
    FEr, taur = return_map_herschel_bulkley(Q @ F, HB_MU, HB_KAPPA, HB_SY, 0.3, HB_DT)
    assert np.allclose(FEr, Q @ FE, atol=1e-10)
    assert np.allclose(taur, Q @ tau @ np.swapaxes(Q, 1, 2), rtol=1e-9, atol=1e-5)
