"""Constitutive models and return maps, fp64, batched over a leading axis.

Each function follows PAPER.md's appendix "Elasticity and plasticity details"
(lines 502-545) in its own notation; corrections of garbled passages are the
SURVEY.md §8(c) readings, recorded in DESIGN.md:
  #2  fixed-corotated volumetric term is lambda (J-1) J * I
  #3  Hencky ("StVK", line 524) is tau = U diag(2 mu eps + lambda sum(eps)) U^T
  #4  von Mises projection divides by ||eps_hat|| (line 542 prints ||eps||)
  #5  Drucker-Prager and von Mises use Hencky elasticity
  #6  d = 3 in the Drucker-Prager delta-gamma
  #21 rotation-safe SVD (det U = det V = +1, sign folded into sigma_3);
      log-strain models clamp sigma >= 1e-4 before the log.
  #39 Herschel-Bulkley (lines 546-552): the deviatoric relaxation acts on
      s = mu dev(bbar), bbar = det(b)^(-1/3) b; the elastic state keeps the
      rotation and J of F_trial, and bbar_new = s_new / mu + I_bar 1 with I_bar
      chosen so that det(bbar_new) = 1 (isochoric plastic flow).
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
import numpy as np

SIGMA_FLOOR = 1e-4   # reading #21


def lame(E, nu):
    """mu_hat = E/(2(1+nu)), lambda = E nu/((1+nu)(1-2nu)),
    kappa = E/(3(1-2nu))."""
    E = float(E)
    nu = float(nu)
    if not (E > 0.0 and 0.0 <= nu < 0.5):
        raise ValueError("parameter domain: E > 0, 0 <= nu < 0.5")
    mu = E / (2.0 * (1.0 + nu))
    lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    kappa = E / (3.0 * (1.0 - 2.0 * nu))
    return mu, lam, kappa


def dp_alpha(friction_angle_deg):
    """alpha = sqrt(2/3) * 2 sin(phi_f) / (3 - sin(phi_f))."""
    s = np.sin(np.deg2rad(float(friction_angle_deg)))
    return np.sqrt(2.0 / 3.0) * 2.0 * s / (3.0 - s)


def svd_rotation_safe(F):
    """F = U diag(sigma) V^T with det U = det V = +1 (reading #21).

    A library primitive (LAPACK via numpy) is the step; the sign fix folds any
    reflection of U or V into sigma_3 (the smallest singular value), so sigma_3
    may be negative when det F < 0.
    """
    F = np.asarray(F, dtype=np.float64)
    U, s, Vh = np.linalg.svd(F)
    V = np.swapaxes(Vh, -1, -2).copy()
    U = U.copy()
    s = s.copy()
    du = np.linalg.det(U) < 0
    U[du, :, 2] *= -1.0
    s[du, 2] *= -1.0
    dv = np.linalg.det(V) < 0
    V[dv, :, 2] *= -1.0
    s[dv, 2] *= -1.0
    return U, s, V


def _diag_sandwich(A, d, B):
    """A diag(d) B^T for batched 3x3 A, B and (n,3) d."""
    return np.einsum("nij,nj,nkj->nik", A, d, B)


def tau_fixed_corotated(F, mu, lam):
    """PAPER.md line 518 (+ reading #2): tau = 2 mu (F - R) F^T + lambda (J-1) J I,
    R = U V^T from the SVD of F (line 520)."""
    F = np.asarray(F, dtype=np.float64)
    U, s, V = svd_rotation_safe(F)
    R = U @ np.swapaxes(V, -1, -2)
    J = s[:, 0] * s[:, 1] * s[:, 2]
    tau = 2.0 * mu * (F - R) @ np.swapaxes(F, -1, -2)
    tau += (lam * (J - 1.0) * J)[:, None, None] * np.eye(3)
    return tau


def tau_hencky(U, sigma, mu, lam):
    """PAPER.md line 524 with reading #3: tau = U diag(2 mu eps + lambda sum(eps) 1) U^T,
    eps = log(Sigma) (Sigma clamped at 1e-4, reading #21)."""
    eps = np.log(np.maximum(sigma, SIGMA_FLOOR))
    d = 2.0 * mu * eps + lam * eps.sum(axis=1, keepdims=True)
    return _diag_sandwich(U, d, U)


def return_map_drucker_prager(sigma, mu, lam, alpha):
    """PAPER.md lines 528-536 (Klar et al. 2016): returns Z(Sigma).

      Z = 1                               if sum(eps) > 0
      Z = Sigma                           if delta_gamma <= 0 and sum(eps) <= 0
      Z = exp(eps - dg * eps_hat/|eps_hat|) otherwise
      delta_gamma = |eps_hat| + alpha (d lambda + 2 mu) sum(eps) / (2 mu), d = 3.
    """
    s = np.maximum(np.asarray(sigma, dtype=np.float64), SIGMA_FLOOR)
    eps = np.log(s)
    tr = eps.sum(axis=1)
    eps_hat = eps - tr[:, None] / 3.0
    nrm = np.linalg.norm(eps_hat, axis=1)
    dg = nrm + alpha * (3.0 * lam + 2.0 * mu) * tr / (2.0 * mu)
    Z = s.copy()
    expand = tr > 0.0
    proj = (~expand) & (dg > 0.0)
    Z[expand] = 1.0
    if np.any(proj):
        Z[proj] = np.exp(eps[proj] - (dg[proj] / nrm[proj])[:, None] * eps_hat[proj])
    return Z


def return_map_von_mises(sigma, mu, tau_Y):
    """PAPER.md lines 538-545 with reading #4: returns Z(Sigma).

      delta_gamma = |eps_hat|_F - tau_Y/(2 mu)
      Z = Sigma                            if delta_gamma <= 0
      Z = exp(eps - dg * eps_hat/|eps_hat|) otherwise
    (With Hencky elasticity, |tau - sum(tau)/3| <= tau_Y is exactly dg <= 0.)
    """
    s = np.maximum(np.asarray(sigma, dtype=np.float64), SIGMA_FLOOR)
    eps = np.log(s)
    tr = eps.sum(axis=1)
    eps_hat = eps - tr[:, None] / 3.0
    nrm = np.linalg.norm(eps_hat, axis=1)
    dg = nrm - tau_Y / (2.0 * mu)
    Z = s.copy()
    proj = dg > 0.0
    if np.any(proj):
        Z[proj] = np.exp(eps[proj] - (dg[proj] / nrm[proj])[:, None] * eps_hat[proj])
    return Z


def return_map_von_mises_hs(sigma, mu, tau_Y, hardening=0.0, softening=0.0):
    """PAPER.md line 545, von Mises with a per-particle yield stress (readings #30-#32).

    tau_Y: (n,) yield stress of each particle at t_n.  For a live particle
    (tau_Y > 0) the return map is return_map_von_mises with that tau_Y; then
      hardening:  tau_Y^{n+1} = tau_Y^n + 2 mu xi delta_gamma
      softening:  tau_Y^{n+1} = tau_Y^n - theta ||eps - proj(eps)||_F
    (both applied when both coefficients are set), with eps = log(Sigma) and
    proj(eps) = log(Z), only where the map projects (delta_gamma > 0).  "When
    tau_Y reaches zero, the material is considered damaged and its Lame parameters
    are set to zero": with softening (theta > 0), tau_Y^{n+1} <= 0 -> 0 and the
    particle is damaged from this update on: it keeps Z = Sigma (no return map;
    mu = 0 leaves delta_gamma undefined) and zero stress (the caller zeroes tau
    where the returned `damaged` is set).  Without softening tau_Y only grows
    (a zero initial yield stress is perfect plasticity, not damage).
    Returns (Z, tau_Y_new, damaged).
    """
    s = np.maximum(np.asarray(sigma, dtype=np.float64), SIGMA_FLOOR)
    tau_Y = np.broadcast_to(np.asarray(tau_Y, dtype=np.float64), s.shape[:1]).copy()
    live = ~((softening > 0.0) & ~(tau_Y > 0.0))
    eps = np.log(s)
    tr = eps.sum(axis=1)
    eps_hat = eps - tr[:, None] / 3.0
    nrm = np.linalg.norm(eps_hat, axis=1)
    dg = nrm - tau_Y / (2.0 * mu)
    Z = s.copy()
    proj = live & (dg > 0.0)
    if np.any(proj):
        Z[proj] = np.exp(eps[proj] - (dg[proj] / nrm[proj])[:, None] * eps_hat[proj])
    tY = tau_Y.copy()
    if np.any(proj):
        plastic = np.linalg.norm(eps[proj] - np.log(Z[proj]), axis=1)   # ||eps - proj(eps)||_F
        tY[proj] = tau_Y[proj] + 2.0 * mu * hardening * dg[proj] - softening * plastic
    tY = np.where(tY > 0.0, tY, 0.0)
    damaged = (softening > 0.0) & ~(tY > 0.0)
    return Z, tY, damaged


def elastoplastic_update(F_trial, model, mu, lam, alpha=0.0, tau_Y=0.0, kappa=None, eta=0.0, dt=1.0):
    """F^E = returnMap(F_trial), tau = tau(F^E).

    model 0 fixed-corotated (F^E = F_trial), 1 Drucker-Prager, 2 von Mises,
    4 the appendix's "StVK elasticity": tau = U (2 mu eps + lambda sum(eps) 1) U^T with
    eps = log(Sigma) and F^E = F_trial, i.e. Hencky elasticity without a return map (reading #3 for U^T),
    5 Herschel-Bulkley (reading #39; sigma_Y = tau_Y, viscosity eta, substep dt,
    bulk modulus kappa).
    Returns (F_E, tau).
    """
    F_trial = np.asarray(F_trial, dtype=np.float64)
    if model == 0:
        return F_trial.copy(), tau_fixed_corotated(F_trial, mu, lam)
    if model == 5:
        return return_map_herschel_bulkley(F_trial, mu, kappa, tau_Y, eta, dt)
    U, s, V = svd_rotation_safe(F_trial)
    if model == 4:
        return F_trial.copy(), tau_hencky(U, s, mu, lam)
    if model == 1:
        Z = return_map_drucker_prager(s, mu, lam, alpha)
    elif model == 2:
        Z = return_map_von_mises(s, mu, tau_Y)
    else:
        raise ValueError("model")
    F_E = _diag_sandwich(U, Z, V)
    return F_E, tau_hencky(U, Z, mu, lam)


def elastoplastic_update_vm_hs(F_trial, mu, lam, tau_Y, hardening=0.0, softening=0.0):
    """von Mises with hardening / softening and damage (readings
    #30-#32): F^E = U Z V^T, tau = tau(F^E) with zero Lame parameters for damaged
    particles.  Returns (F_E, tau, tau_Y_new)."""
    F_trial = np.asarray(F_trial, dtype=np.float64)
    U, s, V = svd_rotation_safe(F_trial)
    Z, tY, damaged = return_map_von_mises_hs(s, mu, tau_Y, hardening, softening)
    F_E = _diag_sandwich(U, Z, V)
    tau = tau_hencky(U, Z, mu, lam)
    tau[damaged] = 0.0
    return F_E, tau, tY


def tau_herschel_bulkley(F, mu, kappa):
    """tau = kappa/2 (J^2 - 1) I + mu dev[det(b)^(-1/3) b], b = F F^T
    (b^E of the elastic state), J = det F.  (J = 0: the deviatoric term is dropped.)"""
    F = np.asarray(F, dtype=np.float64)
    J = np.linalg.det(F)
    b = F @ np.swapaxes(F, -1, -2)
    detb = np.linalg.det(b)
    scale = np.where(detb > 0.0, np.abs(detb) ** (-1.0 / 3.0), 0.0)
    bbar = scale[:, None, None] * b
    dev = bbar - (np.trace(bbar, axis1=1, axis2=2) / 3.0)[:, None, None] * np.eye(3)
    return 0.5 * kappa * (J * J - 1.0)[:, None, None] * np.eye(3) + mu * dev


def return_map_herschel_bulkley(F_trial, mu, kappa, sigma_Y, eta, dt):
    """PAPER.md lines 546-552 (Yue et al. 2015 with h = 1) and reading #39.

    s^trial = dev(tau^trial) = mu dev(bbar^trial), s^trial = ||s^trial||.  If
    s^trial - sqrt(2/3) sigma_Y > 0:
        s = s^trial - (s^trial - sqrt(2/3) sigma_Y) / (1 + eta / (2 mu dt)),
        s (tensor) = s * s^trial / ||s^trial||.
    Elastic state (#39): bbar_new = s / mu + I_bar 1 with det(bbar_new) = 1, J and the
    rotation of F_trial kept: in the principal frame of F_trial = U diag(sigma) V^T,
    F^E = U diag(sign * sqrt(|J|^(2/3) bbar_new_i)) V^T.  Returns (F_E, tau(F_E)).
    """
    F_trial = np.asarray(F_trial, dtype=np.float64)
    U, sg, V = svd_rotation_safe(F_trial)
    J = np.prod(sg, axis=1)
    aJ = np.abs(J)
    j23 = aJ ** (2.0 / 3.0)
    ok = aJ > 0.0
    bbar = np.where(ok[:, None], sg * sg / np.where(ok, j23, 1.0)[:, None], 1.0)
    mean = bbar.mean(axis=1)
    d = bbar - mean[:, None]                       # dev(bbar) (principal)
    st = mu * np.linalg.norm(d, axis=1)            # s^trial
    y = np.sqrt(2.0 / 3.0) * sigma_Y
    plastic = ok & (st - y > 0.0)
    F_E = F_trial.copy()
    if np.any(plastic):
        s_new = st - (st - y) / (1.0 + eta / (2.0 * mu * dt))
        dn = d[plastic] * (s_new[plastic] / st[plastic])[:, None]   # s / mu
        # I_bar: the root of prod(dn_i + I) = 1 (Newton from the trial mean; the
        # product is increasing and convex there and >= 1 at the start)
        Ib = mean[plastic].copy()
        for _ in range(60):
            f = np.prod(dn + Ib[:, None], axis=1) - 1.0
            fp = ((dn[:, 1] + Ib) * (dn[:, 2] + Ib) + (dn[:, 0] + Ib) * (dn[:, 2] + Ib)
                  + (dn[:, 0] + Ib) * (dn[:, 1] + Ib))
            Ib = Ib - f / fp
        bnew = dn + Ib[:, None]
        sig = np.sqrt(j23[plastic][:, None] * bnew)
        sig[:, 2] *= np.sign(J[plastic])
        F_E[plastic] = _diag_sandwich(U[plastic], sig, V[plastic])
    return F_E, tau_herschel_bulkley(F_E, mu, kappa)
