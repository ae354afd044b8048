"""fp64 explicit MPM substep (§3.3), particles in index order.

One substep from state (x, v, C, F, tau) at t_n = n dt:

  1 P2G   (line 176, Eq.(6))
      m_i   = sum_p w_ip m_p
      m_i v_i = sum_p w_ip m_p (v_p + C_p (x_i - x_p))       [APIC]
      force folded into the momentum (reading #14):
        GRADW: - dt sum_p tau_p grad(w_ip) V0             (Eq. (6) literally)
        MLS  : - dt sum_p (4/dx^2) w_ip tau_p (x_i - x_p) V0  (reading #1)
  2 grid update (line 177): v_i = (m_i v_i)/m_i + dt g if m_i > 0 else 0
      (reading #15), then walls (#11, #12), then the moving plate (#12).
  3 G2P   (lines 178-180)
      v_p = sum w v_i ; C_p = 12/(dx^2 (b+1)) sum w v_i (x_i - x_p)^T, b = 2 (#7)
      x_p += dt v_p ; F_trial = (I + dt G) F_E,
        G = sum v_i grad(w)^T (GRADW) or C_p (MLS)
      F_E = returnMap(F_trial), tau = tau(F_E)          (constitutive.py)

Quadratic B-spline (line 165, degree b = 2, reading #7):
  t = x/dx, base = floor(t - 1/2), f = t - base in [1/2, 3/2)
  w = (1/2 (3/2 - f)^2, 3/4 - (f - 1)^2, 1/2 (f - 1/2)^2)
  dw/dx = (f - 3/2, -2 (f - 1), f - 1/2) / dx
Nodes x_i = i dx (reading #8, #10).

The grid is kept sparse: node ids of every touched node (np.unique), so any
grid size works.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .constitutive import lame, dp_alpha, elastoplastic_update, elastoplastic_update_vm_hs, tau_fixed_corotated, \
    svd_rotation_safe, tau_hencky, tau_herschel_bulkley

OFFSETS = np.array([(a, b, c) for a in range(3) for b in range(3) for c in range(3)],
                   dtype=np.int64)  # (27,3), lexicographic


class OutOfDomain(ValueError):
    """A particle left the safe region x/dx in [0.5, N - 1.5)."""

    def __init__(self, index):
        super().__init__(f"particle {index} out of domain")
        self.index = int(index)


@dataclass
class Params:
    grid_res: tuple            # (Nx, Ny, Nz) nodes per axis
    dx: float
    dt: float
    model: int                 # 0 FC, 1 DP, 2 VM, 3 NSF, 4 Hencky ("StVK"), 5 Herschel-Bulkley
    mu: float
    lam: float
    alpha: float = 0.0         # DP
    tau_Y: float = 0.0         # VM
    mass: float = 0.0          # m_p (uniform)
    V0: float = 0.0            # V_p^0 (uniform)
    gravity: tuple = (0.0, -9.8, 0.0)
    bc: tuple = (0,) * 6       # faces -x,+x,-y,+y,-z,+z ; 0 none, 1 sticky, 2 slip
    bc_width: int = 3
    plate_enabled: int = 0
    plate_y0: float = 0.0
    plate_velocity: tuple = (0.0, 0.0, 0.0)
    force_mode: int = 0        # 0 MLS, 1 GRADW
    transfer: int = 0          # 0 APIC, 1 PIC, 2 RPIC (reading #38)
    hardening: float = 0.0     # VM xi   (#30)
    softening: float = 0.0     # VM theta (#30)
    kappa: float = 0.0         # bulk modulus E / (3 (1 - 2 nu)) (Table, Herschel-Bulkley)
    viscosity: float = 0.0     # Herschel-Bulkley eta (#39)

    @property
    def inv_dx(self):
        return 1.0 / self.dx


def params_from_config(cfg) -> Params:
    """Derive the method constants from a scenes.Config (Lame: lines 504-512;
    V0 default dx^3/8 for 8 ppc (reading #16); m_p = rho V0)."""
    mu, lam, kappa = lame(cfg.E, cfg.nu)
    dx = 1.0 / cfg.grid_res
    V0 = cfg.particle_volume if cfg.particle_volume > 0 else dx ** 3 / 8.0
    return Params(grid_res=(cfg.grid_res,) * 3, dx=dx, dt=cfg.dt, model=cfg.model,
                  mu=mu, lam=lam, alpha=dp_alpha(cfg.friction_angle_deg),
                  tau_Y=cfg.yield_stress, mass=cfg.rho * V0, V0=V0,
                  gravity=tuple(cfg.gravity), bc=tuple(cfg.bc), bc_width=cfg.bc_width,
                  plate_enabled=cfg.plate_enabled, plate_y0=cfg.plate_y0,
                  plate_velocity=tuple(cfg.plate_velocity), force_mode=cfg.force_mode,
                  transfer=getattr(cfg, "transfer", 0), hardening=getattr(cfg, "hardening", 0.0),
                  softening=getattr(cfg, "softening", 0.0), kappa=kappa,
                  viscosity=getattr(cfg, "viscosity", 0.0))


# ---------------------------------------------------------------------------

def check_domain(x, P: Params):
    t = np.asarray(x, dtype=np.float64) * P.inv_dx
    N = np.asarray(P.grid_res, dtype=np.float64)
    bad = ~np.all((t >= 0.5) & (t < N - 1.5), axis=1)
    if np.any(bad):
        raise OutOfDomain(np.flatnonzero(bad)[0])


def bspline_quadratic(x, inv_dx):
    """Returns base (n,3) int64, f (n,3), w (n,3axes,3nodes), dw (n,3,3)."""
    t = np.asarray(x, dtype=np.float64) * inv_dx
    base = np.floor(t - 0.5).astype(np.int64)
    f = t - base
    w = np.stack([0.5 * (1.5 - f) ** 2, 0.75 - (f - 1.0) ** 2, 0.5 * (f - 0.5) ** 2], axis=-1)
    dw = np.stack([f - 1.5, -2.0 * (f - 1.0), f - 0.5], axis=-1) * inv_dx
    return base, f, w, dw


def _stencil(x, P: Params):
    """Per (particle, node) quantities for the 27 nodes: node index, W, d = x_i - x_p,
    grad W.  Shapes (n,27,3) / (n,27) / (n,27,3) / (n,27,3)."""
    base, f, w, dw = bspline_quadratic(x, P.inv_dx)
    a, b, c = OFFSETS[:, 0], OFFSETS[:, 1], OFFSETS[:, 2]
    wa, wb, wc = w[:, 0, a], w[:, 1, b], w[:, 2, c]
    W = wa * wb * wc
    gW = np.stack([dw[:, 0, a] * wb * wc, wa * dw[:, 1, b] * wc, wa * wb * dw[:, 2, c]], axis=-1)
    node = base[:, None, :] + OFFSETS[None, :, :]
    d = (OFFSETS[None, :, :] - f[:, None, :]) * P.dx
    return node, W, d, gW


def _linear_id(node, P: Params):
    Nx, Ny, Nz = P.grid_res
    return (node[..., 0] * Ny + node[..., 1]) * Nz + node[..., 2]


def p2g(x, v, C, tau, P: Params):
    """Step 1 (line 176 + Eq. (6)).  Returns (ids, node (k,3), m (k,), mv (k,3)) over
    every node touched by a stencil, ids sorted ascending."""
    x = np.asarray(x, np.float64)
    v = np.asarray(v, np.float64)
    C = np.asarray(C, np.float64)
    tau = np.asarray(tau, np.float64)
    node, W, d, gW = _stencil(x, P)
    m = P.mass
    # APIC momentum: w m (v_p + C_p d); PIC: w m v_p
    if P.transfer == 1:
        mom = W[..., None] * m * np.broadcast_to(v[:, None, :], d.shape)
    else:
        mom = W[..., None] * m * (v[:, None, :] + np.einsum("pij,pnj->pni", C, d))
    if P.force_mode == 0:   # MLS force (reading #1): -dt V0 (4/dx^2) w tau d
        mom -= P.dt * P.V0 * (4.0 / P.dx ** 2) * W[..., None] * np.einsum("pij,pnj->pni", tau, d)
    else:                   # Eq. (6): -dt tau grad(w) V0
        mom -= P.dt * P.V0 * np.einsum("pij,pnj->pni", tau, gW)
    ids = _linear_id(node, P).reshape(-1)
    uid, inv = np.unique(ids, return_inverse=True)
    k = uid.shape[0]
    gm = np.bincount(inv, weights=(W * m).reshape(-1), minlength=k)
    gp = np.stack([np.bincount(inv, weights=mom[..., a].reshape(-1), minlength=k)
                   for a in range(3)], axis=-1)
    Nx, Ny, Nz = P.grid_res
    gnode = np.stack([uid // (Ny * Nz), (uid // Nz) % Ny, uid % Nz], axis=-1)
    return uid, gnode, gm, gp


def grid_update(gnode, gm, gp, P: Params, step: int):
    """Step 2 (line 177) with readings #11-#15.  Returns v_i (k,3)."""
    vi = np.zeros_like(gp)
    act = gm > 0.0
    vi[act] = gp[act] / gm[act][:, None] + P.dt * np.asarray(P.gravity)
    N = P.grid_res
    wdt = P.bc_width
    for face in range(6):
        axis, high = face // 2, face % 2
        kind = P.bc[face]
        if kind == 0:
            continue
        region = (gnode[:, axis] >= N[axis] - wdt) if high else (gnode[:, axis] < wdt)
        if kind == 1:      # sticky: v = 0
            vi[region] = 0.0
        elif kind == 2:    # slip: remove the normal component pointing into the wall
            comp = vi[region, axis]
            vi[region, axis] = np.minimum(comp, 0.0) if high else np.maximum(comp, 0.0)
    if P.plate_enabled:
        y_plate = P.plate_y0 + P.plate_velocity[1] * (step * P.dt)
        region = gnode[:, 1] * P.dx >= y_plate
        vi[region] = np.asarray(P.plate_velocity)
    vi[~act] = 0.0
    return vi


def g2p(x, F, uid, vi, P: Params, want_F=True):
    """Step 3 (lines 178-180) up to F_trial.  Returns (x', v', C', F_trial)."""
    x = np.asarray(x, np.float64)
    node, W, d, gW = _stencil(x, P)
    ids = _linear_id(node, P)
    pos = np.searchsorted(uid, ids)
    vn = vi[pos]                                             # (n,27,3)
    v_new = np.einsum("pn,pni->pi", W, vn)
    B = np.einsum("pn,pni,pnj->pij", W, vn, d)
    C_new = (12.0 / (P.dx ** 2 * (2 + 1))) * B               # 12/(dx^2 (b+1)), b = 2
    x_new = x + P.dt * v_new
    F_tr = None
    if want_F:
        G = C_new if P.force_mode == 0 else np.einsum("pni,pnj->pij", vn, gW)
        F_tr = (np.eye(3) + P.dt * G) @ np.asarray(F, np.float64)
    if P.transfer == 2:
        # RPIC ("RPIC can be added in the computation of C_p", reading #38):
        # C_p keeps only its skew-symmetric (rigid-rotation) part; F_trial above
        # used the full velocity gradient
        C_new = 0.5 * (C_new - np.transpose(C_new, (0, 2, 1)))
    return x_new, v_new, C_new, F_tr


def initial_tau(F, P: Params):
    """tau^0 = tau(F^0) at load (reading #9); F^0 is taken as elastic."""
    F = np.asarray(F, np.float64)
    if P.model == 0:
        return tau_fixed_corotated(F, P.mu, P.lam)
    if P.model == 5:
        return tau_herschel_bulkley(F, P.mu, P.kappa)
    U, s, V = svd_rotation_safe(F)
    return tau_hencky(U, s, P.mu, P.lam)


def substep(state: dict, P: Params, step: int, check=True) -> dict:
    """One full-order substep.  state: x, v, C, F, tau (float arrays, any float dtype)."""
    x, v, C, F, tau = (np.asarray(state[k], np.float64) for k in ("x", "v", "C", "F", "tau"))
    if check:
        check_domain(x, P)
    uid, gnode, gm, gp = p2g(x, v, C, tau, P)
    vi = grid_update(gnode, gm, gp, P, step)
    x_new, v_new, C_new, F_tr = g2p(x, F, uid, vi, P)
    out = {}
    if P.model == 2 and (P.hardening != 0.0 or P.softening != 0.0):
        # per-particle yield stress (#30-#32); state["tau_Y"] defaults to the material's
        tY = np.asarray(state.get("tau_Y", np.full(x.shape[0], P.tau_Y)), np.float64)
        F_E, tau_new, out["tau_Y"] = elastoplastic_update_vm_hs(F_tr, P.mu, P.lam, tY, P.hardening, P.softening)
    else:
        F_E, tau_new = elastoplastic_update(F_tr, P.model, P.mu, P.lam, P.alpha, P.tau_Y, P.kappa, P.viscosity, P.dt)
    if check:
        check_domain(x_new, P)
    out.update({"x": x_new, "v": v_new, "C": C_new, "F": F_E, "tau": tau_new,
                "grid": {"ids": uid, "node": gnode, "m": gm, "mv": gp, "v": vi}})
    return out


def run(state: dict, P: Params, n: int, step0: int = 0) -> dict:
    s = {k: np.asarray(state[k], np.float64) for k in ("x", "v", "C", "F", "tau", "tau_Y") if k in state}
    for k in range(n):
        s = substep(s, P, step0 + k)
        s.pop("grid")
    return s


def block_keys(x, P: Params, block=4):
    """Binning key: linear id of the block x block x block cell
    block containing base_p = floor(x_p/dx - 1/2).  Integer; unique per particle.
    parity unpinned beyond its definition (it is the definition)."""
    base, _, _, _ = bspline_quadratic(x, P.inv_dx)
    nb = [g // block for g in P.grid_res]
    bb = base // block
    return (bb[:, 0] * nb[1] + bb[:, 1]) * nb[2] + bb[:, 2]
