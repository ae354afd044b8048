"""Reduced-order substep on the integration points (§5.1-5.2),
batched over independent scenes (BASELINE.json config 5), fp64.

Per scene s and substep n:
  z_s(n) = z_s(0) + n dz_s                      (reading #26)
  tau_p  = h(X_p, z_s(n))                       (line 253, Eq. (9))
  one MPM step (§3.3) on the scene's points with that tau and NO F / SVD /
  return map (lines 219, 493): P2G, grid update, G2P updating x, v, C.
Each scene owns its own grid_res^3 grid.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
import numpy as np

from .mlp import nsf_stress, voigt_to_matrix
from .mpm import p2g, grid_update, g2p, check_domain


def reduced_substep(state, P, offsets, X_ref, mlp, sigma_tau, z0, dz, step,
                    mode="emulate", tau_override=None):
    """state: x, v, C (n,.) arrays.  offsets: (S+1,) scene boundaries.
    tau_override: optional (n,6) Voigt stress used instead of the MLP (lets a
    parity test feed the GPU's own MLP output as part of the identical state)."""
    x = np.asarray(state["x"], np.float64)
    v = np.asarray(state["v"], np.float64)
    C = np.asarray(state["C"], np.float64)
    check_domain(x, P)
    n = x.shape[0]
    xo, vo, Co = np.empty_like(x), np.empty_like(v), np.empty_like(C)
    tau_all = np.empty((n, 6))
    for s in range(len(offsets) - 1):
        a, b = int(offsets[s]), int(offsets[s + 1])
        if b == a:
            continue
        if tau_override is not None:
            tv = np.asarray(tau_override[a:b], np.float64)
        else:
            z = np.asarray(z0[s], np.float64) + step * np.asarray(dz[s], np.float64)
            tv = nsf_stress(X_ref[a:b], z, mlp, sigma_tau, mode)
        tau_all[a:b] = tv
        tau = voigt_to_matrix(tv)
        uid, gnode, gm, gp = p2g(x[a:b], v[a:b], C[a:b], tau, P)
        vi = grid_update(gnode, gm, gp, P, step)
        xn, vn, Cn, _ = g2p(x[a:b], None, uid, vi, P, want_F=False)
        xo[a:b], vo[a:b], Co[a:b] = xn, vn, Cn
    check_domain(xo, P)
    return {"x": xo, "v": vo, "C": Co, "tau": tau_all}


def reduced_run(state, P, offsets, X_ref, mlp, sigma_tau, z0, dz, n, step0=0, mode="emulate"):
    s = {k: np.asarray(state[k], np.float64) for k in ("x", "v", "C")}
    for k in range(n):
        s = reduced_substep(s, P, offsets, X_ref, mlp, sigma_tau, z0, dz, step0 + k, mode)
    return s
