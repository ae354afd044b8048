"""Parity helpers: run the CUDA path (through the C ABI binding) and the fp64
oracle from the same fp32 state and compare field by field.

Metric (SURVEY.md §8(c) "Parity metrics"):
    e_f = ||a_f - b_f||_2 / max(||b_f||_2, sqrt(N) * s_f)
with floors s_f: x 0, v |g| dt, C max_p |v_ref,p| / dx, F 1, tau 0.1 E.
Bar: e_f <= 1e-5 for one substep from an identical state (BASELINE.json
north_star), <= 1e-3 on positions after 200 substeps (elastic config).
"""
import numpy as np

import oracle
from oracle import mpm

VOIGT = [(0, 0), (1, 1), (2, 2), (1, 2), (0, 2), (0, 1)]
BAR_STEP = 1e-5
BAR_TRAJ = 1e-3


def voigt_to_mat(t):
    t = np.asarray(t, np.float64)
    T = np.zeros(t.shape[:-1] + (3, 3))
    for k, (i, j) in enumerate(VOIGT):
        T[..., i, j] = t[..., k]
        T[..., j, i] = t[..., k]
    return T


def rel_err(a, b, floor=0.0):
    a = np.asarray(a, np.float64).reshape(len(a), -1)
    b = np.asarray(b, np.float64).reshape(len(b), -1)
    n = a.shape[0]
    den = max(np.linalg.norm(b), np.sqrt(n) * floor)
    if den == 0.0:
        return float(np.linalg.norm(a - b))
    return float(np.linalg.norm(a - b) / den)


def floors(cfg, ref_v):
    g = float(np.linalg.norm(cfg.gravity))
    vmax = float(np.max(np.linalg.norm(ref_v, axis=1))) if len(ref_v) else 0.0
    return {"x": 0.0, "v": g * cfg.dt, "C": vmax * cfg.grid_res, "F": 1.0, "tau": 0.1 * cfg.E}


def gpu_state(sim):
    st = sim.read()
    out = {k: np.asarray(v, np.float64) for k, v in st.items()}
    if "tau" in out:
        out["tau_voigt"] = out["tau"]
        out["tau"] = voigt_to_mat(out["tau"])
    return out


def oracle_step(state, cfg, step):
    P = mpm.params_from_config(cfg)
    return mpm.substep(state, P, step)


def compare(gpu, ref, cfg, fields=("x", "v", "C", "F", "tau")):
    fl = floors(cfg, ref["v"])
    return {f: rel_err(gpu[f], ref[f], fl[f]) for f in fields}


def single_step_parity(sim, cfg, step_index):
    """Read the GPU state S_k, advance the GPU one substep, advance the oracle one
    substep from the same (fp32) S_k; return per-field errors."""
    s0 = gpu_state(sim)
    sim.substep(1)
    sim.sync()
    s1 = gpu_state(sim)
    ref = oracle_step({k: s0[k] for k in ("x", "v", "C", "F", "tau")}, cfg, step_index)
    return compare(s1, ref, cfg), s1, ref
