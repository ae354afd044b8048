"""Pins for oracle/mpm.py: B-spline worked examples and moment identities,
P2G conservation laws, the discrete virial of Eq. (6), grid-update worked
example and BC semantics, affine reproduction, APIC round trip, free fall in
closed form, the literal C1 run, static systems (CPU only)."""
import json
import os

import numpy as np
import pytest

import scenes
from oracle import mpm
from oracle.mpm import Params, bspline_quadratic, p2g, grid_update, g2p, substep, OFFSETS

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def P_free(force_mode=0, N=32, **kw):
    d = dict(grid_res=(N, N, N), dx=1.0 / N, dt=1e-3, model=0, mu=2.0, lam=3.0,
             mass=0.7, V0=1.3e-4, gravity=(0.0, 0.0, 0.0), bc=(0,) * 6, force_mode=force_mode)
    d.update(kw)
    return Params(**d)


def rand_state(rng, n, N=32, lo=0.3, hi=0.7, stress=True):
    x = rng.uniform(lo, hi, size=(n, 3))
    v = rng.normal(size=(n, 3))
    C = rng.normal(scale=5.0, size=(n, 3, 3))
    tau = rng.normal(scale=10.0, size=(n, 3, 3)) if stress else np.zeros((n, 3, 3))
    tau = 0.5 * (tau + np.swapaxes(tau, 1, 2))
    F = np.eye(3) + 0.1 * rng.normal(size=(n, 3, 3))
    return x, v, C, F, tau


@pytest.mark.parametrize("ex", GOLD["bspline_1d"])
def test_bspline_worked(ex):
    dx = 1.0 / 16
    x = np.array([[(5 + ex["f"]) * dx] * 3])   # base = 5, f as given
    base, f, w, dw = bspline_quadratic(x, 16.0)
    assert np.all(base == 5)
    assert np.allclose(w[0, 0], ex["w"], atol=1e-15)


def test_bspline_moments():
    """sum w = 1, sum dw = 0, sum w d = 0, sum w d d^T = dx^2/4 I, sum x_i grad(w)^T = I
    (quadratic B-spline identities behind the 12/(dx^2 (b+1)) factor, PAPER.md 178)."""
    rng = np.random.default_rng(0)
    P = P_free()
    x = rng.uniform(0.2, 0.8, size=(1000, 3))
    node, W, d, gW = mpm._stencil(x, P)
    assert np.allclose(W.sum(1), 1.0, atol=1e-14)
    assert np.allclose(gW.sum(1), 0.0, atol=1e-11)
    assert np.allclose(np.einsum("pn,pni->pi", W, d), 0.0, atol=1e-16)
    M2 = np.einsum("pn,pni,pnj->pij", W, d, d)
    assert np.allclose(M2, P.dx ** 2 / 4 * np.eye(3), atol=1e-17)
    xi = node * P.dx
    assert np.allclose(np.einsum("pni,pnj->pij", xi, gW), np.eye(3), atol=1e-11)


def test_bspline_exact_powers_of_two():
    """Reading #10: t = x * (1/dx) with dx = 2^-k is exact, so base/f agree bit-for-bit
    between fp32 positions and the fp64 oracle."""
    rng = np.random.default_rng(1)
    x32 = rng.uniform(0.1, 0.9, size=(10000, 3)).astype(np.float32)
    t32 = x32 * np.float32(256.0)
    b32 = np.floor(t32 - np.float32(0.5))
    f32 = t32 - b32
    base, f, _, _ = bspline_quadratic(x32, 256.0)
    assert np.array_equal(base, b32.astype(np.int64))
    assert np.array_equal(f, f32.astype(np.float64))


@pytest.mark.parametrize("fm", [0, 1])
def test_p2g_mass_momentum_conservation(fm):
    """PAPER.md 176 + Eq.(6): sum m_i = sum m_p, sum m_i v_i = sum m_p v_p (forces and
    the affine term cancel since sum grad(w) = 0 and sum w d = 0)."""
    rng = np.random.default_rng(2)
    P = P_free(fm)
    x, v, C, F, tau = rand_state(rng, 300)
    _, _, gm, gp = p2g(x, v, C, tau, P)
    assert np.isclose(gm.sum(), 300 * P.mass, rtol=1e-14)
    assert np.allclose(gp.sum(0), P.mass * v.sum(0), rtol=1e-12, atol=1e-11)


@pytest.mark.parametrize("fm", [0, 1])
def test_p2g_angular_momentum(fm):
    """APIC angular momentum (PAPER.md 222): sum_i x_i x p_i = sum_p [x_p x m v_p +
    m dx^2/4 (C_zy - C_yz, C_xz - C_zx, C_yx - C_xy)]; symmetric tau exerts no torque."""
    rng = np.random.default_rng(3)
    P = P_free(fm)
    x, v, C, F, tau = rand_state(rng, 200)
    _, gnode, gm, gp = p2g(x, v, C, tau, P)
    L_grid = np.cross(gnode * P.dx, gp).sum(0)
    ax = np.stack([C[:, 2, 1] - C[:, 1, 2], C[:, 0, 2] - C[:, 2, 0], C[:, 1, 0] - C[:, 0, 1]], 1)
    L_p = (np.cross(x, P.mass * v) + P.mass * P.dx ** 2 / 4 * ax).sum(0)
    assert np.allclose(L_grid, L_p, rtol=1e-11, atol=1e-12)


@pytest.mark.parametrize("fm", [0, 1])
def test_force_virial(fm):
    """Discrete divergence of a uniform stress (Eq.(6) with q = x): the grid force of one
    particle satisfies sum_i f_i = 0 and sum_i f_i x_i^T = -V0 tau_p, in both force
    forms.  Pins the magnitude and sign of the stress term."""
    rng = np.random.default_rng(4)
    P = P_free(fm)
    for _ in range(5):
        x, v, C, F, tau = rand_state(rng, 1)
        _, gnode, gm, gp0 = p2g(x, v, C, np.zeros_like(tau), P)
        _, _, _, gp1 = p2g(x, v, C, tau, P)
        f = (gp1 - gp0) / P.dt          # force folded into momentum: dt f_i
        assert np.allclose(f.sum(0), 0.0, atol=1e-9)
        virial = np.einsum("ni,nj->ij", f, gnode * P.dx)
        assert np.allclose(virial, -P.V0 * tau[0], rtol=1e-10, atol=1e-12)


def test_single_particle_pressure_gradw():
    """SPEC.md 183: tau = -p I on one particle -> f_i = p grad(w_ip) V0 (Eq.(6))."""
    P = P_free(1)
    x = np.array([[0.51, 0.47, 0.5]])
    p = 3.0
    _, gnode, gm, gp0 = p2g(x, np.zeros((1, 3)), np.zeros((1, 3, 3)), np.zeros((1, 3, 3)), P)
    _, _, _, gp1 = p2g(x, np.zeros((1, 3)), np.zeros((1, 3, 3)), -p * np.eye(3)[None], P)
    node, W, d, gW = mpm._stencil(x, P)
    f = (gp1 - gp0) / P.dt
    order = np.argsort(mpm._linear_id(node[0], P))
    assert np.allclose(f, p * gW[0][order] * P.V0, rtol=1e-12)


def test_grid_update_worked_and_bcs():
    ex = GOLD["grid_update"][0]
    P = P_free(dt=ex["dt"], gravity=tuple(ex["g"]))
    rng = np.random.default_rng(5)
    gnode = rng.integers(5, 27, size=(50, 3))
    gm = rng.uniform(0.1, 1.0, 50)
    v0 = rng.normal(size=(50, 3))
    vi = grid_update(gnode, gm, gm[:, None] * v0, P, 0)
    assert np.allclose(vi - v0, ex["dv"], atol=1e-15)
    # inactive nodes -> 0
    gm2 = gm.copy()
    gm2[:10] = 0.0
    assert np.all(grid_update(gnode, gm2, gm[:, None] * v0, P, 0)[:10] == 0)
    # sticky walls within 3 nodes of every face, slip removes only the inward normal
    gnode = np.array([[1, 10, 10], [30, 10, 10], [10, 2, 10], [10, 29, 10], [10, 10, 0],
                      [10, 10, 31], [10, 10, 10], [3, 28, 10]])
    vin = np.array([[-1., 2, 3], [1., 2, 3], [1, -2., 3], [1, 2., 3], [1, 2, -3.],
                    [1, 2, 3.], [1, 2, 3.], [-1, 1, 1.]])
    gm = np.ones(8)
    Ps = P_free(bc=(1,) * 6, gravity=(0, 0, 0))
    vs = grid_update(gnode, gm, vin, Ps, 0)
    assert np.all(vs[:6] == 0) and np.array_equal(vs[6:], vin[6:])
    Pl = P_free(bc=(2,) * 6, gravity=(0, 0, 0))
    vl = grid_update(gnode, gm, vin, Pl, 0)
    expect = vin.copy()
    for k, (a, hi) in enumerate([(0, 0), (0, 1), (1, 0), (1, 1), (2, 0), (2, 1)]):
        expect[k, a] = min(vin[k, a], 0) if hi else max(vin[k, a], 0)
    assert np.array_equal(vl, expect)
    # separating slip velocity is kept
    vout = -vin
    vl2 = grid_update(gnode[:6], gm[:6], vout[:6], Pl, 0)
    for k, (a, hi) in enumerate([(0, 0), (0, 1), (1, 0), (1, 1), (2, 0), (2, 1)]):
        assert vl2[k, a] == (min(vout[k, a], 0) if hi else max(vout[k, a], 0))


def test_grid_update_plate():
    """Reading #12: nodes with y_i >= y_p(t_n) = y0 + v_y n dt move with the plate."""
    P = P_free(plate_enabled=1, plate_y0=20 / 32, plate_velocity=(0.0, -0.5, 0.0),
               gravity=(0, 0, 0), dt=2e-2)
    gnode = np.array([[10, 19, 10], [10, 20, 10], [10, 21, 10]])
    vi = grid_update(gnode, np.ones(3), np.ones((3, 3)), P, 0)
    assert np.array_equal(vi[0], [1, 1, 1]) and np.all(vi[1:] == [0, -0.5, 0])
    # after 4 steps the plate is at 20/32 - 0.04 = 0.585 -> node 19 (0.59375) inside
    vi = grid_update(gnode, np.ones(3), np.ones((3, 3)), P, 4)
    assert np.all(vi == [0, -0.5, 0])


@pytest.mark.parametrize("fm", [0, 1])
def test_affine_reproduction(fm):
    """Grid v_i = A x_i + b -> v_p = A x_p + b, C_p = A, F_trial = (I + dt A) F
    (quadratic B-spline reproduces affine fields; PAPER.md 178-179)."""
    rng = np.random.default_rng(6)
    P = P_free(fm)
    x, v, C, F, tau = rand_state(rng, 100)
    A = rng.normal(size=(3, 3))
    b = rng.normal(size=3)
    node, _, _, _ = mpm._stencil(x, P)
    uid = np.unique(mpm._linear_id(node, P))
    Nn = P.grid_res[0]
    gnode = np.stack([uid // Nn ** 2, (uid // Nn) % Nn, uid % Nn], -1)
    vi = gnode * P.dx @ A.T + b
    xn, vn, Cn, Ftr = g2p(x, F, uid, vi, P)
    assert np.allclose(vn, x @ A.T + b, atol=1e-12)
    assert np.allclose(Cn, A, atol=1e-9)
    assert np.allclose(Ftr, (np.eye(3) + P.dt * A) @ F, atol=1e-12)
    assert np.allclose(xn, x + P.dt * vn, atol=1e-15)


def test_apic_round_trip():
    """Particles sampling v = A x + b with C_p = A, no force, no gravity: P2G gives
    v_i = A x_i + b on massive nodes and G2P returns the same (v_p, C_p)."""
    rng = np.random.default_rng(7)
    P = P_free(0)
    sc = scenes.block_scene("rt", 32, (10, 10, 10), (16, 15, 17), scenes.FIXED_COROTATED, 7)
    x = sc.x.astype(np.float64)
    A = rng.normal(size=(3, 3))
    b = rng.normal(size=3)
    v = x @ A.T + b
    C = np.broadcast_to(A, (x.shape[0], 3, 3))
    uid, gnode, gm, gp = p2g(x, v, C, np.zeros_like(C), P)
    vi = grid_update(gnode, gm, gp, P, 0)
    act = gm > 0
    assert np.allclose(vi[act], gnode[act] * P.dx @ A.T + b, atol=1e-11)
    xn, vn, Cn, _ = g2p(x, np.broadcast_to(np.eye(3), C.shape), uid, vi, P)
    assert np.allclose(vn, v, atol=1e-11) and np.allclose(Cn, A, atol=1e-8)


def test_static_system_invariant():
    sc = scenes.block_scene("st", 32, (10, 10, 10), (14, 13, 15), scenes.VON_MISES, 8)
    P = mpm.params_from_config(sc.cfg)
    P.gravity = (0.0, 0.0, 0.0)
    P.plate_enabled = 0
    st = {"x": sc.x, "v": np.zeros_like(sc.x, dtype=np.float64), "C": np.zeros((sc.n, 3, 3)),
          "F": np.broadcast_to(np.eye(3), (sc.n, 3, 3)), "tau": np.zeros((sc.n, 3, 3))}
    out = substep(st, P, 0)
    assert np.allclose(out["x"], sc.x, atol=0) and np.all(out["v"] == 0)
    assert np.allclose(out["F"], np.eye(3), atol=1e-15) and np.allclose(out["tau"], 0, atol=1e-9)


def test_free_fall_closed_form_spec():
    """SPEC.md 209: g = (0,-10,0), dt = 1e-3, no walls, zero stress: after 100 steps
    v_y = -1.0 exactly (to 1e-10), y = y0 - dt^2 g n(n+1)/2."""
    ex = GOLD["free_fall"][0]
    P = P_free(dt=ex["dt"], gravity=tuple(ex["g"]), N=64)
    sc = scenes.block_scene("ff", 64, (28, 40, 28), (30, 42, 30), scenes.FIXED_COROTATED, 9)
    n = sc.n
    st = {"x": sc.x.astype(np.float64), "v": np.zeros((n, 3)), "C": np.zeros((n, 3, 3)),
          "F": np.broadcast_to(np.eye(3), (n, 3, 3)).copy(), "tau": np.zeros((n, 3, 3))}
    s = mpm.run(st, P, ex["steps"])
    k = ex["steps"]
    assert np.allclose(s["v"][:, 1], ex["v_y"], atol=1e-10)
    assert np.allclose(s["x"][:, 1], sc.x[:, 1] + ex["dt"] ** 2 * ex["g"][1] * k * (k + 1) / 2,
                       atol=1e-12)
    assert np.allclose(s["C"], 0, atol=1e-8) and np.allclose(s["F"], np.eye(3), atol=1e-12)


def test_c1_literal_is_free_fall():
    """C1 as specified never reaches a wall node within 200 substeps, so
    every particle follows x^n = x^0 + n dt v0 + dt^2 g n(n+1)/2, v^n = v0 + n dt g, and
    F = I, C = 0, tau = 0 stay (up to rounding)."""
    sc = scenes.c1()
    P = mpm.params_from_config(sc.cfg)
    n = sc.n
    st = {"x": sc.x, "v": sc.v, "C": sc.C, "F": sc.F,
          "tau": mpm.initial_tau(sc.F, P)}
    K = sc.cfg.substeps
    s = mpm.run(st, P, K)
    g = sc.cfg.gravity[1]
    dt = sc.cfg.dt
    assert np.allclose(s["v"][:, 1], -1.0 + K * dt * g, atol=1e-11)
    y = sc.x[:, 1].astype(np.float64) + K * dt * (-1.0) + dt ** 2 * g * K * (K + 1) / 2
    assert np.allclose(s["x"][:, 1], y, atol=1e-12)
    assert np.allclose(s["x"][:, [0, 2]], sc.x[:, [0, 2]], atol=1e-15)
    assert np.max(np.abs(s["F"] - np.eye(3))) < 1e-12
    assert np.max(np.abs(s["C"])) < 1e-8 and np.max(np.abs(s["tau"])) < 1e-7


def test_out_of_domain():
    P = P_free()
    x = np.array([[0.5, 0.5, 0.5], [0.5, 0.01, 0.5]])
    with pytest.raises(mpm.OutOfDomain) as e:
        mpm.check_domain(x, P)
    assert e.value.index == 1


def test_brute_force_consistency_tiny():
    """Consistency check (not a pin: it re-types the same formulas): a pure-Python
    loop transcription on 4 particles agrees with the vectorised oracle to 1e-13."""
    rng = np.random.default_rng(10)
    for fm in (0, 1):
        P = P_free(fm, gravity=(0.0, -9.8, 0.0), bc=(1, 2, 1, 2, 2, 1))
        x, v, C, F, tau = rand_state(rng, 4, lo=0.1, hi=0.2)
        grid = {}
        for p in range(4):
            t = x[p] / P.dx
            base = np.floor(t - 0.5).astype(int)
            f = t - base
            w = [[0.5 * (1.5 - f[a]) ** 2, 0.75 - (f[a] - 1) ** 2, 0.5 * (f[a] - 0.5) ** 2] for a in range(3)]
            dw = [[(f[a] - 1.5) / P.dx, -2 * (f[a] - 1) / P.dx, (f[a] - 0.5) / P.dx] for a in range(3)]
            for i in range(3):
                for j in range(3):
                    for k in range(3):
                        Wt = w[0][i] * w[1][j] * w[2][k]
                        gw = np.array([dw[0][i] * w[1][j] * w[2][k], w[0][i] * dw[1][j] * w[2][k],
                                       w[0][i] * w[1][j] * dw[2][k]])
                        node = (base[0] + i, base[1] + j, base[2] + k)
                        d = np.array(node) * P.dx - x[p]
                        m, mv = grid.get(node, (0.0, np.zeros(3)))
                        m += Wt * P.mass
                        mv = mv + Wt * P.mass * (v[p] + C[p] @ d)
                        if fm == 0:
                            mv = mv - P.dt * P.V0 * 4 / P.dx ** 2 * Wt * tau[p] @ d
                        else:
                            mv = mv - P.dt * P.V0 * tau[p] @ gw
                        grid[node] = (m, mv)
        uid, gnode, gm, gp = p2g(x, v, C, tau, P)
        for r in range(len(uid)):
            m, mv = grid[tuple(gnode[r])]
            assert np.isclose(gm[r], m, rtol=1e-13) and np.allclose(gp[r], mv, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("fm", [0, 1])
def test_pic_transfer(fm):
    """PIC: m_i v_i = sum_p w m_p v_p.  Linear momentum is
    conserved; the grid's angular momentum is exactly sum_p x_p x m v_p (the
    B-spline's first moment), i.e. the particles' affine spin is dropped, unlike
    APIC (test_p2g_angular_momentum); mass is unchanged; and the PIC and APIC
    momenta differ by exactly the affine term."""
    import dataclasses
    rng = np.random.default_rng(7)
    P = P_free(fm)
    Ppic = dataclasses.replace(P, transfer=1)
    x, v, C, F, tau = rand_state(rng, 150)
    zero = np.zeros_like(tau)
    _, gnode, gm, gp = p2g(x, v, C, zero, Ppic)
    assert np.allclose(gp.sum(0), (P.mass * v).sum(0), rtol=1e-12, atol=1e-14)
    L_grid = np.cross(gnode * P.dx, gp).sum(0)
    assert np.allclose(L_grid, np.cross(x, P.mass * v).sum(0), rtol=1e-11, atol=1e-13)
    _, gnode_a, gm_a, gp_a = p2g(x, v, C, zero, P)
    assert np.array_equal(gnode, gnode_a) and np.allclose(gm, gm_a, rtol=1e-14)
    _, _, _, gp_c = p2g(x, np.zeros_like(v), C, zero, P)   # APIC with v = 0: the affine term alone
    assert np.allclose(gp_a - gp, gp_c, rtol=1e-10, atol=1e-14)


def _grid_field(P, x, fn):
    node, _, _, _ = mpm._stencil(x, P)
    uid = np.unique(mpm._linear_id(node, P))
    Nn = P.grid_res[0]
    gnode = np.stack([uid // Nn ** 2, (uid // Nn) % Nn, uid % Nn], -1)
    return uid, fn(gnode * P.dx)


@pytest.mark.parametrize("fm", [0, 1])
def test_rpic_rigid_rotation_and_symmetric_part(fm):
    """RPIC (reading #38): G2P keeps only the skew-symmetric part
    of C_p.  A rigid rotation v_i = W x_i + b (W skew) is reproduced exactly (C_p = W,
    as under APIC); a pure strain rate v_i = S x_i (S symmetric) leaves C_p = 0 under
    RPIC and S under APIC, while F_trial uses the full velocity gradient in both
    (reading #38: the projection only feeds the transfer)."""
    import dataclasses
    rng = np.random.default_rng(11)
    P = P_free(fm)
    Pr = dataclasses.replace(P, transfer=2)
    x, v, C, F, tau = rand_state(rng, 100)
    w = rng.normal(size=3)
    Wsk = np.array([[0.0, -w[2], w[1]], [w[2], 0.0, -w[0]], [-w[1], w[0], 0.0]])
    b = rng.normal(size=3)
    uid, vi = _grid_field(P, x, lambda xi: xi @ Wsk.T + b)
    xn, vn, Cn, Ftr = g2p(x, F, uid, vi, Pr)
    assert np.allclose(vn, x @ Wsk.T + b, atol=1e-12) and np.allclose(Cn, Wsk, atol=1e-9)
    assert np.allclose(Cn + np.transpose(Cn, (0, 2, 1)), 0.0, atol=0)          # exactly skew
    A = rng.normal(size=(3, 3))
    S = A + A.T
    uid, vi = _grid_field(P, x, lambda xi: xi @ S.T)
    _, _, Cr, Fr = g2p(x, F, uid, vi, Pr)
    _, _, Ca, Fa = g2p(x, F, uid, vi, P)
    assert np.allclose(Cr, 0.0, atol=1e-9) and np.allclose(Ca, S, atol=1e-9)
    assert np.allclose(Fr, (np.eye(3) + P.dt * S) @ F, atol=1e-12) and np.array_equal(Fr, Fa)


def test_rpic_keeps_apic_angular_momentum():
    """The particles' angular momentum depends on C only through its skew part
    (test_p2g_angular_momentum), so after any G2P the RPIC state carries exactly the
    grid angular momentum and linear momentum the APIC state does, while its P2G
    momenta differ from APIC's by the symmetric part of C alone."""
    import dataclasses
    rng = np.random.default_rng(12)
    P = P_free(0)
    Pr = dataclasses.replace(P, transfer=2)
    x, v, C, F, tau = rand_state(rng, 200)
    uid, vi = _grid_field(P, x, lambda xi: np.sin(3.0 * xi) + xi @ rng.normal(size=(3, 3)))
    _, va, Ca, _ = g2p(x, F, uid, vi, P)
    _, vr, Cr, _ = g2p(x, F, uid, vi, Pr)
    assert np.array_equal(va, vr)
    zero = np.zeros_like(tau)
    _, gna, gma, gpa = p2g(x, va, Ca, zero, P)
    _, gnr, gmr, gpr = p2g(x, vr, Cr, zero, P)
    assert np.allclose(gpa.sum(0), gpr.sum(0), rtol=1e-12, atol=1e-13)
    La, Lr = np.cross(gna * P.dx, gpa).sum(0), np.cross(gnr * P.dx, gpr).sum(0)
    assert np.allclose(La, Lr, rtol=1e-11, atol=1e-13)
    Csym = 0.5 * (Ca + np.transpose(Ca, (0, 2, 1)))
    _, _, _, gps = p2g(x, np.zeros_like(va), Csym, zero, P)
    assert np.allclose(gpa - gpr, gps, rtol=1e-10, atol=1e-13)
    assert np.linalg.norm(Csym) > 1e-3     # the case is not degenerate
