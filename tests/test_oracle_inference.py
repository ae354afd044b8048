"""Pins for oracle/inference.py, CPU only.

  - an MLP whose hidden pre-activations stay positive is affine (ELU = identity),
    so in "exact" mode x, v and C are closed forms of the weights: v must be
    W_2 W_1[:, 3:] (z_n - z_prev) / dt (sign, which latent is "previous", dt);
  - an identity deformation field (g(X, z) = X) on a lattice with 2 points per
    cell and axis: one sample particle gives I = its 27 stencil nodes and N = the
    particles whose stencil base is within 2 cells per axis: 10^3 particles;
  - I and N by explicit loops over nodes and particles (the line-269 definition
    written out) on random small inputs, S subset of N, and the point order.
"""
import itertools

import numpy as np

from oracle.inference import field, infer_state, integration_set, ordered_points, stencil_node_ids


def affine_net(rng, r, out, H=8, c=50.0):
    W1 = rng.uniform(-0.5, 0.5, size=(H, 3 + r))
    b1 = np.full(H, c)                       # |W1 u| < c for |u| <= 10: ELU is the identity
    W2 = rng.uniform(-1.0, 1.0, size=(out, H))
    b2 = rng.uniform(-1.0, 1.0, size=out)
    return {"W": [W1, W2], "b": [b1, b2]}


def identity_net(r, c=5.0):
    W1 = np.zeros((3, 3 + r))
    W1[:, :3] = np.eye(3)
    return {"W": [W1, np.eye(3)], "b": [np.full(3, c), np.full(3, -c)]}


def test_inference_affine_closed_forms():
    rng = np.random.default_rng(5)
    r, dt = 4, 1e-4
    g, l = affine_net(rng, r, 3), affine_net(rng, r, 9)
    X = rng.uniform(0.3, 0.7, size=(50, 3))
    z_n, z_p = rng.normal(size=r), rng.normal(size=r)
    x, v, C = infer_state(X, z_n, z_p, g, l, dt, mode="exact")
    A = g["W"][1] @ g["W"][0]                 # the affine map's linear part
    x_cf = X @ A[:, :3].T + A[:, 3:] @ z_n + g["W"][1] @ g["b"][0] + g["b"][1]
    assert np.allclose(x, x_cf, rtol=0, atol=1e-12)
    assert np.allclose(v, np.broadcast_to(A[:, 3:] @ (z_n - z_p) / dt, v.shape), rtol=1e-8, atol=1e-6)
    Al = l["W"][1] @ l["W"][0]
    C_cf = X @ Al[:, :3].T + Al[:, 3:] @ z_n + l["W"][1] @ l["b"][0] + l["b"][1]
    assert np.allclose(C, C_cf.reshape(-1, 3, 3), rtol=0, atol=1e-12)
    # the same latent twice: the particles are at rest
    _, v0, _ = infer_state(X, z_n, z_n, g, l, dt, mode="exact")
    assert np.all(v0 == 0.0)


def test_integration_set_identity_lattice():
    N, dx = 32, 1.0 / 32
    cells = np.arange(6, 26)
    off = np.array([0.25, 0.75])
    ax = (cells[:, None] + off[None, :]).reshape(-1) * dx
    X = np.stack(np.meshgrid(ax, ax, ax, indexing="ij"), -1).reshape(-1, 3)
    g = identity_net(2)
    assert np.array_equal(field(X, np.zeros(2), g, "exact"), X)
    s = np.argmin(np.linalg.norm(X - (15 + 0.75) * dx, axis=1))   # base (15, 15, 15)
    Nidx, I = integration_set(X, [s], np.zeros(2), g, (N, N, N), dx, mode="exact")
    assert len(I) == 27
    assert len(Nidx) == 10 ** 3
    base = np.floor(X[Nidx] / dx - 0.5).astype(int)
    assert base.min() == 13 and base.max() == 17


def test_integration_set_brute_force():
    rng = np.random.default_rng(6)
    N, dx, r = 16, 1.0 / 16, 3
    g = {"W": [rng.uniform(-0.3, 0.3, (8, 3 + r)), rng.uniform(-0.05, 0.05, (3, 8))],
         "b": [rng.uniform(-0.5, 0.5, 8), np.full(3, 0.5)]}
    X = rng.uniform(0.3, 0.7, size=(400, 3))
    z = rng.normal(size=r)
    S = rng.choice(400, 7, replace=False)
    Nidx, I = integration_set(X, S, z, g, (N, N, N), dx, mode="emulate")
    x = field(X, z, g, "emulate")
    # the definition written out with loops
    I_bf = set()
    for p in S:
        b = [int(np.floor(x[p, a] / dx - 0.5)) for a in range(3)]
        for o in itertools.product(range(3), repeat=3):
            I_bf.add(tuple(b[a] + o[a] for a in range(3)))
    N_bf = []
    for p in range(len(X)):
        b = [int(np.floor(x[p, a] / dx - 0.5)) for a in range(3)]
        if any(tuple(b[a] + o[a] for a in range(3)) in I_bf for o in itertools.product(range(3), repeat=3)):
            N_bf.append(p)
    assert sorted((i * N + j) * N + k for i, j, k in I_bf) == list(I)
    assert N_bf == list(Nidx)
    assert set(S) <= set(Nidx)
    order = ordered_points(Nidx, S)
    assert list(order[:len(S)]) == list(S) and sorted(order) == sorted(Nidx)
    assert len(np.unique(order)) == len(order)


def test_stencil_ids_match_the_transfer_stencil():
    dx = 1.0 / 8
    x = np.array([[0.5 + 0.3 * dx, 0.5, 0.5 - 0.2 * dx]])
    ids = stencil_node_ids(x, (8, 8, 8), dx)
    # base = floor(t - 1/2): t = (4.3, 4.0, 3.8) -> (3, 3, 3)
    assert ids[0, 0] == (3 * 8 + 3) * 8 + 3 and ids[0, -1] == (5 * 8 + 5) * 8 + 5
