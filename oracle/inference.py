"""Network inference and the sample / integration particle sets of the reduced
model (§5.1 lines 251-254 and §5.4), fp64.

Network inference at t_n for particles with reference positions X_p (line 252-253):
    x_p^n = g(X_p, z_n),   v_p^n = (g(X_p, z_n) - g(X_p, z_{n-1})) / dt,   C_p^n = l(X_p, z_n)
with g the deformation field (out 3) and l the affine-velocity field (out 9,
row-major C); both use the stress field's numerics (reading #20, oracle/mlp.py).

Integration set (line 269):
    I = { grid nodes i : exists p in S with N_i(x_p) != 0 },  x_p = g(X_p, z_n)
    N = { p in P : exists i in I with N_i(g(X_p, z_n)) != 0 }
where N_i(x) != 0 is read as "i is one of the 27 stencil nodes base + {0,1,2}^3,
base = floor(x/dx - 1/2)" (reading #33: the quadratic B-spline weight of a
stencil node vanishes only on a measure-zero set).
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
import numpy as np

from .mlp import mlp_forward


def field(X, z, net, mode="emulate"):
    """net(X_p, z) for points X (n, 3) and one latent z (r,): (n, out)."""
    X = np.asarray(X, np.float64)
    z = np.asarray(z, np.float64)
    u = np.concatenate([X, np.broadcast_to(z, (X.shape[0], z.shape[-1]))], axis=1)
    return mlp_forward(u, net["W"], net["b"], mode)


def infer_state(X, z_n, z_prev, g, l, dt, mode="emulate"):
    """Lines 252-253 for one scene: returns x (n,3), v (n,3), C (n,3,3)."""
    x = field(X, z_n, g, mode)
    x_prev = field(X, z_prev, g, mode)
    v = (x - x_prev) / dt
    C = field(X, z_n, l, mode).reshape(-1, 3, 3)
    return x, v, C


def stencil_node_ids(x, grid_res, dx):
    """Linear ids (i N1 + j) N2 + k of the 27 stencil nodes of each point: (n, 27)."""
    x = np.asarray(x, np.float64)
    base = np.floor(x / dx - 0.5).astype(np.int64)
    off = np.array([(a, b, c) for a in range(3) for b in range(3) for c in range(3)], np.int64)
    nodes = base[:, None, :] + off[None, :, :]
    N = np.asarray(grid_res, np.int64)
    return (nodes[..., 0] * N[1] + nodes[..., 1]) * N[2] + nodes[..., 2]


def integration_set(X_all, sample_idx, z_n, g, grid_res, dx, mode="emulate"):
    """Line 269 for one scene: indices (ascending) of N among X_all, and I (sorted node ids).
    sample_idx: indices of S in X_all."""
    X_all = np.asarray(X_all, np.float64)
    xs = field(X_all[np.asarray(sample_idx)], z_n, g, mode)
    I = np.unique(stencil_node_ids(xs, grid_res, dx))
    xp = field(X_all, z_n, g, mode)
    hit = np.isin(stencil_node_ids(xp, grid_res, dx), I).any(axis=1)
    return np.nonzero(hit)[0], I


def ordered_points(N_idx, sample_idx):
    """The point order the GPU uses for a scene: S in the given order, then N \\ S ascending."""
    s = np.asarray(sample_idx, np.int64)
    rest = np.setdiff1d(np.asarray(N_idx, np.int64), s, assume_unique=False)
    return np.concatenate([s, rest])
