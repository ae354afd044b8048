"""Network inversion (§5.3, Eq. (10)), fp64.

    z_{n+1} = argmin_z  sum_{p in S} || g(X_p, z) - x_p^{n+1} ||_2^2

solved per scene by Gauss-Newton from z_n (line 263: "converging in 2-3
iterations"; one iteration is the first-order Taylor variant of the same
line).  g is the neural deformation field (lines 204-209, architecture lines
498-500: input 3 + r, output 3, ELU hidden layers), here with the same
numerics as the stress field (reading #20): bf16 weights, layer-1 input fp32,
hidden activations rounded to bf16 (RNE) before each later layer, fp32 bias and
ELU ("emulate"), or no rounding at all ("exact").

The Jacobian dg/dz is propagated in forward mode alongside the activations:
tangent of the layer-1 input = unit vector e_{3+k}; through a hidden layer
t <- ELU'(a) * (W r(t)) with ELU'(a) = 1 (a > 0) else exp(a), the primal
pre-activation a; the output layer is linear.  In "emulate" mode the tangents
are rounded to bf16 at the same points as the activations (the GPU keeps them
in the same bf16 operand tiles).

Normal equations in fp64: H = sum_p J_p^T J_p, g = sum_p J_p^T (g_p - x_p),
z <- z - H^-1 g.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
import numpy as np

from oracle.mlp import elu, round_bf16


def g_with_tangents(X, z, mlp, mode="emulate"):
    """Values g(X_p, z) (n, out) and Jacobians dg/dz (n, out, r)."""
    X = np.asarray(X, dtype=np.float64)
    z = np.asarray(z, dtype=np.float64)
    n, r = X.shape[0], z.shape[-1]
    u = np.concatenate([X, np.broadcast_to(z, (n, r))], axis=1)
    T = np.zeros((n, r, u.shape[1]))
    for k in range(r):
        T[:, k, 3 + k] = 1.0
    rnd = round_bf16 if mode == "emulate" else (lambda t: t)
    h = u
    L = len(mlp["W"])
    for k in range(L):
        W = np.asarray(mlp["W"][k], dtype=np.float64)
        b = np.asarray(mlp["b"][k], dtype=np.float64)
        inp, tin = (h, T) if k == 0 else (rnd(h), rnd(T))
        a = inp @ W.T + b
        ta = tin @ W.T
        if k < L - 1:
            h = elu(a)
            d = np.where(a > 0.0, 1.0, np.exp(np.minimum(a, 0.0)))
            T = d[:, None, :] * ta
        else:
            h, T = a, ta
    return h, np.transpose(T, (0, 2, 1))


def gauss_newton(X, x_target, z0, mlp, iters, mode="emulate"):
    """Gauss-Newton for one scene: returns (z, list of residual norms before each iteration)."""
    z = np.asarray(z0, dtype=np.float64).copy()
    res_norms = []
    for _ in range(iters):
        g, J = g_with_tangents(X, z, mlp, mode)
        res = g - np.asarray(x_target, dtype=np.float64)
        res_norms.append(float(np.linalg.norm(res)))
        H = np.einsum("pik,pil->kl", J, J)
        grad = np.einsum("pik,pi->k", J, res)
        z = z - np.linalg.solve(H, grad)
    return z, res_norms


def invert_scenes(X_ref, x, scene_offsets, n_sample, z0, mlp, iters, mode="emulate"):
    """Per scene s, sample = its first n_sample points (load order); returns (n_scenes, r)."""
    out = []
    for s, (a, b) in enumerate(zip(scene_offsets[:-1], scene_offsets[1:])):
        m = min(n_sample, int(b - a))
        zs, _ = gauss_newton(X_ref[a:a + m], x[a:a + m], z0[s], mlp, iters, mode)
        out.append(zs)
    return np.array(out)
