"""Neural stress field h(X, z) (§4.2 Eq. (9); network
architecture lines 498-500), fp64.

  u   = (X, z) in R^{3+r}
  h_1 = ELU(W_1 u + b_1)                 (layer-1 input unrounded, reading #20)
  h_k = ELU(W_k r(h_{k-1}) + b_k),  k = 2..L
  y   = W_out r(h_L) + b_out
  tau = sigma_tau * Voigt^{-1}(y),  Voigt order (xx, yy, zz, yz, xz, xy)

ELU(a) = a if a > 0 else exp(a) - 1 (alpha = 1; Clevert et al., cited line 500).
r() = round to bf16 (RNE) in "emulate" mode, identity in "exact" mode.  W_k are
the stored bf16 weight values (inputs, see scenes.xavier_bf16_mlp).
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
import numpy as np

VOIGT = [(0, 0), (1, 1), (2, 2), (1, 2), (0, 2), (0, 1)]


def elu(a):
    a = np.asarray(a, dtype=np.float64)
    return np.where(a > 0.0, a, np.expm1(np.minimum(a, 0.0)))


def round_bf16(a):
    """Round float64 values to the nearest bfloat16 (8 significant bits), ties to
    even; returns float64.  (Normal range only; zero stays zero.)"""
    a = np.asarray(a, dtype=np.float64)
    m, e = np.frexp(a)                 # a = m 2^e, |m| in [0.5, 1)
    q = np.round(m * 256.0) / 256.0    # numpy rounds half to even
    return np.ldexp(q, e)


def mlp_forward(u, Ws, bs, mode="emulate"):
    """u: (n, in_dim).  Ws: list of (out, in) float arrays; bs: list of (out,)."""
    h = np.asarray(u, dtype=np.float64)
    L = len(Ws)
    r = round_bf16 if mode == "emulate" else (lambda t: t)
    for k in range(L):
        W = np.asarray(Ws[k], dtype=np.float64)
        b = np.asarray(bs[k], dtype=np.float64)
        inp = h if k == 0 else r(h)
        a = inp @ W.T + b
        h = elu(a) if k < L - 1 else a
    return h


def voigt_to_matrix(y):
    y = np.asarray(y, dtype=np.float64)
    T = np.zeros(y.shape[:-1] + (3, 3))
    for k, (i, j) in enumerate(VOIGT):
        T[..., i, j] = y[..., k]
        T[..., j, i] = y[..., k]
    return T


def nsf_stress(X, z, mlp, sigma_tau, mode="emulate"):
    """tau_p = sigma_tau * h(X_p, z) for points X (n,3) and one latent z (r,).
    Returns (n,6) Voigt."""
    X = np.asarray(X, dtype=np.float64)
    z = np.asarray(z, dtype=np.float64)
    u = np.concatenate([X, np.broadcast_to(z, (X.shape[0], z.shape[-1]))], axis=1)
    return sigma_tau * mlp_forward(u, mlp["W"], mlp["b"], mode)
