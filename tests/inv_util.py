"""Test helpers for the network-inversion parity (tests/test_gpu_inversion.py):
the seeded scene, and the spread of one Gauss-Newton step under fp32 accumulation.

A GPU evaluates the bf16-emulating network with fp32 accumulation (bf16 x bf16
products are exact in fp32; only the summation rounds).  A different summation
order flips some bf16 rounding decisions of the activations, and the Gauss-Newton
step of a random network is very sensitive to those (reading #37).  So
the parity bar of the GPU step is derived from the spread of correct fp32
evaluations: the oracle's network evaluated here with sequential fp32
accumulation in several summation orders (same rounding points as
oracle/inversion.py), each giving one Gauss-Newton step.
"""
import numpy as np

import oracle.inversion as OI
import scenes
from oracle.mlp import elu, round_bf16


def inversion_scene(n_scenes=3, per_scene=256, seed=3):
    gnet = scenes.deformation_field(77)
    sc = scenes.c5_small(n_scenes=n_scenes, per_scene=per_scene)
    rng = np.random.default_rng(seed)
    z_star = rng.normal(size=(n_scenes, 6)).astype(np.float32)
    x = sc.x.copy()
    for s, (a, b) in enumerate(zip(sc.scene_offsets[:-1], sc.scene_offsets[1:])):
        x[a:b], _ = OI.g_with_tangents(sc.X_ref[a:b], z_star[s], gnet, "emulate")
    sc.x = x.astype(np.float32)
    sc.z0 = (z_star + 0.1 * rng.normal(size=z_star.shape)).astype(np.float32)
    sc.dz = np.zeros_like(sc.z0)
    return sc, gnet, z_star


def _g_tangents_fp32(X, z, mlp, seed):
    """g and dg/dz as oracle.inversion.g_with_tangents("emulate"), but every matmul
    accumulated in fp32, sequentially, in a seeded permutation of the inputs
    (seed 0: natural order); bias added in fp32."""
    X = np.asarray(X, np.float64)
    z = np.asarray(z, np.float64)
    n, r = X.shape[0], z.shape[-1]
    u = np.concatenate([X.astype(np.float32).astype(np.float64), np.broadcast_to(z, (n, r))], axis=1)
    T = np.zeros((n, r, u.shape[1]))
    for k in range(r):
        T[:, k, 3 + k] = 1.0
    rng = np.random.default_rng(seed)
    h = u
    L = len(mlp["W"])
    for k in range(L):
        W = np.asarray(mlp["W"][k], np.float64)
        b = np.asarray(mlp["b"][k], np.float64)
        inp, tin = (h, T) if k == 0 else (round_bf16(h), round_bf16(T))
        order = rng.permutation(W.shape[1]) if seed else np.arange(W.shape[1])
        a = np.zeros(inp.shape[:-1] + (W.shape[0],), np.float32)
        ta = np.zeros(tin.shape[:-1] + (W.shape[0],), np.float32)
        for i in order:
            a = a + (inp[..., i:i + 1] * W[:, i]).astype(np.float32)
            ta = ta + (tin[..., i:i + 1] * W[:, i]).astype(np.float32)
        a = (a + b.astype(np.float32)).astype(np.float64)
        ta = ta.astype(np.float64)
        if k < L - 1:
            h = elu(a)
            d = np.where(a > 0.0, 1.0, np.exp(np.minimum(a, 0.0)))
            T = d[:, None, :] * ta
        else:
            h, T = a, ta
    return h, np.transpose(T, (0, 2, 1))


def fp32_spread(sc, gnet, x, z_start, n_sample, orders=6, per_order=False):
    """Per summation order, |z_fp32 - z_oracle| / |z_oracle - z_start| of one
    Gauss-Newton step; returns (max or list, emulate-vs-exact gap / step)."""
    zo = OI.invert_scenes(sc.X_ref, x, sc.scene_offsets, n_sample, z_start, gnet, 1, "emulate")
    ze = OI.invert_scenes(sc.X_ref, x, sc.scene_offsets, n_sample, z_start, gnet, 1, "exact")
    step = np.linalg.norm(zo - z_start)
    out = []
    orig = OI.g_with_tangents
    try:
        for s in range(orders):
            OI.g_with_tangents = lambda X, z, mlp, mode="emulate", s_=s: _g_tangents_fp32(X, z, mlp, s_)
            zf = OI.invert_scenes(sc.X_ref, x, sc.scene_offsets, n_sample, z_start, gnet, 1, "emulate")
            out.append(float(np.linalg.norm(zf - zo) / step))
    finally:
        OI.g_with_tangents = orig
    gap = float(np.linalg.norm(ze - zo) / step)
    return (out if per_order else max(out)), gap


def fp32_objective_spread(XS, targets, z_start, gnet, iters, orders=8):
    """For one scene: the oracle's Gauss-Newton result z_o from z_start (emulate
    mode, fp64), the Eq. (10) objective at z_start and z_o, and the largest excess
    f(z_fp32) - f(z_o) over `orders` fp32-accumulated evaluations of the same
    network (each running its own Gauss-Newton).  Objectives are evaluated by the
    fp64 emulating oracle."""
    XS = np.asarray(XS, np.float64)
    t = np.asarray(targets, np.float64)
    off = np.array([0, XS.shape[0]])
    n = XS.shape[0]

    def f(z):
        return float(np.sum((OI.g_with_tangents(XS, np.asarray(z, np.float64), gnet, "emulate")[0] - t) ** 2))
    zo = OI.invert_scenes(XS, t, off, n, np.asarray(z_start, np.float64)[None], gnet, iters, "emulate")[0]
    f0, fo = f(z_start), f(zo)
    worst = 0.0
    orig = OI.g_with_tangents
    try:
        for s in range(orders):
            OI.g_with_tangents = lambda X, z, mlp, mode="emulate", s_=s: _g_tangents_fp32(X, z, mlp, s_)
            zf = OI.invert_scenes(XS, t, off, n, np.asarray(z_start, np.float64)[None], gnet, iters, "emulate")[0]
            OI.g_with_tangents = orig
            worst = max(worst, f(zf) - fo)
    finally:
        OI.g_with_tangents = orig
    return zo, f0, fo, worst
