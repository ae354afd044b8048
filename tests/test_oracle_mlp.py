"""Pins for oracle/mlp.py and oracle/reduced.py (CPU only)."""
import json
import os

import numpy as np
import pytest
import torch

import scenes
import oracle
from oracle import mpm
from oracle.mlp import elu, round_bf16, mlp_forward, nsf_stress, voigt_to_matrix

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


@pytest.mark.parametrize("ex", GOLD["elu"])
def test_elu_worked(ex):
    assert elu(np.array(ex["a"])) == pytest.approx(ex["elu"], abs=1e-16)


def test_elu_c1():
    h = 1e-7
    assert (elu(h) - elu(-h)) / (2 * h) == pytest.approx(1.0, abs=1e-6)


def test_round_bf16_vs_torch():
    """Library routine: torch's float32 -> bfloat16 conversion is RNE."""
    rng = np.random.default_rng(0)
    a = (rng.normal(size=100000) * np.exp(rng.normal(size=100000) * 3)).astype(np.float32)
    ref = torch.from_numpy(a).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(round_bf16(a.astype(np.float64)), ref)
    # exact ties go to even
    t = np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8])
    assert np.array_equal(round_bf16(t), [1.0, 1.0 + 4 * 2 ** -8])


def test_mlp_vs_torch_fp64():
    """mlp_forward equals a torch fp64 Linear/ELU stack with the same weights, with the
    bf16 rounding points applied in the same places (reading #20)."""
    sc = scenes.c5_small()
    mlp = sc.mlp
    rng = np.random.default_rng(1)
    u = rng.normal(size=(500, 9))
    for mode in ("exact", "emulate"):
        h = torch.from_numpy(u)
        L = len(mlp["W"])
        for k in range(L):
            W = torch.from_numpy(mlp["W"][k].astype(np.float64))
            b = torch.from_numpy(mlp["b"][k].astype(np.float64))
            inp = h if (k == 0 or mode == "exact") else h.float().to(torch.bfloat16).double()
            a = torch.nn.functional.linear(inp, W, b)
            h = torch.nn.functional.elu(a) if k < L - 1 else a
        ours = mlp_forward(u, mlp["W"], mlp["b"], mode)
        if mode == "exact":
            assert np.allclose(ours, h.numpy(), rtol=1e-12, atol=1e-12)
        else:
            # torch rounds fp64 -> fp32 -> bf16 (double rounding), so only the coarse
            # agreement is checked here; test_mlp_emulate_rounding_points_exact pins
            # the emulate mode exactly against a bit-level single rounding
            assert np.allclose(ours, h.numpy(), rtol=1e-2, atol=1e-2)


def _bf16_rne_bits(t):
    """Independent fp64 -> bf16 round-to-nearest-even on the IEEE bit pattern:
    keep the sign, exponent and top 7 of the 52 stored mantissa bits, add half an
    ulp minus one plus the kept lsb, truncate (the carry runs into the exponent as
    it should).  Also returns, per element, the distance of the dropped bits from
    the tie point 2^44 (small = a rounding decision within summation-order noise)."""
    b = t.contiguous().view(torch.int64)
    drop = b & ((1 << 45) - 1)
    lsb = (b >> 45) & 1
    r = (b + ((1 << 44) - 1) + lsb) & ~((1 << 45) - 1)
    return r.view(torch.float64), (drop - (1 << 44)).abs()


def _emulate_torch(u, Ws, bs, where="after_elu", round_input=False):
    """The emulate-mode MLP (reading #20) in torch fp64 with the rounding points
    written out: u -> a_1 = W_1 u + b_1 -> h_1 = ELU(a_1) -> r(h_1) -> a_2 ... ->
    y = W_L r(h_{L-1}) + b_L.  `where` / `round_input` move the rounding points
    (mutations used to show that the pin below detects them)."""
    h = torch.from_numpy(np.asarray(u, np.float64))
    near = torch.full((h.shape[0],), 1 << 62, dtype=torch.int64)
    L = len(Ws)

    def rnd(t):
        nonlocal near
        r, d = _bf16_rne_bits(t)
        near = torch.minimum(near, d.reshape(t.shape[0], -1).min(dim=1).values)
        return r

    for k in range(L):
        W = torch.from_numpy(np.asarray(Ws[k], np.float64))
        b = torch.from_numpy(np.asarray(bs[k], np.float64))
        inp = h
        if (k > 0 and where == "after_elu") or (k == 0 and round_input):
            inp = rnd(h)
        a = torch.nn.functional.linear(inp, W, b)
        if k < L - 1:
            if where == "before_elu":
                a = rnd(a)
            h = torch.nn.functional.elu(a)
        else:
            h = a
    return h.numpy(), near.numpy()


def test_mlp_emulate_rounding_points_exact():
    """The emulate mode's rounding points, pinned exactly: mlp_forward(emulate) equals
    an independent torch fp64 implementation with a bit-level fp64 -> bf16 RNE to
    1e-12 on every row whose rounding decisions are not within 2^-40 relative of a
    tie (summation-order noise could flip those; they must be rare).  Moving a
    rounding point (before the ELU, on the layer-1 input, or dropping one) changes
    the result by far more than the pin allows."""
    sc = scenes.c5_small()
    Ws, bs = sc.mlp["W"], sc.mlp["b"]
    rng = np.random.default_rng(7)
    X = rng.uniform(0.3, 0.7, size=(2000, 3))
    u = np.concatenate([X, rng.normal(size=(2000, 6))], axis=1)
    ours = mlp_forward(u, Ws, bs, "emulate")
    ref, near = _emulate_torch(u, Ws, bs)
    clean = near > (1 << 12)
    assert clean.mean() >= 0.99, clean.mean()
    scale = np.max(np.abs(ref))
    assert np.max(np.abs(ours[clean] - ref[clean])) <= 1e-12 * scale
    # the round_bf16 used by the oracle agrees with the bit-level rounding everywhere
    t = torch.from_numpy(rng.normal(size=100000) * np.exp(rng.normal(size=100000) * 5))
    assert np.array_equal(round_bf16(t.numpy()), _bf16_rne_bits(t)[0].numpy())
    # sensitivity: each misplaced rounding point moves the output by >> 1e-12
    for kw in ({"where": "before_elu"}, {"round_input": True}, {"where": "none"}):
        mut, _ = _emulate_torch(u, Ws, bs, **kw)
        assert np.max(np.abs(mut - ref)) > 1e-6 * scale, kw


def test_mlp_special_cases():
    rng = np.random.default_rng(2)
    dims = [9, 16, 16, 6]
    Ws = [np.zeros((o, i)) for i, o in zip(dims[:-1], dims[1:])]
    bs = [rng.normal(size=o) for o in dims[1:]]
    u = rng.normal(size=(10, 9))
    assert np.allclose(mlp_forward(u, Ws, bs), bs[-1])
    W = rng.normal(size=(6, 9))
    b = rng.normal(size=6)
    assert np.allclose(mlp_forward(u, [W], [b]), u @ W.T + b)


def test_voigt_order():
    y = np.arange(1, 7, dtype=float)
    T = voigt_to_matrix(y)
    assert np.array_equal(T, [[1, 6, 5], [6, 2, 4], [5, 4, 3]])


def test_nsf_stress_scale():
    sc = scenes.c5_small()
    X = sc.X_ref[:5]
    t1 = nsf_stress(X, sc.z0[0], sc.mlp, 1.0)
    t100 = nsf_stress(X, sc.z0[0], sc.mlp, 100.0)
    assert np.allclose(t100, 100 * t1)


def test_reduced_zero_stress_is_free_fall():
    """With tau = 0 the reduced step is the full-order step with zero stress: points
    away from the walls fall freely (closed form)."""
    sc = scenes.c5_small(n_scenes=2, per_scene=50)
    P = mpm.params_from_config(sc.cfg)
    st = {"x": sc.x, "v": sc.v, "C": sc.C}
    zero = {"W": [np.zeros_like(w) for w in sc.mlp["W"]], "b": [np.zeros_like(b) for b in sc.mlp["b"]]}
    K = 20
    s = oracle.reduced_run(st, P, sc.scene_offsets, sc.X_ref, zero, 100.0, sc.z0, sc.dz, K)
    g, dt = sc.cfg.gravity[1], sc.cfg.dt
    assert np.allclose(s["v"][:, 1], K * dt * g, atol=1e-12)
    assert np.allclose(s["x"][:, 1], sc.x[:, 1] + dt ** 2 * g * K * (K + 1) / 2, atol=1e-13)


def test_reduced_matches_full_order_mpm_part():
    """The reduced step's MPM part is the full-order P2G/grid/G2P with the given tau."""
    sc = scenes.c5_small(n_scenes=2, per_scene=80)
    P = mpm.params_from_config(sc.cfg)
    rng = np.random.default_rng(3)
    st = {"x": sc.x, "v": rng.normal(size=sc.x.shape) * 0.1, "C": np.zeros((sc.n, 3, 3))}
    out = oracle.reduced_substep(st, P, sc.scene_offsets, sc.X_ref, sc.mlp, 100.0,
                                 sc.z0, sc.dz, step=3)
    for s in range(2):
        a, b = sc.scene_offsets[s], sc.scene_offsets[s + 1]
        tau = voigt_to_matrix(out["tau"][a:b])
        Pfc = mpm.Params(**{**P.__dict__, "model": 0})
        full = mpm.substep({"x": sc.x[a:b], "v": st["v"][a:b], "C": st["C"][a:b],
                            "F": np.broadcast_to(np.eye(3), (b - a, 3, 3)), "tau": tau}, Pfc, 3)
        assert np.allclose(full["x"], out["x"][a:b], rtol=0, atol=1e-15)
        assert np.allclose(full["C"], out["C"][a:b], rtol=1e-13, atol=1e-12)
    z3 = sc.z0[1].astype(np.float64) + 3 * sc.dz[1].astype(np.float64)
    assert np.allclose(out["tau"][a:b], nsf_stress(sc.X_ref[a:b], z3, sc.mlp, 100.0))
