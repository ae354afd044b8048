"""Seeded synthetic inputs shared by the fp64 oracle and the CUDA path.

This module holds NO arithmetic of the method (no B-spline weights, no stress,
no transfer).  It only draws the random numbers the method is fed -- particle
positions, velocities, latent vectors, MLP weights -- and records the
configuration constants of BASELINE.json's five configs (C1..C5) plus a few
small test variants.  Both `oracle/` and `paper_2310_17790_b200/` consume
what it returns; neither imports the other.

Readings (SURVEY.md §8(c) / DESIGN.md "Readings"):
  #10  grid: N nodes per axis, x_i = i*dx, dx = 1/N (a power of two).
  #11  wall region: node index < width (low face) or >= N - width (high face).
  #16  seeding: stratified, each cell's 2x2x2 sub-cells get one jittered point,
       x = (c + (s + u)/2) dx, u ~ U[0,1)^3.  V0 = dx^3/8 unless stated.
  #17  C2/C3: particle counts are binding, body size flexes.
  #18  C4: 64 balls of 125,000 uniform points.
  #19  C5: shared reference set, per-scene subsets of 2,048.
  #20  MLP: Xavier-uniform weights rounded RNE to bf16, biases U(+-1/sqrt(fan_in)).
  #26  C5 latent drift z(n) = z0 + n*dz, dz = 1e-4 * zdot.

Seeds: C1..C5 = 17791..17795; streams are split with
numpy.random.SeedSequence(seed).spawn(k).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, asdict
from typing import Optional

import numpy as np

# ---------------------------------------------------------------------------
# model / bc / force-mode codes (mirror include/nsf_mpm.h enums; plain ints)
FIXED_COROTATED, DRUCKER_PRAGER, VON_MISES, NEURAL_STRESS, HENCKY, HERSCHEL_BULKLEY = 0, 1, 2, 3, 4, 5
TRANSFER_APIC, TRANSFER_PIC, TRANSFER_RPIC = 0, 1, 2
BC_NONE, BC_STICKY, BC_SLIP = 0, 1, 2
FORCE_MLS, FORCE_GRADW = 0, 1

SEEDS = {"C1": 17791, "C2": 17792, "C3": 17793, "C4": 17794, "C5": 17795}


@dataclass
class Config:
    """Plain configuration record (SI units).  No derived quantities."""
    name: str
    grid_res: int                 # nodes per axis (cubic grid), dx = 1/grid_res
    dt: float
    substeps: int
    model: int
    E: float
    nu: float
    rho: float
    friction_angle_deg: float = 30.0
    yield_stress: float = 0.0
    hardening: float = 0.0         # VM hardening coefficient xi
    softening: float = 0.0         # VM softening coefficient theta
    viscosity: float = 0.0         # Herschel-Bulkley eta (Pa s); sigma_Y = yield_stress
    gravity: tuple = (0.0, -9.8, 0.0)
    bc: tuple = (BC_STICKY,) * 6   # faces -x,+x,-y,+y,-z,+z
    bc_width: int = 3
    plate_enabled: int = 0
    plate_y0: float = 0.0
    plate_velocity: tuple = (0.0, 0.0, 0.0)
    force_mode: int = FORCE_MLS
    deterministic: int = 0         # 1: fixed-point (bitwise reproducible) P2G on the GPU
    transfer: int = TRANSFER_APIC  # P2G momentum transfer
    particle_volume: float = 0.0   # <=0 -> dx^3/8
    n_scenes: int = 1
    stress_scale: float = 100.0    # sigma_tau for the NSF output (reading #20)

    @property
    def dx(self) -> float:
        return 1.0 / self.grid_res

    def as_dict(self):
        return asdict(self)


@dataclass
class Scene:
    """Particle state in the caller layout (row-major AoS, float32)."""
    cfg: Config
    x: np.ndarray                  # (n,3)
    v: np.ndarray                  # (n,3)
    C: np.ndarray                  # (n,3,3)
    F: np.ndarray                  # (n,3,3)
    scene_offsets: Optional[np.ndarray] = None   # (n_scenes+1,) int64 (C5)
    X_ref: Optional[np.ndarray] = None           # (n,3) reference positions (C5)
    mlp: Optional[dict] = None                   # C5 network (bf16 bits + fp32 biases)
    z0: Optional[np.ndarray] = None              # (n_scenes, r) float32
    dz: Optional[np.ndarray] = None              # (n_scenes, r) float32

    @property
    def n(self) -> int:
        return int(self.x.shape[0])


# ---------------------------------------------------------------------------
# configs (BASELINE.json "configs", in file order)

def config(name: str) -> Config:
    if name == "C1":
        return Config("C1", 32, 1e-4, 200, FIXED_COROTATED, 1e4, 0.3, 1000.0,
                      bc=(BC_STICKY,) * 6)
    if name == "C2":
        return Config("C2", 128, 5e-5, 1000, DRUCKER_PRAGER, 3.5e5, 0.3, 1600.0,
                      friction_angle_deg=30.0, bc=(BC_SLIP,) * 6)
    if name == "C3":
        n = 256
        return Config("C3", n, 2e-5, 500, VON_MISES, 1e6, 0.3, 3000.0,
                      yield_stress=5e4,
                      bc=(BC_SLIP, BC_SLIP, BC_STICKY, BC_SLIP, BC_SLIP, BC_SLIP),
                      plate_enabled=1, plate_y0=53.0 / n,
                      plate_velocity=(0.0, -0.5, 0.0))
    if name == "C4":
        r = 0.05
        return Config("C4", 512, 1e-5, 100, FIXED_COROTATED, 5e4, 0.35, 1000.0,
                      bc=(BC_SLIP,) * 6,
                      particle_volume=(4.0 / 3.0) * math.pi * r ** 3 / 125000.0)
    if name == "C5":
        return Config("C5", 64, 1e-4, 100, NEURAL_STRESS, 1e4, 0.3, 1000.0,
                      bc=(BC_STICKY,) * 6, particle_volume=0.064 / 200000.0,
                      n_scenes=256, stress_scale=100.0)
    raise KeyError(name)


# ---------------------------------------------------------------------------
# helpers (sampling only)

def _streams(seed: int, k: int):
    return [np.random.default_rng(s) for s in np.random.SeedSequence(seed).spawn(k)]


def stratified_cells(lo, hi, dx: float, rng) -> np.ndarray:
    """8 particles per cell: one per 2x2x2 sub-cell, jittered uniformly.

    lo, hi: integer cell bounds per axis (hi exclusive).  Returns (n,3) float64
    positions in cell order (cell-major, then sub-cell).
    """
    lo = np.asarray(lo, dtype=np.int64)
    hi = np.asarray(hi, dtype=np.int64)
    axes = [np.arange(lo[a], hi[a]) for a in range(3)]
    cells = np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1).reshape(-1, 1, 3)
    sub = np.stack(np.meshgrid([0, 1], [0, 1], [0, 1], indexing="ij"), axis=-1).reshape(1, 8, 3)
    u = rng.random((cells.shape[0], 8, 3))
    x = (cells + (sub + u) * 0.5) * dx
    return x.reshape(-1, 3)


def _finish(cfg, x, v, C=None, F=None, **kw) -> Scene:
    n = x.shape[0]
    if C is None:
        C = np.zeros((n, 3, 3))
    if F is None:
        F = np.broadcast_to(np.eye(3), (n, 3, 3))
    return Scene(cfg=cfg,
                 x=np.ascontiguousarray(x, dtype=np.float32),
                 v=np.ascontiguousarray(v, dtype=np.float32),
                 C=np.ascontiguousarray(C, dtype=np.float32),
                 F=np.ascontiguousarray(F, dtype=np.float32), **kw)


# ---------------------------------------------------------------------------
# the five configs

def c1(seed: int = SEEDS["C1"]) -> Scene:
    """Elastic cube drop: cells [12,20)^3 of 32^3, 8 ppc, v = (0,-1,0)."""
    cfg = config("C1")
    (rx,) = _streams(seed, 1)
    x = stratified_cells((12, 12, 12), (20, 20, 20), cfg.dx, rx)
    v = np.tile([0.0, -1.0, 0.0], (x.shape[0], 1))
    return _finish(cfg, x, v)


def c1_spin(seed: int = SEEDS["C1"], omega=(0.0, 0.0, 5.0), noise=0.1) -> Scene:
    """Test-only variant: C1 plus rigid spin about the cube centre (C0 = [w]x)
    and seeded N(0, noise^2) velocity noise (SURVEY.md §8(c) trajectory bars)."""
    base = c1(seed)
    cfg = base.cfg
    rng = _streams(seed + 1000, 1)[0]
    x = base.x.astype(np.float64)
    centre = np.full(3, 0.5)
    w = np.asarray(omega, dtype=np.float64)
    W = np.array([[0.0, -w[2], w[1]], [w[2], 0.0, -w[0]], [-w[1], w[0], 0.0]])
    v = base.v.astype(np.float64) + (x - centre) @ W.T + rng.normal(0.0, noise, x.shape)
    C = np.broadcast_to(W, (x.shape[0], 3, 3))
    return _finish(cfg, x, v, C)


def c2(seed: int = SEEDS["C2"]) -> Scene:
    """Sand column: cells x,z in [53,75), y in [3,55) of 128^3, seeded 200,000
    of the 201,344 stratified slots (reading #17)."""
    cfg = config("C2")
    rx, rs = _streams(seed, 2)
    x = stratified_cells((53, 3, 53), (75, 55, 75), cfg.dx, rx)
    keep = np.sort(rs.choice(x.shape[0], 200000, replace=False))
    x = x[keep]
    return _finish(cfg, x, np.zeros_like(x))


def c3(seed: int = SEEDS["C3"]) -> Scene:
    """Metal block: cells x,z in [103,153), y in [3,53) of 256^3 = 1,000,000
    particles; rigid plate from y = 53 dx moving at -0.5 m/s."""
    cfg = config("C3")
    (rx,) = _streams(seed, 1)
    x = stratified_cells((103, 3, 103), (153, 53, 153), cfg.dx, rx)
    return _finish(cfg, x, np.zeros_like(x))


def _uniform_ball(rng, n, radius):
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    r = radius * rng.random(n) ** (1.0 / 3.0)
    return d * r[:, None]


def c4(seed: int = SEEDS["C4"], n_balls: int = 64, per_ball: int = 125000) -> Scene:
    """64 fixed-corotated balls (r = 0.05) on 512^3, centres U[0.1,0.9]^3,
    rigid per-ball velocity uniform in the ball |v| <= 2 m/s (reading #18)."""
    cfg = config("C4")
    rc, rv, rp = _streams(seed, 3)
    centres = rc.uniform(0.1, 0.9, size=(n_balls, 3))
    vel = _uniform_ball(rv, n_balls, 2.0)
    x = np.concatenate([centres[b] + _uniform_ball(rp, per_ball, 0.05) for b in range(n_balls)])
    v = np.repeat(vel, per_ball, axis=0)
    return _finish(cfg, x, v)


def xavier_bf16_mlp(rng, dims, bias_rng=None):
    """Random-init MLP per reading #20.

    Weights: Xavier-uniform +-sqrt(6/(fan_in+fan_out)) drawn in fp64 and rounded
    to bf16 (round-to-nearest-even on the fp32 value's top 16 bits).  Biases:
    U(+-1/sqrt(fan_in)) in fp32.  Returned weights are the bf16 bit patterns
    (uint16, layer-major, row-major [out][in]) and their exact float values.
    """
    bias_rng = bias_rng or rng
    Ws_bits, Ws_val, bs = [], [], []
    for fan_in, fan_out in zip(dims[:-1], dims[1:]):
        a = math.sqrt(6.0 / (fan_in + fan_out))
        w = rng.uniform(-a, a, size=(fan_out, fan_in)).astype(np.float32)
        bits = w.view(np.uint32)
        # RNE to the upper 16 bits (values are finite and normal)
        rounded = (bits + np.uint32(0x7FFF) + ((bits >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)
        b16 = rounded.astype(np.uint16)
        Ws_bits.append(b16)
        Ws_val.append((b16.astype(np.uint32) << np.uint32(16)).view(np.float32))
        bb = 1.0 / math.sqrt(fan_in)
        bs.append(bias_rng.uniform(-bb, bb, size=fan_out).astype(np.float32))
    return {"dims": list(dims), "W_bits": Ws_bits, "W": Ws_val, "b": bs}


def c5(seed: int = SEEDS["C5"], n_scenes: int = 256, per_scene: int = 2048,
       n_ref: int = 200000, r: int = 6, width: int = 128, n_hidden: int = 4,
       drift: bool = True) -> Scene:
    """Reduced-order batch (reading #19, #20, #26)."""
    cfg = config("C5")
    cfg.n_scenes = n_scenes
    rref, rsub, rz, rzd, rw, rb = _streams(seed, 6)
    X = rref.uniform(0.3, 0.7, size=(n_ref, 3))
    idx = np.concatenate([np.sort(rsub.choice(n_ref, per_scene, replace=False))
                          for _ in range(n_scenes)])
    x = X[idx]
    z0 = rz.normal(size=(n_scenes, r)).astype(np.float32)
    dz = (1e-4 * rzd.normal(size=(n_scenes, r))).astype(np.float32) if drift \
        else np.zeros((n_scenes, r), np.float32)
    dims = [3 + r] + [width] * n_hidden + [6]
    mlp = xavier_bf16_mlp(rw, dims, rb)
    offsets = np.arange(n_scenes + 1, dtype=np.int64) * per_scene
    sc = _finish(cfg, x, np.zeros_like(x), scene_offsets=offsets,
                 X_ref=np.ascontiguousarray(x, dtype=np.float32), mlp=mlp, z0=z0, dz=dz)
    return sc


def deformation_field(seed: int = SEEDS["C5"] + 1000, r: int = 6, width: int = 128, n_hidden: int = 4) -> dict:
    """Random-init neural deformation field g(X, z) -> x,
    reading #20's initialisation, with the output layer scaled by 1/16 (exact in bf16)
    and its bias set to 0.5 so that g stays inside the unit domain: a stand-in for the
    trained network the network inversion (Eq. (10)) runs on."""
    g = xavier_bf16_mlp(np.random.default_rng(seed), [3 + r] + [width] * n_hidden + [3])
    w = (g["W"][-1] / np.float32(16.0)).astype(np.float32)
    g["W"][-1] = w
    g["W_bits"][-1] = (w.view(np.uint32) >> np.uint32(16)).astype(np.uint16)
    g["b"][-1] = np.full(3, 0.5, np.float32)
    return g


def deformation_field_near_identity(seed: int = SEEDS["C5"] + 3000, r: int = 6, width: int = 128,
                                    n_hidden: int = 4, eps: float = 0.03) -> dict:
    """A random-init deformation field that stays close to the identity, g(X, z) ~ r(X) +
    eps * (random smooth function of X and z), r() = bf16 rounding: hidden units 0..2
    carry X_a through every layer (weight 1, bias 0; X > 0 so ELU is the identity) and
    the output adds eps x reading #20's random output layer (weights rounded to bf16).
    A stand-in for a trained g whose body is not collapsed, for the integration-set
    construction."""
    g = xavier_bf16_mlp(np.random.default_rng(seed), [3 + r] + [width] * n_hidden + [3])
    L = len(g["W"])
    for k in range(L):
        W = g["W"][k].copy()
        b = g["b"][k].copy()
        if k == 0:
            W[:3, :] = 0.0
            W[:3, :3] = np.eye(3, dtype=np.float32)
            b[:3] = 0.0
        elif k < L - 1:
            W[:3, :] = 0.0
            W[:, :3] = 0.0
            W[:3, :3] = np.eye(3, dtype=np.float32)
            b[:3] = 0.0
        else:
            W = W * np.float32(eps)
            W[:, :3] = np.eye(3, dtype=np.float32)
            b[:] = 0.0
        bits = W.astype(np.float32).view(np.uint32)
        rounded = (bits + np.uint32(0x7FFF) + ((bits >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)
        g["W_bits"][k] = rounded.astype(np.uint16)
        g["W"][k] = (g["W_bits"][k].astype(np.uint32) << np.uint32(16)).view(np.float32)
        g["b"][k] = b.astype(np.float32)
    return g


def affine_field(seed: int = SEEDS["C5"] + 2000, r: int = 6, width: int = 128, n_hidden: int = 4) -> dict:
    """Random-init neural affine-velocity field l(X, z) -> C (9, row-major; PAPER.md
    line 253), reading #20's initialisation with the output layer scaled by 1/16 and
    zero output bias: a stand-in for the trained network of network inference."""
    l = xavier_bf16_mlp(np.random.default_rng(seed), [3 + r] + [width] * n_hidden + [9])
    w = (l["W"][-1] / np.float32(16.0)).astype(np.float32)
    l["W"][-1] = w
    l["W_bits"][-1] = (w.view(np.uint32) >> np.uint32(16)).astype(np.uint16)
    l["b"][-1] = np.zeros(9, np.float32)
    return l


def reference_body(seed: int = SEEDS["C5"], n_ref: int = 200000) -> np.ndarray:
    """C5's shared reference body (reading #19): n_ref points U[0.3, 0.7]^3 (the same
    stream c5() draws its per-scene samples from)."""
    rref = _streams(seed, 6)[0]
    return rref.uniform(0.3, 0.7, size=(n_ref, 3))


# ---------------------------------------------------------------------------
# small parity variants (several tiles + ragged tails, oracle-friendly sizes)

def block_scene(name: str, grid_res: int, lo, hi, model: int, seed: int,
                keep: Optional[int] = None, v0=(0.0, 0.0, 0.0), vnoise: float = 0.0,
                Fnoise: float = 0.0, Cnoise: float = 0.0, **cfg_over) -> Scene:
    """Stratified block of cells [lo,hi) on a grid_res^3 grid with optional
    seeded perturbations of v, C and F (used to exercise every branch)."""
    base = {FIXED_COROTATED: config("C1"), DRUCKER_PRAGER: config("C2"),
            VON_MISES: config("C3"), HENCKY: config("C3"), HERSCHEL_BULKLEY: config("C3")}[model]
    cfg = Config(**{**base.as_dict(), "name": name, "grid_res": grid_res, "model": model})
    if model == VON_MISES:
        cfg.plate_y0 = hi[1] / grid_res
    for k, val in cfg_over.items():
        setattr(cfg, k, val)
    rx, rs, rv, rf, rc = _streams(seed, 5)
    x = stratified_cells(lo, hi, cfg.dx, rx)
    if keep is not None and keep < x.shape[0]:
        x = x[np.sort(rs.choice(x.shape[0], keep, replace=False))]
    n = x.shape[0]
    v = np.tile(np.asarray(v0, dtype=np.float64), (n, 1)) + rv.normal(0.0, 1.0, (n, 3)) * vnoise
    C = rc.normal(0.0, 1.0, (n, 3, 3)) * Cnoise
    F = np.eye(3) + rf.normal(0.0, 1.0, (n, 3, 3)) * Fnoise
    return _finish(cfg, x, v, C, F)


def c5_small(seed: int = SEEDS["C5"], n_scenes: int = 3, per_scene: int = 300, **kw) -> Scene:
    return c5(seed, n_scenes=n_scenes, per_scene=per_scene, n_ref=5000, **kw)


def by_name(name: str) -> Scene:
    return {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5, "C1spin": c1_spin}[name]()
