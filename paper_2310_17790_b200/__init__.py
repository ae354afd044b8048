"""Python binding of the nsf_mpm C ABI (include/nsf_mpm.h).

Argument marshalling only: every step of the substep runs in the CUDA kernels
of libnsf_mpm.so (sm_100a).  There is no CPU fallback: importing this package
without the built library, or calling it without a CUDA device, raises.

Functions keep the C names (nsf_mpm_create, nsf_mpm_load_particles, ...).
Arrays may be numpy arrays (host, on_device=0) or torch CUDA tensors
(on_device=1); torch supplies device memory and the stream.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NSF_MPM_LIB") or os.path.join(_PKG, "libnsf_mpm.so")   # override: A/B of library builds

NSF_OK, NSF_ERR_INVALID_ARGUMENT, NSF_ERR_OUT_OF_DOMAIN, NSF_ERR_NONFINITE, NSF_ERR_CUDA, \
    NSF_ERR_OUT_OF_MEMORY, NSF_ERR_BAD_STATE = range(7)
STATUS_NAMES = ["NSF_OK", "NSF_ERR_INVALID_ARGUMENT", "NSF_ERR_OUT_OF_DOMAIN", "NSF_ERR_NONFINITE",
                "NSF_ERR_CUDA", "NSF_ERR_OUT_OF_MEMORY", "NSF_ERR_BAD_STATE"]
NSF_FIXED_COROTATED, NSF_DRUCKER_PRAGER, NSF_VON_MISES, NSF_NEURAL_STRESS, NSF_HENCKY, NSF_HERSCHEL_BULKLEY = range(6)
NSF_TRANSFER_APIC, NSF_TRANSFER_PIC, NSF_TRANSFER_RPIC = range(3)
NSF_BC_NONE, NSF_BC_STICKY, NSF_BC_SLIP = range(3)
NSF_FORCE_MLS, NSF_FORCE_GRADW = range(2)
NSF_FIELD_X, NSF_FIELD_V, NSF_FIELD_C, NSF_FIELD_F, NSF_FIELD_TAU, NSF_FIELD_TAU_Y = 1, 2, 4, 8, 16, 32
FIELD_SHAPES = {NSF_FIELD_X: (3,), NSF_FIELD_V: (3,), NSF_FIELD_C: (3, 3), NSF_FIELD_F: (3, 3),
                NSF_FIELD_TAU: (6,), NSF_FIELD_TAU_Y: ()}

EXPORTS = ["nsf_mpm_abi_version", "nsf_mpm_create", "nsf_mpm_set_stream", "nsf_mpm_set_allocator",
           "nsf_mpm_load_particles", "nsf_mpm_load_stress_field", "nsf_mpm_set_latents",
           "nsf_mpm_load_deformation_field", "nsf_mpm_invert_latents",
           "nsf_mpm_load_affine_field", "nsf_mpm_infer_state", "nsf_mpm_build_integration_set",
           "nsf_mpm_substep", "nsf_mpm_eval_stress_field", "nsf_mpm_read_state", "nsf_mpm_sync",
           "nsf_mpm_step_count", "nsf_mpm_inverted_count", "nsf_mpm_last_error", "nsf_mpm_destroy",
           "nsf_mpm_debug_bins", "nsf_mpm_debug_grid", "nsf_mpm_set_profiling",
           "nsf_mpm_kernel_times", "nsf_mpm_launches_per_substep", "nsf_mpm_launch_count", "nsf_mpm_rom_step",
           "nsf_mpm_debug_stats"]


class nsf_material(C.Structure):
    _fields_ = [("model", C.c_int32), ("E", C.c_double), ("nu", C.c_double), ("rho", C.c_double),
                ("friction_angle_deg", C.c_double), ("yield_stress", C.c_double),
                ("gravity", C.c_double * 3), ("bc", C.c_int32 * 6), ("bc_width", C.c_int32),
                ("plate_enabled", C.c_int32), ("plate_y0", C.c_double),
                ("plate_velocity", C.c_double * 3), ("force_mode", C.c_int32),
                ("deterministic", C.c_int32), ("n_scenes", C.c_int32),
                ("particle_volume", C.c_double), ("stress_scale", C.c_double), ("transfer", C.c_int32),
                ("hardening", C.c_double), ("softening", C.c_double), ("viscosity", C.c_double)]


class NsfError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 7 else status}: {msg}")
        self.status = status


_lib = None
ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)


def lib():
    """Load libnsf_mpm.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing; run `python -m paper_2310_17790_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, u32, dp = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.POINTER
    sig = {
        "nsf_mpm_abi_version": (i32, []),
        "nsf_mpm_create": (i32, [dp(i32), C.c_double, C.c_double, dp(nsf_material), dp(vp)]),
        "nsf_mpm_set_stream": (i32, [vp, vp]),
        "nsf_mpm_set_allocator": (i32, [vp, ALLOC_FN, FREE_FN, vp]),
        "nsf_mpm_load_particles": (i32, [vp, i64, vp, vp, vp, vp, vp, i32]),
        "nsf_mpm_load_stress_field": (i32, [vp, i32, i32, i32, i32, vp, vp, vp, i32]),
        "nsf_mpm_set_latents": (i32, [vp, i32, vp, vp, i32]),
        "nsf_mpm_load_deformation_field": (i32, [vp, i32, i32, i32, i32, vp, vp, i32]),
        "nsf_mpm_invert_latents": (i32, [vp, i32, i32, vp, i32]),
        "nsf_mpm_load_affine_field": (i32, [vp, i32, i32, i32, i32, vp, vp, i32]),
        "nsf_mpm_infer_state": (i32, [vp, vp, i32]),
        "nsf_mpm_build_integration_set": (i32, [vp, i64, vp, i32, vp, vp, dp(i64), i32]),
        "nsf_mpm_rom_step": (i32, [vp, i64, vp, i32, vp, vp, i32, vp, dp(i64), i32]),
        "nsf_mpm_debug_stats": (i32, [vp, dp(i64), i32]),
        "nsf_mpm_substep": (i32, [vp, i32]),
        "nsf_mpm_eval_stress_field": (i32, [vp, vp, i64, vp, vp, i32]),
        "nsf_mpm_read_state": (i32, [vp, u32, dp(vp), i32]),
        "nsf_mpm_sync": (i32, [vp]),
        "nsf_mpm_step_count": (i64, [vp]),
        "nsf_mpm_inverted_count": (i64, [vp]),
        "nsf_mpm_last_error": (C.c_char_p, [vp]),
        "nsf_mpm_destroy": (None, [vp]),
        "nsf_mpm_debug_bins": (i32, [vp, vp, vp, i32]),
        "nsf_mpm_debug_grid": (i32, [vp, i32, vp, i32]),
        "nsf_mpm_set_profiling": (i32, [vp, i32]),
        "nsf_mpm_kernel_times": (i32, [vp, dp(C.c_char_p), dp(C.c_double), dp(i64), i32]),
        "nsf_mpm_launches_per_substep": (i32, [vp]),
        "nsf_mpm_launch_count": (i64, [vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


# ---------------------------------------------------------------------------
# marshalling helpers

def _is_torch(a):
    return type(a).__module__.startswith("torch")


def _ptr(a, dtype=np.float32):
    """(pointer, on_device, keepalive) for a numpy array / torch tensor / None.

    For CUDA tensors torch's current stream is synchronised first, so the data
    is complete before the library's stream reads it (header: on_device
    pointers must be stream-ordered with the handle's stream)."""
    if a is None:
        return None, None, None
    if _is_torch(a):
        import torch
        if not a.is_contiguous():
            a = a.contiguous()
        if a.is_cuda:
            torch.cuda.current_stream(a.device).synchronize()
        return a.data_ptr(), (1 if a.is_cuda else 0), a
    arr = np.ascontiguousarray(a, dtype=dtype)
    return arr.ctypes.data, 0, arr


def _check(h, status):
    if status != NSF_OK:
        msg = lib().nsf_mpm_last_error(h)
        raise NsfError(status, msg.decode() if msg else "")


def _same_residency(*flags):
    f = [x for x in flags if x is not None]
    if len(set(f)) > 1:
        raise ValueError("mix of host and device arrays in one call")
    return f[0] if f else 0


def make_material(cfg) -> nsf_material:
    """nsf_material from a scenes.Config-like object (attribute access)."""
    m = nsf_material()
    m.model = cfg.model
    m.E, m.nu, m.rho = cfg.E, cfg.nu, cfg.rho
    m.friction_angle_deg = cfg.friction_angle_deg
    m.yield_stress = cfg.yield_stress
    m.gravity = (C.c_double * 3)(*cfg.gravity)
    m.bc = (C.c_int32 * 6)(*cfg.bc)
    m.bc_width = cfg.bc_width
    m.plate_enabled = cfg.plate_enabled
    m.plate_y0 = cfg.plate_y0
    m.plate_velocity = (C.c_double * 3)(*cfg.plate_velocity)
    m.force_mode = cfg.force_mode
    m.deterministic = int(getattr(cfg, "deterministic", 0))
    m.n_scenes = cfg.n_scenes
    m.particle_volume = cfg.particle_volume
    m.stress_scale = cfg.stress_scale
    m.transfer = int(getattr(cfg, "transfer", 0))
    m.hardening = float(getattr(cfg, "hardening", 0.0))
    m.softening = float(getattr(cfg, "softening", 0.0))
    m.viscosity = float(getattr(cfg, "viscosity", 0.0))
    return m


# ---------------------------------------------------------------------------
# the C names

def nsf_mpm_abi_version() -> int:
    return lib().nsf_mpm_abi_version()


def nsf_mpm_create(grid_res: Sequence[int], dx: float, dt: float, material: nsf_material):
    h = C.c_void_p()
    gr = (C.c_int32 * 3)(*grid_res)
    st = lib().nsf_mpm_create(gr, float(dx), float(dt), C.byref(material), C.byref(h))
    if st != NSF_OK:
        raise NsfError(st, "nsf_mpm_create rejected the arguments")
    return h


def nsf_mpm_set_stream(h, stream_ptr: int):
    _check(h, lib().nsf_mpm_set_stream(h, C.c_void_p(stream_ptr)))


def nsf_mpm_set_allocator(h, alloc, release, ctx=None):
    _check(h, lib().nsf_mpm_set_allocator(h, alloc, release, ctx))


def nsf_mpm_load_particles(h, x, v, Cm=None, F=None, scene_offsets=None):
    n = int(x.shape[0])
    px, dx_, kx = _ptr(x)
    pv, dv, kv = _ptr(v)
    pc, dc, kc = _ptr(Cm)
    pf, df, kf = _ptr(F)
    po, _, ko = (None, None, None) if scene_offsets is None else _ptr(
        np.asarray(scene_offsets, dtype=np.int64), np.int64)
    on = _same_residency(dx_, dv, dc, df)
    if scene_offsets is not None and _is_torch(scene_offsets):
        po, don, ko = _ptr(scene_offsets, np.int64)
        if don != on:
            raise ValueError("scene_offsets residency must match x")
    _check(h, lib().nsf_mpm_load_particles(h, n, px, pv, pc, pf, po, on))


def nsf_mpm_load_stress_field(h, in_dim, width, n_hidden, out_dim, W_bf16, b, X_ref=None):
    pw, dw, kw = _ptr(W_bf16, np.uint16)
    pb, db, kb = _ptr(b)
    px, dx_, kx = _ptr(X_ref)
    on = _same_residency(dw, db, dx_)
    _check(h, lib().nsf_mpm_load_stress_field(h, in_dim, width, n_hidden, out_dim, pw, pb, px, on))


def nsf_mpm_set_latents(h, r, z, dz=None):
    pz, dzn, kz = _ptr(z)
    pd, ddn, kd = _ptr(dz)
    on = _same_residency(dzn, ddn)
    _check(h, lib().nsf_mpm_set_latents(h, r, pz, pd, on))


def nsf_mpm_load_deformation_field(h, in_dim, width, n_hidden, out_dim, W_bf16, b):
    pw, dw, kw = _ptr(W_bf16, np.uint16)
    pb, db, kb = _ptr(b)
    on = _same_residency(dw, db)
    _check(h, lib().nsf_mpm_load_deformation_field(h, in_dim, width, n_hidden, out_dim, pw, pb, on))


def nsf_mpm_load_affine_field(h, in_dim, width, n_hidden, out_dim, W_bf16, b):
    pw, dw, kw = _ptr(W_bf16, np.uint16)
    pb, db, kb = _ptr(b)
    on = _same_residency(dw, db)
    _check(h, lib().nsf_mpm_load_affine_field(h, in_dim, width, n_hidden, out_dim, pw, pb, on))


def nsf_mpm_infer_state(h, z_prev=None):
    """Network inference x, v, C (header); z_prev: None or n_scenes x r (numpy / CUDA tensor)."""
    pz, dz_, kz = _ptr(z_prev)
    _check(h, lib().nsf_mpm_infer_state(h, pz, dz_ or 0))


def nsf_mpm_build_integration_set(h, X_all, sample_idx, z_prev=None, n_scenes=1):
    """Sample / integration particles (header).  X_all: n_ref x 3; sample_idx: n_scenes x
    n_sample int32 (numpy, or both CUDA tensors).  Returns |N_s| per scene (numpy int64)."""
    px, dx_, kx = _ptr(X_all)
    ps, ds, ks = _ptr(sample_idx, np.int32)
    pz, dzz, kz = _ptr(z_prev)
    on = _same_residency(dx_, ds, dzz) if z_prev is not None else _same_residency(dx_, ds)
    n_ref = int(X_all.shape[0])
    n_sample = int(np.prod(sample_idx.shape)) // n_scenes
    counts = (C.c_int64 * n_scenes)()
    _check(h, lib().nsf_mpm_build_integration_set(h, n_ref, px, n_sample, ps, pz, counts, on))
    return np.array(counts[:], dtype=np.int64)


def nsf_mpm_rom_step(h, X_all, sample_idx, gn_iters: int, n_scenes: int, r: int, z_prev=None):
    """One reduced-model time step (inference on N -> substep -> inversion; header).
    X_all: n_ref x 3, sample_idx: n_scenes x n_sample (numpy).  Returns (z_{n+1}
    (n_scenes, r) float32, |N_s| (n_scenes,) int64)."""
    X_all = np.ascontiguousarray(X_all, dtype=np.float32)
    sidx = np.ascontiguousarray(sample_idx, dtype=np.int32)
    n_sample = int(np.prod(sidx.shape)) // n_scenes
    z = np.empty((n_scenes, r), dtype=np.float32)
    counts = (C.c_int64 * n_scenes)()
    zp = None if z_prev is None else np.ascontiguousarray(z_prev, dtype=np.float32)
    _check(h, lib().nsf_mpm_rom_step(h, X_all.shape[0], X_all.ctypes.data, n_sample, sidx.ctypes.data,
                                     None if zp is None else zp.ctypes.data, gn_iters, z.ctypes.data, counts, 0))
    return z, np.array(counts[:], dtype=np.int64)


STAT_NAMES = ["segments", "particles", "staged", "listed", "inline", "out_of_tile", "passes", "cyc_tile",
              "cyc_phase1", "cyc_phase2", "out_of_block", "cyc_p2_acc", "cyc_p2_help", "tail_ns", "kern_ns", "ctas"]


def nsf_mpm_debug_stats(h) -> dict:
    """Work counters of the statistics build (header); raises NsfError otherwise."""
    out = (C.c_int64 * 16)()
    _check(h, lib().nsf_mpm_debug_stats(h, out, 16))
    return {k: int(out[i]) for i, k in enumerate(STAT_NAMES)}


def nsf_mpm_invert_latents(h, n_sample: int, n_iters: int, z_out=None):
    """Gauss-Newton network inversion (header).  z_out: None, a float32 numpy array
    (n_scenes x r) or a CUDA tensor, filled with z_hat."""
    po, don, ko = _ptr(z_out)
    _check(h, lib().nsf_mpm_invert_latents(h, int(n_sample), int(n_iters), po, don or 0))
    return z_out


def nsf_mpm_substep(h, n: int):
    _check(h, lib().nsf_mpm_substep(h, int(n)))


def nsf_mpm_eval_stress_field(h, z, points, out=None):
    m = int(points.shape[0])
    pp, dpn, kp = _ptr(points)
    pz, dzn, kz = _ptr(z)
    on = _same_residency(dpn, dzn)
    if out is None:
        if on:
            import torch
            out = torch.empty((m, 6), dtype=torch.float32, device=points.device)
        else:
            out = np.empty((m, 6), dtype=np.float32)
    po, don, ko = _ptr(out)
    _check(h, lib().nsf_mpm_eval_stress_field(h, pz, m, pp, po, on))
    return out


def nsf_mpm_read_state(h, mask: int, n: int, device=None):
    """Returns a list of arrays (numpy if device is None, else torch tensors on it)."""
    outs = []
    for bit in (1, 2, 4, 8, 16, 32):
        if mask & bit:
            shape = (n,) + FIELD_SHAPES[bit]
            if device is None:
                outs.append(np.empty(shape, dtype=np.float32))
            else:
                import torch
                outs.append(torch.empty(shape, dtype=torch.float32, device=device))
    ptrs = (C.c_void_p * len(outs))(*[(o.data_ptr() if device is not None else o.ctypes.data) for o in outs])
    _check(h, lib().nsf_mpm_read_state(h, mask, ptrs, 1 if device is not None else 0))
    return outs


def nsf_mpm_sync(h):
    _check(h, lib().nsf_mpm_sync(h))


def nsf_mpm_step_count(h) -> int:
    return lib().nsf_mpm_step_count(h)


def nsf_mpm_inverted_count(h) -> int:
    return lib().nsf_mpm_inverted_count(h)


def nsf_mpm_last_error(h) -> str:
    s = lib().nsf_mpm_last_error(h)
    return s.decode() if s else ""


def nsf_mpm_destroy(h):
    lib().nsf_mpm_destroy(h)


def nsf_mpm_debug_bins(h, n_blocks: int, n: int):
    counts = np.empty(n_blocks, dtype=np.int32)
    perm = np.empty(max(n, 1), dtype=np.int32)
    _check(h, lib().nsf_mpm_debug_bins(h, counts.ctypes.data, perm.ctypes.data, 0))
    return counts, perm[:n]


def nsf_mpm_debug_grid(h, stage: int, n_scenes: int, N: Sequence[int]):
    out = np.empty((n_scenes, N[0], N[1], N[2], 4), dtype=np.float32)
    _check(h, lib().nsf_mpm_debug_grid(h, stage, out.ctypes.data, 0))
    return out


def nsf_mpm_set_profiling(h, enable: bool):
    _check(h, lib().nsf_mpm_set_profiling(h, 1 if enable else 0))


def nsf_mpm_kernel_times(h) -> dict:
    k = lib().nsf_mpm_kernel_times(h, None, None, None, 0)
    names = (C.c_char_p * max(k, 1))()
    ms = (C.c_double * max(k, 1))()
    cnt = (C.c_int64 * max(k, 1))()
    lib().nsf_mpm_kernel_times(h, names, ms, cnt, k)
    return {names[i].decode(): (ms[i], cnt[i]) for i in range(k)}


def nsf_mpm_launches_per_substep(h) -> int:
    return lib().nsf_mpm_launches_per_substep(h)


def nsf_mpm_launch_count(h) -> int:
    return lib().nsf_mpm_launch_count(h)


# ---------------------------------------------------------------------------
class Simulator:
    """Thin owner of a handle (create/destroy + the calls above)."""

    def __init__(self, cfg, stream: Optional[int] = None, torch_allocator: bool = False):
        self.cfg = cfg
        self.N = (cfg.grid_res,) * 3
        self.h = nsf_mpm_create(self.N, 1.0 / cfg.grid_res, cfg.dt, make_material(cfg))
        self.n = 0
        self._keep = []
        if stream is not None:
            nsf_mpm_set_stream(self.h, stream)
        if torch_allocator:
            self._use_torch_allocator()

    def _use_torch_allocator(self):
        import torch

        def _alloc(nbytes, stream, ctx):
            return torch.cuda.caching_allocator_alloc(int(nbytes), stream=stream or 0)

        def _free(ptr, stream, ctx):
            torch.cuda.caching_allocator_delete(ptr)

        a, f = ALLOC_FN(_alloc), FREE_FN(_free)
        self._keep += [a, f]
        nsf_mpm_set_allocator(self.h, a, f)

    def load(self, x, v, Cm=None, F=None, scene_offsets=None):
        nsf_mpm_load_particles(self.h, x, v, Cm, F, scene_offsets)
        self.n = int(x.shape[0])

    def load_scene(self, sc):
        self.load(sc.x, sc.v, sc.C, sc.F, sc.scene_offsets)
        if sc.mlp is not None:
            dims = sc.mlp["dims"]
            W = np.concatenate([w.reshape(-1) for w in sc.mlp["W_bits"]])
            b = np.concatenate(sc.mlp["b"])
            nsf_mpm_load_stress_field(self.h, dims[0], dims[1], len(dims) - 2, dims[-1], W, b, sc.X_ref)
            nsf_mpm_set_latents(self.h, dims[0] - 3, sc.z0, sc.dz)

    def substep(self, n=1):
        nsf_mpm_substep(self.h, n)

    def load_deformation_field(self, mlp):
        dims = mlp["dims"]
        W = np.concatenate([w.reshape(-1) for w in mlp["W_bits"]])
        b = np.concatenate(mlp["b"])
        nsf_mpm_load_deformation_field(self.h, dims[0], dims[1], len(dims) - 2, dims[-1], W, b)
        self._r = dims[0] - 3

    def load_affine_field(self, mlp):
        dims = mlp["dims"]
        W = np.concatenate([w.reshape(-1) for w in mlp["W_bits"]])
        b = np.concatenate(mlp["b"])
        nsf_mpm_load_affine_field(self.h, dims[0], dims[1], len(dims) - 2, dims[-1], W, b)

    def infer_state(self, z_prev=None):
        """x = g(X, z_n), v = (x - g(X, z_prev)) / dt, C = l(X, z_n) for every point."""
        nsf_mpm_infer_state(self.h, z_prev)

    def build_integration_set(self, X_all, sample_idx, z_prev=None):
        """Replace the points by S then N \\ S per scene (header); returns |N_s|."""
        counts = nsf_mpm_build_integration_set(self.h, X_all, sample_idx, z_prev, self.cfg.n_scenes)
        self.n = int(counts.sum())
        return counts

    def rom_step(self, X_all, sample_idx, gn_iters=3, z_prev=None):
        """One latent-space step: returns z_{n+1}, |N_s|."""
        z, counts = nsf_mpm_rom_step(self.h, X_all, sample_idx, gn_iters, self.cfg.n_scenes, self._r, z_prev)
        self.n = int(counts.sum())
        return z, counts

    def invert_latents(self, n_sample, n_iters=3):
        """Network inversion; returns z_hat (n_scenes x r)."""
        out = np.empty((self.cfg.n_scenes, self._r), dtype=np.float32)
        nsf_mpm_invert_latents(self.h, n_sample, n_iters, out)
        return out

    def sync(self):
        nsf_mpm_sync(self.h)

    def inverted_count(self) -> int:
        """Particle updates that produced det F_E <= 0 since the load (#21)."""
        return nsf_mpm_inverted_count(self.h)

    def read(self, mask=NSF_FIELD_X | NSF_FIELD_V | NSF_FIELD_C | NSF_FIELD_F | NSF_FIELD_TAU, device=None):
        outs = nsf_mpm_read_state(self.h, mask, self.n, device)
        names = [nm for bit, nm in ((1, "x"), (2, "v"), (4, "C"), (8, "F"), (16, "tau"), (32, "tau_Y")) if mask & bit]
        return dict(zip(names, outs))

    def close(self):
        if self.h:
            nsf_mpm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
