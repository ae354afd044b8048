"""Network inversion GPU vs oracle (diagnostic)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402


def deformation_net(seed):
    import scenes
    return scenes.deformation_field(seed)


def main():
    import scenes
    import paper_2310_17790_b200 as nsf
    from oracle.inversion import invert_scenes, g_with_tangents
    gnet = deformation_net(77)
    sc = scenes.c5_small(n_scenes=3, per_scene=256)
    rng = np.random.default_rng(3)
    z_star = rng.normal(size=(3, 6)).astype(np.float32)
    x = sc.x.copy()
    for s, (a, b) in enumerate(zip(sc.scene_offsets[:-1], sc.scene_offsets[1:])):
        g, _ = g_with_tangents(sc.X_ref[a:b], z_star[s], gnet, "emulate")
        x[a:b] = g
    sc.x = x.astype(np.float32)
    sc.z0 = (z_star + 0.1 * rng.normal(size=z_star.shape)).astype(np.float32)
    sc.dz = np.zeros_like(sc.z0)
    for iters in (1, 2, 4):
        sim = nsf.Simulator(sc.cfg)
        sim.load_scene(sc)
        sim.load_deformation_field(gnet)
        st = sim.read(nsf.NSF_FIELD_X)
        zg = sim.invert_latents(64, iters)
        sim.close()
        zo = invert_scenes(sc.X_ref, st["x"], sc.scene_offsets, 64, sc.z0.astype(np.float64), gnet, iters, "emulate")
        print(f"iters {iters}: |gpu-oracle|/|oracle-start| {np.linalg.norm(zg - zo) / np.linalg.norm(zo - sc.z0):.2e}"
              f"  |gpu-z*|/|z*| {np.linalg.norm(zg - z_star) / np.linalg.norm(z_star):.2e}"
              f"  |oracle-z*|/|z*| {np.linalg.norm(zo - z_star) / np.linalg.norm(z_star):.2e}"
              f"  start {np.linalg.norm(sc.z0 - z_star) / np.linalg.norm(z_star):.2e}")


if __name__ == "__main__":
    main()


def after_substeps():
    import paper_2310_17790_b200 as nsf
    from oracle.inversion import invert_scenes
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
    from tests.test_gpu_inversion import _scene, _invert
    for k in (1, 3, 10, 40):
        sc, gnet, _ = _scene()
        sc.dz = (1e-4 * np.random.default_rng(9).normal(size=sc.z0.shape)).astype(np.float32)
        zg, x = _invert(nsf, sc, gnet, 64, 1, substeps=k)
        z_start = sc.z0.astype(np.float64) + k * sc.dz.astype(np.float64)
        zo = invert_scenes(sc.X_ref, x, sc.scene_offsets, 64, z_start, gnet, 1, "emulate")
        print(k, np.linalg.norm(zg - zo) / np.linalg.norm(zo - z_start), np.linalg.norm(zo - z_start))


def timing():
    import torch
    import paper_2310_17790_b200 as nsf
    sc = __import__("scenes").c5()
    gnet = deformation_net(77)
    sim = nsf.Simulator(sc.cfg)
    sim.load_scene(sc)
    sim.load_deformation_field(gnet)
    sim.substep(3)
    sim.sync()
    for iters in (1, 3):
        sim.invert_latents(64, iters)
        torch.cuda.synchronize()
        import time
        t0 = time.perf_counter()
        for _ in range(10):
            sim.invert_latents(64, iters)
        torch.cuda.synchronize()
        print(f"C5 inversion 256 scenes x 64 samples, {iters} GN iters: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms (host-timed, incl. sync)")
    sim.close()


def conditioning(n_sample=256):
    import paper_2310_17790_b200 as nsf
    from oracle.inversion import invert_scenes
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
    from tests.test_gpu_inversion import _scene, _invert
    sc, gnet, _ = _scene()
    zg, x = _invert(nsf, sc, gnet, n_sample, 1)
    zo = invert_scenes(sc.X_ref, x, sc.scene_offsets, n_sample, sc.z0.astype(np.float64), gnet, 1, "emulate")
    ze = invert_scenes(sc.X_ref, x, sc.scene_offsets, n_sample, sc.z0.astype(np.float64), gnet, 1, "exact")
    print(n_sample, "gpu-oracle", np.linalg.norm(zg - zo) / np.linalg.norm(zo - sc.z0),
          "emulate-exact", np.linalg.norm(ze - zo) / np.linalg.norm(zo - sc.z0))
