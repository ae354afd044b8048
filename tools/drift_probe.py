import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
import torch, scenes, paper_2310_17790_b200 as nsf
for name in ("C3", "C2"):
    sc = getattr(scenes, name.lower())()
    N = sc.cfg.grid_res; dx = 1.0 / N
    sim = nsf.Simulator(sc.cfg); sim.load_scene(sc)
    def keys():
        x = sim.read(nsf.NSF_FIELD_X)["x"].astype(np.float32)
        b = np.clip(np.floor(x * np.float32(N) - np.float32(0.5)).astype(int), 0, N - 3)
        return (b // 4), b
    k0, c0 = keys()
    out = []
    for s in range(1, 65):
        sim.substep(1)
        if s in (1, 4, 8, 16, 32, 64):
            k, c = keys()
            out.append((s, float(np.mean(np.any(k != k0, 1))), float(np.mean(np.any(c != c0, 1)))))
    print(name, " ".join(f"s{s}: block {a*100:.2f}% cell {b*100:.2f}%" for s, a, b in out))
    sim.close()
