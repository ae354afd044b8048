import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from tests.test_gpu_far import bullet_scene
from tests.parity_util import gpu_state
import paper_2310_17790_b200 as nsf

def traj(gu, steps=40):
    os.environ["NSF_FUSED_GU"] = gu
    sc, b = bullet_scene()
    sim = nsf.Simulator(sc.cfg)
    sim.load_scene(sc)
    out = []
    for k in range(steps):
        sim.substep(1)
        out.append(gpu_state(sim)["v"])
    sim.close()
    return np.array(out), b

ref, bullets = traj("kernel")
nbad = 0
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    t, _ = traj("kernel")
    d = np.abs(t - ref).max(axis=2)   # [steps, n]
    worst = d.max()
    if worst > 1e-3:
        nbad += 1
        k0 = int(np.argmax(d.max(axis=1) > 1e-3))
        idx = np.where(d[k0] > 1e-3)[0]
        print(f"run {it}: diverges at substep {k0 + 1}, {len(idx)} particles, bullets among them: "
              f"{np.isin(idx, bullets).sum()}, first idx {idx[:8]}", flush=True)
    else:
        print(f"run {it}: ok ({worst:.2e})", flush=True)
print("bad runs", nbad)
