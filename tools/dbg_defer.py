import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from tests.test_gpu_far import bullet_scene
from tests.parity_util import gpu_state
import paper_2310_17790_b200 as nsf

def run(gu, steps=40):
    os.environ["NSF_FUSED_GU"] = gu
    sc, b = bullet_scene()
    sim = nsf.Simulator(sc.cfg)
    sim.load_scene(sc)
    sim.substep(steps)
    sim.sync()
    s = gpu_state(sim)
    sim.close()
    return s

order = sys.argv[1].split(",")
prev = None
ref = None
for gu in order:
    s = run(gu)
    if gu == "kernel" and ref is None: ref = s
    print(gu, "max |dv| vs first kernel", float(np.max(np.abs(s["v"] - ref["v"]))) if ref is not None else "-", flush=True)
