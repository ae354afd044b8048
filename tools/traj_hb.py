import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2310_17790_b200 as nsf
from oracle import mpm
from tests.parity_util import gpu_state, rel_err, single_step_parity
from tests.test_gpu_parity import small_scenes
name = sys.argv[1] if len(sys.argv) > 1 else "HB"
sc = small_scenes()[name]
P = mpm.params_from_config(sc.cfg)
ref = {"x": sc.x, "v": sc.v, "C": sc.C, "F": sc.F, "tau": mpm.initial_tau(sc.F, P)}
sim = nsf.Simulator(sc.cfg); sim.load_scene(sc)
done = 0
for K in (1, 5, 10, 20, 40, 70, 100):
    sim.substep(K - done); sim.sync()
    ref = mpm.run(ref, P, K - done, step0=done); done = K
    g = gpu_state(sim)
    print(name, K, "x", rel_err(g["x"], ref["x"]), "v", rel_err(g["v"], ref["v"]), "F", rel_err(g["F"], ref["F"]),
          "detF gpu/ref", float(np.mean(np.linalg.det(g["F"]))), float(np.mean(np.linalg.det(ref["F"]))))
errs, _, _ = single_step_parity(sim, sc.cfg, done)
print("one step from the GPU state at", done, errs)
sim.close()
