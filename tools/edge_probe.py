import sys, os; sys.path.insert(0, os.getcwd())
import numpy as np, scenes
import paper_2310_17790_b200 as nsf
from tests.test_gpu_edge_cases import edge_scene, MODELS
from tests.parity_util import single_step_parity, voigt_to_mat
for model in ("DP", "VM"):
    sc, inv = edge_scene(MODELS[model], 31 + list(MODELS).index(model))
    os.environ["NSF_FUSED_GU"] = "rot"
    sim = nsf.Simulator(sc.cfg); sim.load_scene(sc)
    errs, s1, ref = single_step_parity(sim, sc.cfg, 0)
    sim.close()
    print(model, errs)
    for f in ("F", "tau"):
        d = np.linalg.norm((s1[f] - ref[f]).reshape(sc.n, -1), axis=1)
        r = np.linalg.norm(ref[f].reshape(sc.n, -1), axis=1)
        o = np.argsort(-d)[:8]
        cls = np.array(["normal"] * sc.n, dtype=object); cls[inv] = "inv"
        F0 = sc.F.astype(np.float64)
        sv = np.linalg.svd(F0, compute_uv=False)
        print(f, [(int(i), cls[i], float(d[i]), float(r[i]), np.round(sv[i], 5).tolist(), float(np.linalg.det(F0[i]))) for i in o])
