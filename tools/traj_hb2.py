import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2310_17790_b200 as nsf
from oracle import mpm
from tests.parity_util import gpu_state, rel_err
from tests.test_gpu_parity import small_scenes
sc = small_scenes()["HB"]
P = mpm.params_from_config(sc.cfg)
sim = nsf.Simulator(sc.cfg); sim.load_scene(sc)
g0 = gpu_state(sim)
# one step: per-particle tau difference stats
sim.substep(1); sim.sync(); g1 = gpu_state(sim)
ref1 = mpm.substep({k: g0[k] for k in ("x", "v", "C", "F", "tau")}, P, 0)
dt_ = np.linalg.norm((g1["tau"] - ref1["tau"]).reshape(sc.n, -1), axis=1)
nt = np.linalg.norm(ref1["tau"].reshape(sc.n, -1), axis=1)
print("step1 tau abs err: mean", dt_.mean(), "max", dt_.max(), "| tau mean", nt.mean())
# signed mean of the difference (bias) of the pressure and of dev norms
pg = np.trace(g1["tau"], axis1=1, axis2=2) / 3; pr = np.trace(ref1["tau"], axis1=1, axis2=2) / 3
print("pressure diff mean", (pg - pr).mean(), "std", (pg - pr).std(), "pressure mean", pr.mean())
dg = np.linalg.det(g1["F"]); dr = np.linalg.det(ref1["F"])
print("detF diff mean", (dg - dr).mean(), "std", (dg - dr).std())
Ftr = None
