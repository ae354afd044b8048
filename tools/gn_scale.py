import os, sys, time, faulthandler
faulthandler.dump_traceback_later(60, exit=True)
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np
import scenes
import paper_2310_17790_b200 as nsf
from inv_probe import deformation_net
ns = int(sys.argv[1]); nsamp = int(sys.argv[2]); per = int(sys.argv[3]) if len(sys.argv) > 3 else 256
sc = scenes.c5_small(n_scenes=ns, per_scene=per)
sim = nsf.Simulator(sc.cfg)
sim.load_scene(sc)
sim.load_deformation_field(deformation_net(77))
if os.environ.get("READ_FIRST"):
    sim.read(nsf.NSF_FIELD_X)
t0 = time.time()
z = sim.invert_latents(nsamp, 1)
print("ok", ns, nsamp, per, round(time.time() - t0, 3), float(np.abs(z).sum()), flush=True)
sim.close()
