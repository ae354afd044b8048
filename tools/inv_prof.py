import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np
import scenes
import paper_2310_17790_b200 as nsf
from inv_probe import deformation_net
sc = scenes.c5()
sim = nsf.Simulator(sc.cfg)
sim.load_scene(sc)
sim.load_deformation_field(deformation_net(77))
sim.substep(2)
sim.invert_latents(64, 2)
sim.sync()
sim.close()
print("ok")
