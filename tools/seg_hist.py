"""Distribution of particles per non-empty 4^3-cell block (= fused-kernel segment)
of a config after a pre-roll: how many phase-1 passes of 256 threads each needs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2310_17790_b200 as nsf  # noqa: E402
import scenes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
sc = scenes.by_name(name)
sim = nsf.Simulator(sc.cfg)
sim.load_scene(sc)
for pre in (0, 64, 250, 499):
    sim.substep(pre - nsf.nsf_mpm_step_count(sim.h))
    nb = (sc.cfg.grid_res // 4) ** 3 * (sc.cfg.n_scenes or 1)
    counts, _ = nsf.nsf_mpm_debug_bins(sim.h, nb, sim.n)
    c = counts[counts > 0]
    passes = np.ceil(c / 256).astype(int)
    print(f"{name} substep {pre}: {len(c)} segments, particles min {c.min()} median {np.median(c):.0f} max {c.max()}; "
          f">512: {np.sum(c > 512)}; passes hist {np.bincount(passes)[1:].tolist()}; "
          f"ideal passes {c.sum() / 256:.0f} vs {passes.sum()}")
sim.close()
