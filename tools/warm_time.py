"""Back-to-back regime: microseconds per substep of nsf_mpm_substep(K) calls (no L2 flush between
substeps, one call), after a pre-roll.  NSF_MPM_LIB picks the library.
    python tools/warm_time.py C3 [preroll] [K] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2310_17790_b200 as nsf  # noqa: E402
import scenes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
pre = int(sys.argv[2]) if len(sys.argv) > 2 else 250
K = int(sys.argv[3]) if len(sys.argv) > 3 else 64
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
sc = scenes.by_name(name)
stream = torch.cuda.Stream()
sim = nsf.Simulator(sc.cfg, stream=stream.cuda_stream)
sim.load_scene(sc)
sim.substep(pre)
sim.sync()
out = []
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    sim.substep(K)
    b.record(stream)
    b.synchronize()
    out.append(a.elapsed_time(b) * 1e3 / K)
sim.close()
print(name, os.path.basename(os.environ.get("NSF_MPM_LIB", "default")), "us/substep back-to-back:",
      " ".join(f"{t:.2f}" for t in out))
