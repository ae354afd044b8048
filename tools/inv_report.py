"""Print the inversion parity numbers quoted in DESIGN.md (reading #37): per sample
size and GPU pass, the step deviation from the emulating oracle, the fp32-order
spread, the emulate-vs-exact gap and the objective-reduction mismatch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2310_17790_b200 as nsf  # noqa: E402
from oracle.inversion import invert_scenes  # noqa: E402
from tests.inv_util import fp32_spread  # noqa: E402
from tests.test_gpu_inversion import _invert, _objective, _scene  # noqa: E402

for simt in ("0", "1"):
    os.environ["NSF_GN_SIMT"] = simt
    for ns in (64, 50, 256):
        sc, gnet, _ = _scene()
        zg, x = _invert(nsf, sc, gnet, ns, 1)
        z0 = sc.z0.astype(np.float64)
        zo = invert_scenes(sc.X_ref, x, sc.scene_offsets, ns, z0, gnet, 1, "emulate")
        spread, gap = fp32_spread(sc, gnet, x, z0, ns, orders=8)
        dev = np.linalg.norm(zg - zo) / np.linalg.norm(zo - z0)
        f0, fo, fg = (_objective(sc, gnet, x, z, ns) for z in (z0, zo, zg))
        print(f"{'simt' if simt == '1' else 'tc  '} n_sample {ns:3d}: step dev {dev:.4f}  fp32 spread {spread:.4f}  "
              f"gap {gap:.3f}  objective mismatch {(fg - fo) / (f0 - fo):+.2e}")
