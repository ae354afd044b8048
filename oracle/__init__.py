"""fp64 CPU oracle for the MLS-MPM (APIC) substep of arXiv 2310.17790.

TEST INFRASTRUCTURE ONLY.  Nothing in the product path
(`paper_2310_17790_b200/`, `include/`) imports, links or executes this
package; only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may use it.

It is a plain, slow, obviously-correct transcription of the paper's algorithm
(§3.3 "MPM algorithm", lines 173-180; appendix) in
float64 numpy, particles in index order, with every reading of a silent or
garbled passage taken from SURVEY.md §8(c) and listed in DESIGN.md.

It shares no code with the CUDA path.  Its only common input is the seeded
generator module `scenes/`, which holds none of the method's arithmetic.

Pinned by tests/test_oracle_*.py against closed forms, invariants, worked
examples, independent library routines and energy finite differences.
Functions that have no such pin say "parity unpinned" in their docstring.
"""
from .constitutive import (lame, svd_rotation_safe, tau_fixed_corotated, tau_hencky,
                           return_map_drucker_prager, return_map_von_mises,
                           dp_alpha, elastoplastic_update)
from .mpm import (Params, params_from_config, bspline_quadratic, p2g, grid_update,
                  g2p, substep, run, initial_tau, block_keys, OutOfDomain)
from .mlp import elu, round_bf16, mlp_forward, nsf_stress, voigt_to_matrix
from .reduced import reduced_substep, reduced_run

__all__ = [n for n in dir() if not n.startswith("_")]
