"""Memory-safety runs with the bounds-checked library (libnsf_mpm_checked.so,
-DNSF_CHECKED=1): every shared-memory slot, velocity-tile read, grid node, block
id, list entry and reorder destination the kernels write is asserted in range
(NSF_CHECK, csrc/params.cuh) and a violation traps.  This stands in for
compute-sanitizer memcheck, which the GPU pool does not allow.  Each scene runs
in its own process (tools/checked_run.py) so a trap cannot poison the others."""
import ctypes
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2310_17790_b200", "libnsf_mpm_checked.so")


@pytest.fixture(scope="module")
def lib_checked():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2310_17790_b200 import build
    build.build(checked=True)   # incremental: rebuilds only what changed since the last build
    return CHECKED


def _run(args, env_extra):
    env = dict(os.environ, NSF_MPM_LIB=CHECKED, **env_extra)
    return subprocess.run([sys.executable, *args], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)


def test_checks_trap(lib_checked):
    """Positive control: a failing NSF_CHECK traps (the kernel reports an error)."""
    code = ("import ctypes, sys; L = ctypes.CDLL(sys.argv[1]); "
            "assert L.nsf_mpm_checked_selftest(0) == 0; sys.exit(10 + L.nsf_mpm_checked_selftest(1))")
    r = _run(["-c", code, lib_checked], {})
    assert r.returncode == 11, r.stdout + r.stderr
    assert "NSF_CHECK failed" in r.stdout + r.stderr


@pytest.mark.parametrize("gu", ["rot", "kernel", "barrier"])
@pytest.mark.parametrize("scene", ["c1_spin", "dense_cluster", "sparse"])
def test_full_order_checked(lib_checked, scene, gu):
    r = _run([os.path.join("tools", "checked_run.py"), scene], {"NSF_FUSED_GU": gu})
    assert r.returncode == 0 and "NSF_CHECK failed" not in r.stdout + r.stderr, r.stdout + r.stderr


@pytest.mark.parametrize("scene", ["c5_small", "det", "gradw"])
def test_other_paths_checked(lib_checked, scene):
    r = _run([os.path.join("tools", "checked_run.py"), scene], {})
    assert r.returncode == 0 and "NSF_CHECK failed" not in r.stdout + r.stderr, r.stdout + r.stderr
