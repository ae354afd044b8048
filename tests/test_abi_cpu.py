"""CPU-side checks of the boundary: the C-ABI library builds for sm_100a, loads,
and exports every symbol include/nsf_mpm.h declares; the binding's struct
layout matches the header.  No compute calls (there is no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nsf_mpm.h")


@pytest.fixture(scope="module")
def built_lib():
    from paper_2310_17790_b200 import build
    return build.build()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nsf_mpm_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for must in ("nsf_mpm_create", "nsf_mpm_load_particles", "nsf_mpm_substep",
                 "nsf_mpm_eval_stress_field", "nsf_mpm_read_state"):
        assert must in names


def test_library_exports_every_declared_symbol(built_lib):
    out = subprocess.run(["nm", "-D", "--defined-only", built_lib], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (nsf_mpm_\w+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(built_lib)
    for n in declared_functions():
        getattr(lib, n)


def test_binding_covers_header(built_lib):
    import paper_2310_17790_b200 as nsf
    assert sorted(nsf.EXPORTS) == declared_functions()
    for n in declared_functions():
        assert callable(getattr(nsf, n))


def test_abi_version(built_lib):
    import paper_2310_17790_b200 as nsf
    hdr = open(os.path.join(ROOT, "include", "nsf_mpm.h")).read()
    ver = int(hdr.split("#define NSF_MPM_ABI_VERSION")[1].split()[0])
    assert nsf.nsf_mpm_abi_version() == ver == 5


def test_material_struct_layout_matches_header(built_lib, tmp_path):
    """Compile a tiny C program against the header and compare offsetof/sizeof with
    the ctypes structure of the binding."""
    import paper_2310_17790_b200 as nsf
    fields = [f[0] for f in nsf.nsf_material._fields_]
    prog = ["#include <stdio.h>", "#include <stddef.h>", '#include "nsf_mpm.h"', "int main(void){",
            'printf("%zu\\n", sizeof(nsf_material));']
    prog += [f'printf("%zu\\n", offsetof(nsf_material, {f}));' for f in fields]
    prog += ["return 0;}"]
    c = tmp_path / "layout.c"
    c.write_text("\n".join(prog))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)], check=True)
    vals = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert vals[0] == ctypes.sizeof(nsf.nsf_material)
    for f, off in zip(fields, vals[1:]):
        assert getattr(nsf.nsf_material, f).offset == off, f


def test_sass_is_sm100a(built_lib):
    out = subprocess.run(["cuobjdump", "--list-elf", built_lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_in_product_path():
    """The product package never imports, links or executes oracle/."""
    pkg = os.path.join(ROOT, "paper_2310_17790_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"\b(import|from)\s+oracle\b", txt), f
                assert "oracle/" not in txt.replace("fp64 oracle", ""), f
