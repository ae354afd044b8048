"""Attribute an ncu SASS page (per-instruction executions and stall samples) to
source lines and enclosing functions, using the cubin's line table.

    ncu -i rep.ncu-rep --page source --csv -k regex:NAME --print-source sass > sass.csv   (on the GPU box)
    python tools/sass_lines.py sass.csv paper_2310_17790_b200/_build/kernels_tiled.cu.o MANGLED_SUBSTRING [top]

The source page of this ncu build does not carry CUDA-line metrics, so the SASS
rows are joined (by offset within the function) with `nvdisasm -g` of the same
cubin: the innermost inlined file:line of each instruction.
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile


def line_table(obj, fn_sub):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
    out, cur, inside = {}, None, False
    for line in dis.splitlines():
        if line.startswith("//-----") and ".text." in line:
            inside = fn_sub in line
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", line)
        if m:
            out[int(m.group(1), 16)] = cur
    return out


def functions_of(path):
    """(start line, name) of every function definition in a source file."""
    starts = []
    for i, l in enumerate(open(path), 1):
        m = re.match(r"\s*(?:template <[^>]*>\s*)?(?:static\s+)?(?:__device__|__global__|__host__)[^(]*?(\w+)\s*\(", l)
        if m and not l.rstrip().endswith(";"):
            starts.append((i, m.group(1)))
    return starts


def main(csv_path, obj, fn_sub, top=40):
    lt = line_table(obj, fn_sub)
    rows = list(csv.reader(open(csv_path)))
    hdr = rows[1]
    ia, ii, iss = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    base = None
    by_line = collections.Counter()
    smp_line = collections.Counter()
    for r in rows[2:]:
        try:
            addr = int(r[ia], 16)
            n, smp = int(r[ii]), int(r[iss])
        except (ValueError, IndexError):
            continue
        base = addr if base is None else base
        key = lt.get(addr - base, ("?", 0))
        by_line[key] += n
        smp_line[key] += smp
    src_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2310_17790_b200", "csrc")
    funcs = {}
    for f in os.listdir(src_dir):
        if f.endswith((".cu", ".cuh")):
            funcs[f] = functions_of(os.path.join(src_dir, f))

    def fn(key):
        f, ln = key
        best = "?"
        for s, name in funcs.get(f, []):
            if s <= ln:
                best = name
        return f"{f}:{best}"
    tot, tots = sum(by_line.values()) or 1, sum(smp_line.values()) or 1
    by_fn, smp_fn = collections.Counter(), collections.Counter()
    for k, v in by_line.items():
        by_fn[fn(k)] += v
        smp_fn[fn(k)] += smp_line[k]
    print(f"warp instructions {tot}, stall samples {tots}")
    print("-- by function (inst %, stall %)")
    for k, v in by_fn.most_common(25):
        print(f"{100 * v / tot:6.1f}% {100 * smp_fn[k] / tots:6.1f}%  {k}")
    print("-- by line (inst %, stall %)")
    for k, v in by_line.most_common(top):
        print(f"{100 * v / tot:6.1f}% {100 * smp_line[k] / tots:6.1f}%  {k[0]}:{k[1]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 40)
