"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel launches, mean duration and share of the summed device time.

    python tools/launch_summary.py gpurun_out/launches.csv [--substeps K]
"""
import csv
import sys
from collections import OrderedDict


def main(path, substeps=None):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = OrderedDict()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        ns = float(r[vi].replace(",", ""))
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ns
    tot = sum(v[1] for v in agg.values()) or 1.0
    print(f"{'kernel':40s} {'launches':>8s} {'mean_us':>9s} {'share':>7s}")
    for k, (c, ns) in agg.items():
        print(f"{k:40s} {c:8d} {ns / c / 1e3:9.2f} {ns / tot:7.3f}")
    if substeps:
        print(f"summed device time per substep: {tot / 1e3 / substeps:.2f} us (cold-cache, serialised)")


if __name__ == "__main__":
    k = None
    if "--substeps" in sys.argv:
        k = int(sys.argv[sys.argv.index("--substeps") + 1])
    main(sys.argv[1], k)
