"""Summarise `ncu --page source --csv --print-source cuda,sass` output per CUDA
source line: warp-stall samples and warp instructions executed.

    ncu -i rep.ncu-rep --page source --csv -k regex:NAME --print-source cuda,sass > src.csv
    python tools/ncu_source_summary.py src.csv [top]
"""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    out = []
    fname = None
    hdr = None
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r or not r[0]:
            continue
        try:
            samples = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            inst = int(r[hdr.index("Instructions Executed")])
        except (ValueError, IndexError):
            continue
        out.append((samples, inst, fname, r[0], r[1][:90]))
    tot_s = sum(o[0] for o in out) or 1
    tot_i = sum(o[1] for o in out) or 1
    print(f"total samples {tot_s}, warp instructions {tot_i}")
    for s, i, f, ln, src in sorted(out, reverse=True)[:top]:
        print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% inst  {f}:{ln:>4}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
