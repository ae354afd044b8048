"""Copy one round's GPU evidence from gpurun_out/ into profiles/r1/ (bench lines,
ncu launch lists + summary, ncu full-capture summaries) and refresh
profiles/ncu_traffic.json (DRAM bytes per launch of the roofline kernels).

    python tools/update_profiles.py r1j
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "r1")
GO = os.path.join(ROOT, "gpurun_out")
KERNEL_KEYS = {"k_g2p2g": "g2p2g", "k_nsf_mlp_tc": "nsf_mlp", "k_g2p_nsf": "g2p_nsf"}


def main(tag):
    os.makedirs(OUT, exist_ok=True)
    for c in ("C1", "C2", "C3", "C4", "C5"):
        src = os.path.join(GO, f"bench_{tag}_{c}.json")
        if os.path.exists(src):
            shutil.copy(src, os.path.join(OUT, f"bench_{c}.json"))
    lines = ["ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised; compare shares, "
             "not absolutes)"]
    for c in ("C3", "C5"):
        src = os.path.join(GO, f"launches_{tag}_{c}.csv")
        if not os.path.exists(src):
            continue
        shutil.copy(src, os.path.join(OUT, f"launches_{c}.csv"))
        lines.append(f"command: python bench.py --config {c} --steps 20 --warmup 3 --no-cpu-baseline --e2e-iters 1")
        lines.append(subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_summary.py"), src],
                                    capture_output=True, text=True).stdout)
    open(os.path.join(OUT, "launches_summary.txt"), "w").write("\n".join(lines))
    traffic = {"_comment": "dram__bytes_read.sum + dram__bytes_write.sum per launch (bytes), one ncu --set full "
                           f"capture per kernel (profiles/r1/ncu_*.txt, tag {tag}), cold cache"}
    for c, name in (("C3", "ncu_C3_g2p2g.txt"), ("C5", "ncu_C5_mlp_g2p.txt")):
        rep = os.path.join(GO, f"prof_{tag}_{c}.ncu-rep")
        if not os.path.exists(rep):
            continue
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "summarize_ncu.py"), rep,
                        os.path.join(OUT, name)], check=True)
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            kname = r[hdr.index("Kernel Name")].split("(")[0].split("<")[0].replace("void ", "").strip()
            key = KERNEL_KEYS.get(kname)
            if not key:
                continue
            tot = 0.0
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                i = hdr.index(m)
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[i]]
                tot += float(r[i].replace(",", "")) * scale
            traffic.setdefault(c, {})[key] = int(tot)   # first captured launch of each kernel
    json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
    print(json.dumps(traffic))


if __name__ == "__main__":
    main(sys.argv[1])
