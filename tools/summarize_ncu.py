"""Write a text summary of an ncu --set full report: per kernel the key counters
(time, DRAM bytes, issue, occupancy, pipes, stall reasons) and the top source
lines by stall samples.

    python tools/summarize_ncu.py gpurun_out/prof.ncu-rep out.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads per instruction"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.per_cycle_active", "warps active per SM"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("lts__t_sectors_op_red.sum", "L2 red sectors"),
]


def ncu(args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def main(rep, out):
    raw = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"]))))
    hdr, units = raw[0], raw[1]
    lines = [f"# ncu --set full summary of {rep.split('/')[-1]}", ""]
    for r in raw[2:]:
        lines.append(f"## {r[hdr.index('Kernel Name')][:100]}")
        for k, label in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"  {label:32s} {r[i]} {units[i]}")
        stalls = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), r[i]) for i, h in enumerate(hdr)
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
        stalls = sorted(((n, float(v.replace(",", "") or 0)) for n, v in stalls), key=lambda t: -t[1])[:8]
        tot = sum(v for _, v in stalls) or 1.0
        lines.append("  top stall reasons (pc samples): " +
                     ", ".join(f"{n} {100 * v / tot:.0f}%" for n, v in stalls))
        lines.append("")
    src = ncu(["-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"])
    rows = list(csv.reader(io.StringIO(src)))
    agg = {}
    fname = None
    shdr = None
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            shdr = r
            continue
        if shdr is None or not r or not r[0].isdigit():
            continue
        try:
            s = int(r[shdr.index("Warp Stall Sampling (All Samples)")])
            n = int(r[shdr.index("Instructions Executed")])
        except (ValueError, IndexError):
            continue
        key = (fname, int(r[0]), r[1].strip()[:90])
        a = agg.setdefault(key, [0, 0])
        a[0] += s
        a[1] += n
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    lines.append("## top source lines (all captured kernels): stall samples %, instructions %")
    for (f, ln, txt), (s, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:30]:
        lines.append(f"  {100 * s / ts:5.1f}% {100 * n / ti:5.1f}%  {f}:{ln}  {txt}")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
