"""Per-substep device time of C3 back-to-back vs. with idle gaps between substeps
(diagnoses clock/power effects), plus an NVML clock readout.

    python tools/gap_test.py [--config C3] [--n 200]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--n", type=int, default=200)
    a = ap.parse_args()
    import torch
    import scenes
    import paper_2310_17790_b200 as nsf
    import pynvml
    pynvml.nvmlInit()
    hd = pynvml.nvmlDeviceGetHandleByIndex(0)
    sc = {"C1": scenes.c1, "C2": scenes.c2, "C3": scenes.c3, "C4": scenes.c4, "C5": scenes.c5}[a.config]()
    st = torch.cuda.Stream()
    sim = nsf.Simulator(sc.cfg, stream=st.cuda_stream)
    sim.load_scene(sc)
    sim.substep(10)
    sim.sync()

    def run(gap_s):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.n)]
        clk = []
        for e0, e1 in ev:
            e0.record(st)
            sim.substep(1)
            e1.record(st)
            if gap_s:
                e1.synchronize()
                time.sleep(gap_s)
            clk.append(pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM))
        ev[-1][1].synchronize()
        t = sorted(x.elapsed_time(y) * 1e3 for x, y in ev)
        return t[len(t) // 2], t[0], t[-1], sorted(clk)[len(clk) // 2], pynvml.nvmlDeviceGetPowerUsage(hd) / 1e3

    for gap in (0.0, 0.002, 0.0, 0.02):
        med, lo, hi, c, pw = run(gap)
        print(f"gap {gap*1e3:5.1f} ms: substep median {med:7.1f} us  min {lo:7.1f}  max {hi:7.1f}  sm_clk {c} MHz  power {pw:.0f} W")
    sim.close()


if __name__ == "__main__":
    main()
