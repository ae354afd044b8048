"""Per-substep device time over a long run: mean per 32-substep window and
mean by phase since the last re-binning (diagnoses drift/ordering effects).

    python tools/trace_steps.py [--config C3] [--n 1024]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--n", type=int, default=1024)
    a = ap.parse_args()
    import numpy as np
    import torch
    import scenes
    import paper_2310_17790_b200 as nsf
    sc = {"C1": scenes.c1, "C2": scenes.c2, "C3": scenes.c3, "C4": scenes.c4, "C5": scenes.c5}[a.config]()
    st = torch.cuda.Stream()
    sim = nsf.Simulator(sc.cfg, stream=st.cuda_stream)
    sim.load_scene(sc)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.n)]
    for e0, e1 in ev:
        e0.record(st)
        sim.substep(1)
        e1.record(st)
    ev[-1][1].synchronize()
    t = np.array([x.elapsed_time(y) * 1e3 for x, y in ev])
    per = int(os.environ.get("NSF_REBIN_EVERY", "32"))
    w = t[: a.n // per * per].reshape(-1, per)
    print("window means (us):", " ".join(f"{v:.0f}" for v in w.mean(1)))
    print("by phase (us):     ", " ".join(f"{v:.0f}" for v in np.median(w, 0)))
    x = sim.read(nsf.NSF_FIELD_X)["x"]
    print("extent", x.min(0), x.max(0))
    sim.close()


if __name__ == "__main__":
    main()
