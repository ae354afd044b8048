"""Substep time of a config with the body translated by whole cells (probe of
how segment alignment to the 4x4x4-cell block lattice affects the fused kernel).

    python tools/align_probe.py --config C3 --shifts 0,0,0 1,1,1 [--steps 100]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--shifts", nargs="+", default=["0,0,0", "1,1,1"])
    ap.add_argument("--steps", type=int, default=100)
    a = ap.parse_args()
    import torch
    import scenes
    import paper_2310_17790_b200 as nsf
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for sh in a.shifts:
        d = [int(t) for t in sh.split(",")]
        sc = {"C1": scenes.c1, "C2": scenes.c2, "C3": scenes.c3, "C4": scenes.c4, "C5": scenes.c5}[a.config]()
        for ax in range(3):
            if d[ax]:
                sc.x[:, ax] += d[ax] * sc.cfg.dx
        stream = torch.cuda.Stream()
        sim = nsf.Simulator(sc.cfg, stream=stream.cuda_stream)
        sim.load_scene(sc)
        sim.substep(5)
        sim.sync()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
        for e0, e1 in ev:
            with torch.cuda.stream(stream):
                flush.fill_(1.0)
            e0.record(stream)
            sim.substep(1)
            e1.record(stream)
        ev[-1][1].synchronize()
        us = sum(e0.elapsed_time(e1) for e0, e1 in ev) * 1e3 / a.steps
        sim.sync()
        sim.close()
        print(f"{a.config} shift {d}: {us:.1f} us/substep", flush=True)


if __name__ == "__main__":
    main()
