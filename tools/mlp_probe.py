"""Time the NSF MLP alone (eval_stress_field on C5's 524,288 points, device
buffers) against the reduced substep (MLP + P2G epilogue, G2P).

    python tools/mlp_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def main():
    import torch
    import scenes
    import paper_2310_17790_b200 as nsf
    sc = scenes.c5()
    sim = nsf.Simulator(sc.cfg)
    sim.load_scene(sc)
    pts = torch.tensor(sc.x, device="cuda", dtype=torch.float32).contiguous()
    z = torch.tensor(sc.z0[0], device="cuda", dtype=torch.float32).contiguous()
    out = torch.empty(pts.shape[0], 6, device="cuda", dtype=torch.float32)
    for _ in range(3):
        nsf.nsf_mpm_eval_stress_field(sim.h, z, pts, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        nsf.nsf_mpm_eval_stress_field(sim.h, z, pts, out)
    e1.record()
    torch.cuda.synchronize()
    print(f"eval_stress_field {pts.shape[0]} points: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us/call")
    sim.substep(5)
    sim.sync()
    e0.record()
    sim.substep(50)
    e1.record()
    torch.cuda.synchronize()
    print(f"reduced substep: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us")
    sim.close()


if __name__ == "__main__":
    main()
