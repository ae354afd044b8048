"""Work counters of the fused kernel per substep window (statistics build):
    NSF_MPM_LIB=paper_2310_17790_b200/_ab/stats.so python tools/stats_run.py C3 [preroll] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_17790_b200 as nsf  # noqa: E402
import scenes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
pre = int(sys.argv[2]) if len(sys.argv) > 2 else 250
K = int(sys.argv[3]) if len(sys.argv) > 3 else 32
sc = scenes.by_name(name)
sim = nsf.Simulator(sc.cfg)
sim.load_scene(sc)
sim.substep(pre)
sim.sync()
nsf.nsf_mpm_debug_stats(sim.h)
if os.environ.get("FLUSH"):   # the bench's regime: L2 flushed before every substep
    import torch
    flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
    for _ in range(K):
        torch.sum(flush)
        torch.cuda.synchronize()
        sim.substep(1)
        sim.sync()
else:
    sim.substep(K)
st = nsf.nsf_mpm_debug_stats(sim.h)
sim.close()
per = {k: v / K for k, v in st.items()}
n = sc.n
print(f"{name} substeps {pre}..{pre + K}: per substep " + ", ".join(f"{k} {v:.0f}" for k, v in per.items()))
tot = per["cyc_tile"] + per["cyc_phase1"] + per["cyc_phase2"]
print(f"  cycles share: tile {per['cyc_tile'] / tot:.2f} phase1 {per['cyc_phase1'] / tot:.2f} "
      f"phase2 {per['cyc_phase2'] / tot:.2f}; per segment: tile {per['cyc_tile'] / per['segments']:.0f} "
      f"p1 {per['cyc_phase1'] / per['segments']:.0f} p2 {per['cyc_phase2'] / per['segments']:.0f} cycles; "
      f"listed {per['listed'] / n:.3%} inline {per['inline'] / n:.3%} out-of-tile {per['out_of_tile'] / n:.3%} "
      f"out-of-block {per['out_of_block'] / n:.3%}; phase 2 of thread 0 (accumulate) "
      f"{per['cyc_p2_acc'] / per['segments']:.0f}, of the last helper {per['cyc_p2_help'] / per['segments']:.0f} cycles")
if per.get("ctas"):
    print(f"  kernel {per['kern_ns'] / 1e3:.1f} us per launch, CTA idle at the end {per['tail_ns'] / per['ctas'] / 1e3:.2f} us "
          f"on average ({per['tail_ns'] / (per['ctas'] * per['kern_ns']):.1%} of the CTA-time), "
          f"{per['ctas'] * K / max(per['segments'] * K, 1):.3f} CTAs per segment")
