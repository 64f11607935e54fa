"""One process, three C2-sized decompositions (512^3 in 2x2x2, 1x1x1 and 16x16x16
blocks): each context warms up with jac_step(2) (autotune, graphs), then runs
jac_profile_sweep(2) -- the launches an ncu capture with --nvtx --nvtx-include
"jac_profile_sweep/" sees (tools/run_ncu_sweeps.sh)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_12734_b200 as jb

for blocks in [(2, 2, 2), (1, 1, 1), (16, 16, 16)]:
    with jb.Jacobi3D((512, 512, 512), blocks) as s:
        s.set_init_hash(1)
        s.step(2)
        ms = s.profile_sweep(2)
        print(f"blocks {blocks}: avg sweep {ms * 1e3:.1f} us -> {16 * 512**3 / (ms * 1e-3) / 1e9:.0f} GB/s algorithmic", flush=True)
