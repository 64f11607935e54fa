#!/bin/bash
# ncu --set full of the final sweep kernels (one GPU): C2 ODF 8 (2x2x2 blocks), ODF 1, 32^3 blocks (32x32 tiles)
# -s 20 skips the 18 autotune sweeps (run at the first profile on the initial field) and two profiled sweeps.
set -x
for b in "2 2 2" "1 1 1" "16 16 16"; do
  tag=$(echo $b | tr -d ' ')
  s=20; [ "$tag" = "161616" ] && s=2
  python tools/profile_sweep.py --dims 512 512 512 --blocks $b --iters 4 > gpurun_out/pf_$tag.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:sweep_tma -s $s -c 1 -o gpurun_out/r02_ncu_blocks$tag \
    python tools/profile_sweep.py --dims 512 512 512 --blocks $b --iters 4 > gpurun_out/pf_ncu_$tag.log 2>&1
done
cat gpurun_out/pf_*.log | grep -v "^==PROF=="
