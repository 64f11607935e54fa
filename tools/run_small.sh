#!/bin/bash
# small-block sweep: tile-variant A/B and one ncu --set full capture of the 32^3-block sweep
export JAC_EXPERIMENT=1
REPS=2 BLOCKS=16x16x16 VARS=3,13,12 python tools/var_probe.py > gpurun_out/var32.txt 2>&1
REPS=2 BLOCKS=8x8x8 VARS=4,14 python tools/var_probe.py > gpurun_out/var64.txt 2>&1
unset JAC_EXPERIMENT
python tools/profile_sweep.py --dims 512 512 512 --blocks 16 16 16 --iters 4 > gpurun_out/prof32b_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:sweep_tma -s 0 -c 1 -o gpurun_out/prof32b \
  python tools/profile_sweep.py --dims 512 512 512 --blocks 16 16 16 --iters 4 > gpurun_out/prof32b_ncu.log 2>&1
cat gpurun_out/var32.txt gpurun_out/var64.txt gpurun_out/prof32b_plain.log
