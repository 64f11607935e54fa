#!/bin/bash
# 1-GPU measurement campaign: bench lines per config, tile-variant check for 32-wide blocks,
# ncu launch list of the default bench command and a full capture of the C2 ODF 8 sweep
# (-s 20: skips the 18 create-time autotune sweeps and the first two profiled ones).
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_n1.json 2> gpurun_out/r02_bench_n1.err
for cfg in c3 c5 j2d; do
  python bench.py --config $cfg --steps 20 --warmup 5 --no-sweep > gpurun_out/r02_bench_${cfg}_n1.json 2> gpurun_out/r02_bench_${cfg}_n1.err
done
for odf in 1 16; do
  python bench.py --config c4 --odf $odf --steps 10 --warmup 3 --no-sweep --no-e2e > gpurun_out/r02_bench_c4_odf${odf}_n1.json 2> gpurun_out/r02_bench_c4_odf${odf}_n1.err
done
export JAC_EXPERIMENT=1
REPS=2 DIMS=64x64x64 BLOCKS=2x2x2 VARS=3,12 python tools/var_probe.py > gpurun_out/var_c1.txt 2>&1
REPS=2 DIMS=1024x1024x1024 BLOCKS=32x32x32 VARS=3,12 python tools/var_probe.py > gpurun_out/var_c5.txt 2>&1
REPS=2 DIMS=512x512x512 BLOCKS=16x16x16 VARS=3,12 python tools/var_probe.py > gpurun_out/var_512_32.txt 2>&1
REPS=2 DIMS=96x66x40 BLOCKS=3x3x5 VARS=3,12 python tools/var_probe.py > gpurun_out/var_rag.txt 2>&1
unset JAC_EXPERIMENT
python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu --no-e2e --no-sustained > gpurun_out/launch_plain.json 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_bench_n1.csv \
  python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu --no-e2e --no-sustained > gpurun_out/launch_ncu.log 2>&1
python tools/profile_sweep.py --dims 512 512 512 --blocks 2 2 2 --iters 4 > gpurun_out/prof_odf8_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:sweep_tma -s 20 -c 1 -o gpurun_out/r02_prof_odf8 \
  python tools/profile_sweep.py --dims 512 512 512 --blocks 2 2 2 --iters 4 > gpurun_out/prof_odf8_ncu.log 2>&1
cat gpurun_out/var_*.txt
