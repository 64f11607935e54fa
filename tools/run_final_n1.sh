#!/bin/bash
# final 1-GPU bench lines (no profiler): the default C2 line and the other configs
python bench.py --steps 20 --warmup 5 > gpurun_out/r02h_bench_n1.json 2> gpurun_out/r02h_bench_n1.err
for cfg in c3 c5 j2d; do
  python bench.py --config $cfg --steps 20 --warmup 5 --no-sweep > gpurun_out/r02h_bench_${cfg}_n1.json 2> gpurun_out/r02h_bench_${cfg}_n1.err
done
for odf in 1 16; do
  python bench.py --config c4 --odf $odf --steps 10 --warmup 3 --no-sweep --no-e2e > gpurun_out/r02h_bench_c4_odf${odf}_n1.json 2> gpurun_out/r02h_bench_c4_odf${odf}_n1.err
done
