#!/bin/bash
# 4-GPU measurement campaign: multi-GPU parity, NEXT-3 microbenchmarks over NVLink, bench lines
# at N = 2 and 4 (one process: every config; torchrun: C2), j2d strong scaling.
set -x
python -m pytest tests/test_multigpu_gpu.py tests/test_microbench_gpu.py "tests/test_fullsize_gpu.py::test_j2d_strong_paper_grid_multi_gpu" -q -m gpu 2>&1 | tail -6 > gpurun_out/r02_t_multi.log
python tools/microbench.py > gpurun_out/r02_microbench_4xB200.json 2> gpurun_out/r02_microbench.err
for n in 2 4; do
  python bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r02_bench_sp_n$n.json 2> gpurun_out/r02_bench_sp_n$n.err
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r02_bench_tr_n$n.json 2> gpurun_out/r02_bench_tr_n$n.err
  for cfg in c3 c5 j2d; do
    python bench.py --gpus $n --config $cfg --steps 20 --warmup 5 --no-sweep > gpurun_out/r02_bench_${cfg}_n$n.json 2> gpurun_out/r02_bench_${cfg}_n$n.err
  done
  python bench.py --gpus $n --config c4 --odf 16 --steps 10 --warmup 3 --no-sweep --no-e2e > gpurun_out/r02_bench_c4_odf16_n$n.json 2> gpurun_out/r02_bench_c4_odf16_n$n.err
  for odf in 1 8 16; do
    python bench.py --gpus $n --config j2d_strong --odf $odf --steps 10 --warmup 3 --no-sweep > gpurun_out/r02_bench_j2d_strong_odf${odf}_n$n.json 2> gpurun_out/r02_bench_j2d_strong_odf${odf}_n$n.err
  done
done
cat gpurun_out/r02_t_multi.log
