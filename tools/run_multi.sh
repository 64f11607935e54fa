#!/bin/bash
# 4-GPU check: multi-GPU parity (single process and torchrun), NVLink microbenchmark
# content checks, single-process and torchrun bench lines.
set -x
python -m pytest tests/test_multigpu_gpu.py tests/test_microbench_gpu.py -q -m gpu 2>&1 | tail -15 > gpurun_out/t4.log
for n in 2 4; do
  python bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/b_sp$n.json 2> gpurun_out/b_sp$n.err
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29513 \
    bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/b_tr$n.json 2> gpurun_out/b_tr$n.err
done
python bench.py --gpus 1 --steps 20 --warmup 5 --no-sweep --no-cpu > gpurun_out/b_sp1.json 2> gpurun_out/b_sp1.err
cat gpurun_out/t4.log
