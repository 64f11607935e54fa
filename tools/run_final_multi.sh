#!/bin/bash
# final C2 bench lines at N = 2 / 4: one process (sp) and torchrun (tr), with the e2e leg
for n in 2 4; do
  python bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r02f_bench_sp_n$n.json 2> gpurun_out/r02f_bench_sp_n$n.err
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29521 \
    bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r02f_bench_tr_n$n.json 2> gpurun_out/r02f_bench_tr_n$n.err
done
python bench.py --gpus 1 --steps 20 --warmup 5 --no-sweep --no-cpu > gpurun_out/r02f_bench_same_n1.json 2> gpurun_out/r02f_bench_same_n1.err
ls -la gpurun_out/r02f_bench_*_n*.json
