F=gpurun_out/final9; mkdir -p $F
R="python -m torch.distributed.run --nnodes 1 --master-addr 127.0.0.1"
for n in 2 4; do $R --nproc-per-node $n --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n > $F/bench_c2_n$n.json 2> $F/bench_c2_n$n.err; done
timeout 1200 python -m pytest tests/test_multigpu_gpu.py -m gpu -q 2>&1 | tail -2 > $F/mp.log
