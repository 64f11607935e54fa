timeout 1200 python -m pytest tests/test_multigpu_gpu.py -m gpu -q 2>&1 | tail -4 > gpurun_out/mp_tests.log
R="python -m torch.distributed.run --nnodes 1 --master-addr 127.0.0.1"
for i in 1 2; do
for n in 1 2 4; do
REPS=2 timeout 300 $R --nproc-per-node $n --master-port $((29800 + RANDOM % 100)) tools/mp_perf.py 2>/dev/null | grep "^N="
done; done > gpurun_out/mp.log 2>&1
