F=gpurun_out/final4; mkdir -p $F
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $F/pytest_gpu.log
R="python -m torch.distributed.run --nnodes 1 --master-addr 127.0.0.1"
for cfg in c2 c3 j2d; do
  CUDA_VISIBLE_DEVICES=0 python bench.py --config $cfg --no-sweep --no-cpu > $F/bench_${cfg}_n1.json 2> $F/bench_${cfg}_n1.err
  for n in 2 4; do $R --nproc-per-node $n --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --config $cfg > $F/bench_${cfg}_n$n.json 2> $F/bench_${cfg}_n$n.err; done
done
for o in 1 16; do
  CUDA_VISIBLE_DEVICES=0 python bench.py --config c4 --odf $o --no-sweep --no-cpu --no-e2e > $F/bench_c4odf${o}_n1.json 2> $F/bench_c4odf${o}_n1.err
  for n in 2 4; do $R --nproc-per-node $n --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --config c4 --odf $o --no-sweep --no-e2e > $F/bench_c4odf${o}_n$n.json 2> $F/bench_c4odf${o}_n$n.err; done
done
CUDA_VISIBLE_DEVICES=0 python bench.py --config c5 --no-sweep --no-cpu --no-e2e > $F/bench_c5_n1.json 2> $F/bench_c5_n1.err
for n in 2 4; do $R --nproc-per-node $n --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --config c5 --no-sweep --no-e2e > $F/bench_c5_n$n.json 2> $F/bench_c5_n$n.err; done
$R --nproc-per-node 4 --master-port $((29500 + RANDOM % 400)) bench.py --gpus 4 --impl reference --steps 3 --warmup 3 > $F/bench_ref_n4.json 2> $F/bench_ref_n4.err
