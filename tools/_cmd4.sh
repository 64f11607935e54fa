F=gpurun_out/final11; mkdir -p $F
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $F/pytest_gpu.log
R="python -m torch.distributed.run --nnodes 1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 python bench.py > $F/bench_c2_n1.json 2> $F/bench_c2_n1.err
for n in 2 4; do $R --nproc-per-node $n --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n > $F/bench_c2_n$n.json 2> $F/bench_c2_n$n.err; done
for cfg in c3; do
  CUDA_VISIBLE_DEVICES=0 python bench.py --config $cfg --no-sweep --no-cpu > $F/bench_${cfg}_n1.json 2> /dev/null
  for n in 2 4; do $R --nproc-per-node $n --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --config $cfg --no-sweep > $F/bench_${cfg}_n$n.json 2> $F/bench_${cfg}_n$n.err; done
done
for o in 1 16; do
  CUDA_VISIBLE_DEVICES=0 python bench.py --config c4 --odf $o --no-sweep --no-cpu --no-e2e > $F/bench_c4odf${o}_n1.json 2> $F/bench_c4odf${o}_n1.err
  for n in 2 4; do $R --nproc-per-node $n --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --config c4 --odf $o --no-sweep --no-e2e > $F/bench_c4odf${o}_n$n.json 2> $F/bench_c4odf${o}_n$n.err; done
done
export CUDA_VISIBLE_DEVICES=0
for b in "1 1 1" "2 2 2"; do
  tag=$(echo $b | tr -d ' ')
  python tools/profile_sweep.py --blocks $b --iters 3 >> $F/pre_full.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sweep -c 1 -o $F/r01b_sweep_blocks$tag -f python tools/profile_sweep.py --blocks $b --iters 2 > /dev/null 2>&1
done
python bench.py --no-sweep --no-cpu --no-e2e --no-sustained --steps 20 --warmup 3 > $F/pre_ncu.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $F/launches_c2.csv python bench.py --no-sweep --no-cpu --no-e2e --no-sustained --steps 20 --warmup 3 > $F/ncu_launch.log 2>&1
