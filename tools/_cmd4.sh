F=gpurun_out/c5final; mkdir -p $F
R="python -m torch.distributed.run --nnodes 1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 python bench.py --config c5 --no-sweep --no-cpu --no-e2e > $F/bench_c5_n1.json 2> $F/bench_c5_n1.err
for n in 2 4; do $R --nproc-per-node $n --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --config c5 --no-sweep --no-e2e > $F/bench_c5_n$n.json 2> $F/bench_c5_n$n.err; done
export CUDA_VISIBLE_DEVICES=0
python tools/profile_sweep.py --blocks 16 16 16 --iters 3 > $F/pre.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep -c 1 -o $F/r01b_sweep_blocks161616 -f python tools/profile_sweep.py --blocks 16 16 16 --iters 2 > /dev/null 2>&1
