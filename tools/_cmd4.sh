F=gpurun_out/final4; mkdir -p $F
R="python -m torch.distributed.run --nnodes 1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 python bench.py --config j2d --no-sweep --no-cpu > $F/bench_j2d_n1.json 2> $F/bench_j2d_n1.err
for n in 2 4; do $R --nproc-per-node $n --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --config j2d > $F/bench_j2d_n$n.json 2> $F/bench_j2d_n$n.err; done
