F=gpurun_out/n4check; mkdir -p $F
R="python -m torch.distributed.run --nnodes 1 --master-addr 127.0.0.1"
for rep in 1 2; do
$R --nproc-per-node 4 --master-port $((29500 + RANDOM % 400)) bench.py --gpus 4 --no-e2e > $F/bench_c2_n4_$rep.json 2> $F/err_$rep.log
JAC_NO_DENSE=1 $R --nproc-per-node 4 --master-port $((29500 + RANDOM % 400)) bench.py --gpus 4 --no-sweep --no-e2e --no-sustained > $F/bench_c2_n4_nodense_$rep.json 2> /dev/null
done
