run() { n=$1; shift; tag=$1; shift; if [ $n = 1 ]; then timeout 600 python bench.py --gpus 1 "$@" > gpurun_out/scale_${tag}_n1.json 2> gpurun_out/scale_${tag}_n1.err; else timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $n "$@" > gpurun_out/scale_${tag}_n$n.json 2> gpurun_out/scale_${tag}_n$n.err; fi; }
for n in 1 2 4; do
run $n c3 --config c3 --steps 50 --warmup 3 --no-sweep --no-cpu --no-e2e
run $n c4odf1 --config c4 --odf 1 --steps 20 --warmup 3 --no-sweep --no-cpu --no-e2e
run $n c4odf16 --config c4 --odf 16 --steps 20 --warmup 3 --no-sweep --no-cpu --no-e2e
run $n c5 --config c5 --steps 50 --warmup 3 --no-sweep --no-cpu --no-e2e
run $n j2d --config j2d --steps 50 --warmup 3 --no-sweep --no-cpu --no-e2e
run $n c2 --steps 100 --warmup 5 --no-sweep --no-cpu --no-e2e
done
