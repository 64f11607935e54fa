F=gpurun_out/driverlike2; mkdir -p $F
python bench.py --gpus 1 --steps 20 --warmup 3 --no-sweep > $F/n1.json 2> $F/n1.err; echo "n1 rc=$?" >> $F/rc.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 20 --warmup 3 > $F/n2.json 2> $F/n2.err; echo "n2 rc=$?" >> $F/rc.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > $F/ref2.json 2> $F/ref2.err; echo "ref2 rc=$?" >> $F/rc.log
