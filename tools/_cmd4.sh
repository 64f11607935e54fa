F=gpurun_out/ranks2; mkdir -p $F
R="python -m torch.distributed.run --nnodes 1 --master-addr 127.0.0.1"
for rep in 1 2; do
  # four independent 1-GPU runs at the same time (no communication at all)
  for g in 0 1 2 3; do CUDA_VISIBLE_DEVICES=$g python bench.py --no-sweep --no-e2e --no-sustained --no-cpu --steps 2000 > $F/conc_${rep}_gpu$g.json 2>/dev/null & done; wait
  for g in 0 1 2 3; do CUDA_VISIBLE_DEVICES=$g python bench.py --no-sweep --no-e2e --no-sustained --no-cpu --steps 2000 > $F/solo_${rep}_gpu$g.json 2>/dev/null; done
  $R --nproc-per-node 4 --master-port $((29500 + RANDOM % 400)) bench.py --gpus 4 --no-sweep --no-e2e --no-sustained --steps 2000 > $F/n4_${rep}.json 2> /dev/null
  JAC_NO_FUSED_SYNC=1 $R --nproc-per-node 4 --master-port $((29500 + RANDOM % 400)) bench.py --gpus 4 --no-sweep --no-e2e --no-sustained --steps 2000 > $F/n4nofused_${rep}.json 2> /dev/null
done
