#!/bin/bash
# final 4-GPU campaign: N = 1, 2, 4 bench lines from ONE lease (same-box scaling), both launchers for C2
set -x
for cfg in c2 c3 c5 j2d; do
  python bench.py --gpus 1 --config $cfg --steps 20 --warmup 5 --no-sweep --no-cpu --no-e2e > gpurun_out/${PFX:-f}_${cfg}_n1.json 2> gpurun_out/${PFX:-f}_${cfg}_n1.err
done
python bench.py --gpus 1 --config c4 --odf 16 --steps 10 --warmup 3 --no-sweep --no-cpu --no-e2e > gpurun_out/${PFX:-f}_c4_n1.json 2> gpurun_out/${PFX:-f}_c4_n1.err
for n in 2 4; do
  python bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/${PFX:-f}_c2_n$n.json 2> gpurun_out/${PFX:-f}_c2_n$n.err
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29519 \
    bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/${PFX:-f}_c2tr_n$n.json 2> gpurun_out/${PFX:-f}_c2tr_n$n.err
  for cfg in c3 c5 j2d; do
    python bench.py --gpus $n --config $cfg --steps 20 --warmup 5 --no-sweep --no-e2e > gpurun_out/${PFX:-f}_${cfg}_n$n.json 2> gpurun_out/${PFX:-f}_${cfg}_n$n.err
  done
  python bench.py --gpus $n --config c4 --odf 16 --steps 10 --warmup 3 --no-sweep --no-e2e > gpurun_out/${PFX:-f}_c4_n$n.json 2> gpurun_out/${PFX:-f}_c4_n$n.err
  for odf in 1 16; do
    python bench.py --gpus $n --config j2d_strong --odf $odf --steps 10 --warmup 3 --no-sweep > gpurun_out/${PFX:-f}_j2ds_odf${odf}_n$n.json 2> gpurun_out/${PFX:-f}_j2ds_odf${odf}_n$n.err
  done
done
ls gpurun_out/${PFX:-f}_*.json | wc -l
