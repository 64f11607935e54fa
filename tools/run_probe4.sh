#!/bin/bash
# 4-GPU lease: N=4 coupling probe, NVLink counters at N=2 and N=4, ncu of the 32^3-block sweep
set -x
N=4 python tools/n4_probe.py > gpurun_out/n4_probe.txt 2>&1
N=2 python tools/n4_probe.py > gpurun_out/n2_probe.txt 2>&1
for n in 2 4; do
  N=$n python tools/nvlink_probe.py > gpurun_out/nvl_plain_n$n.txt 2>&1 &&
  N=$n ncu --metrics nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,nvltx__bytes.sum,nvlrx__bytes.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:sweep_tma -s 4 -c 4 --csv --log-file gpurun_out/nvl_ncu_n$n.csv \
    python tools/nvlink_probe.py > gpurun_out/nvl_ncu_n$n.log 2>&1
done
python tools/profile_sweep.py --dims 512 512 512 --blocks 16 16 16 --iters 4 > gpurun_out/prof32_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:sweep_tma -s 0 -c 1 -o gpurun_out/prof32 \
  python tools/profile_sweep.py --dims 512 512 512 --blocks 16 16 16 --iters 4 > gpurun_out/prof32_ncu.log 2>&1
tail -5 gpurun_out/*.txt
