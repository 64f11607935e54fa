#!/bin/bash
# NVLink bytes of x-split remote faces (x-ghost arrays): current tree vs _prev (8-byte x-face stores)
M=nvltx__bytes_data_user.sum,nvltx__bytes.sum,gpu__time_duration.sum
for tree in cur prev; do
  R=""; [ $tree = prev ] && R=$PWD/_prev
  PROBE_ROOT=$R N=2 GRID=2x1x1 python tools/nvlink_probe.py > gpurun_out/nvlx_plain_$tree.txt 2>&1 &&
  PROBE_ROOT=$R N=2 GRID=2x1x1 ncu --metrics $M --clock-control none -k regex:sweep_tma -s 4 -c 2 --csv \
    --log-file gpurun_out/nvlx_ncu_$tree.csv python tools/nvlink_probe.py > gpurun_out/nvlx_ncu_$tree.log 2>&1
done
cat gpurun_out/nvlx_plain_cur.txt
