#!/bin/bash
set -x
N=4 python tools/spread_probe.py > gpurun_out/spread_n4.txt 2>&1
N=2 SPREADS=first,50 python tools/spread_probe.py > gpurun_out/spread_n2.txt 2>&1
N=4 CFG=c3 SPREADS=first,50 R=2 python tools/spread_probe.py > gpurun_out/spread_c3_n4.txt 2>&1
N=4 python tools/nvlink_probe.py > gpurun_out/nvl_plain_n4b.txt 2>&1 &&
N=4 ncu --metrics nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:sweep_tma -s 4 -c 4 --csv --log-file gpurun_out/nvl_ncu_n4b.csv \
    python tools/nvlink_probe.py > gpurun_out/nvl_ncu_n4b.log 2>&1
cat gpurun_out/spread_*.txt
