#!/bin/bash
set -x
N=4 SPREADS=first,10,20,30,40 R=3 python tools/spread_probe.py > gpurun_out/spread2_c2_n4.txt 2>&1
N=2 SPREADS=first,20,30 R=3 python tools/spread_probe.py > gpurun_out/spread2_c2_n2.txt 2>&1
N=4 ODF=64 SPREADS=first,20,30 R=2 python tools/spread_probe.py > gpurun_out/spread2_c2odf64_n4.txt 2>&1
N=4 CFG=c3 SPREADS=first,20,30 R=2 python tools/spread_probe.py > gpurun_out/spread2_c3_n4.txt 2>&1
N=4 CFG=c5 SPREADS=first,20,30 R=2 python tools/spread_probe.py > gpurun_out/spread2_c5_n4.txt 2>&1
N=4 CFG=c4 ODF=16 SPREADS=first,20,30 R=2 K=20 python tools/spread_probe.py > gpurun_out/spread2_c4_n4.txt 2>&1
cat gpurun_out/spread2_*.txt
