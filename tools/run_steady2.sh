#!/bin/bash
export JAC_EXPERIMENT=1
SETTLE=3000 N=500 K=3 ODFS=8,1 SETTINGS="JAC_AUTOTUNE=1;JAC_VARIANT=15;JAC_VARIANT=0;JAC_VARIANT=15,JAC_ZCHUNK=32" \
  python tools/steady_probe.py > gpurun_out/steady_r02b.txt 2>&1
cat gpurun_out/steady_r02b.txt
