#!/bin/bash
# power-capped steady state, C2 ODF 8 / ODF 1: z-chunk and column-group settings
export JAC_EXPERIMENT=1
SETTLE=3000 N=500 K=3 ODFS=8,1 SETTINGS="JAC_AUTOTUNE=1;JAC_ZCHUNK=32;JAC_ZCHUNK=32,JAC_GCOLS=444;JAC_VARIANT=5;JAC_VARIANT=5,JAC_ZCHUNK=32" \
  python tools/steady_probe.py > gpurun_out/steady_r02.txt 2>&1
cat gpurun_out/steady_r02.txt
