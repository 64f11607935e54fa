#!/bin/bash
export JAC_EXPERIMENT=1
SETS="default;JAC_ZCHUNK=4;JAC_ZCHUNK=6;JAC_ZCHUNK=8;JAC_ZCHUNK=10" BLOCKS=1x1x1,2x2x2,2x2x4,4x4x4 python tools/zchunk_probe.py 2>&1 | tail -4
SETS="default;JAC_ZCHUNK=8" DIMS=768x768x768 BLOCKS=2x2x2 python tools/zchunk_probe.py 2>&1 | tail -1
SETS="default;JAC_ZCHUNK=8" DIMS=1536x1536x1536 BLOCKS=1x1x1,2x2x4 R=2 python tools/zchunk_probe.py 2>&1 | tail -2
SETTLE=3000 N=500 K=3 ODFS=8,1 SETTINGS="JAC_AUTOTUNE=1;JAC_ZCHUNK=8;JAC_ZCHUNK=16" python tools/steady_probe.py 2>&1 | tail -6
