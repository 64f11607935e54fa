F=gpurun_out/w8; mkdir -p $F
VARS=0,5,15 BLOCKS=1x1x1,2x2x2,2x2x4,4x4x4 timeout 600 python tools/var_probe.py > $F/probe.log 2>&1
