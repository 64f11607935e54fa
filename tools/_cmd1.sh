F=gpurun_out/order; mkdir -p $F
KNOB=JAC_ORDER_EXP VALUES=0,1,2 BLOCKS=2x2x2,2x2x4 timeout 600 python tools/env_probe.py > $F/probe.log 2>&1
