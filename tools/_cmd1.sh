F=gpurun_out/long; mkdir -p $F
timeout 300 python tools/long_run.py > $F/long.log 2>&1
