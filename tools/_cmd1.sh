F=gpurun_out/ncu2; mkdir -p $F
python tools/profile_sweep.py --blocks 16 16 16 --iters 3 > $F/pre.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep -c 1 -o $F/r01b_sweep_blocks161616 -f python tools/profile_sweep.py --blocks 16 16 16 --iters 2 > /dev/null 2>&1
python tools/profile_sweep.py --dims 32768 32768 1 --blocks 2 4 1 --flags 512 --iters 3 >> $F/pre.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep -c 1 -o $F/r01b_sweep2d_32768sq_odf8 -f python tools/profile_sweep.py --dims 32768 32768 1 --blocks 2 4 1 --flags 512 --iters 2 > /dev/null 2>&1
ls $F >> $F/pre.log
