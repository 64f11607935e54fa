F=gpurun_out/ncu3; mkdir -p $F
for b in "2 2 4" "4 4 4" "8 8 8"; do
  tag=$(echo $b | tr -d ' ')
  python tools/profile_sweep.py --blocks $b --iters 3 >> $F/pre.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sweep -c 1 -o $F/r01b_sweep_blocks$tag -f python tools/profile_sweep.py --blocks $b --iters 2 > /dev/null 2>&1
done
