F=gpurun_out/final3; mkdir -p $F
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $F/smoke.log 2>&1
python bench.py > $F/bench_c2_n1.json 2> $F/bench_c2_n1.err
python bench.py --config j2d --no-cpu > $F/bench_j2d_n1.json 2> $F/bench_j2d_n1.err
python bench.py --impl reference --steps 3 --warmup 3 > $F/bench_ref_n1.json 2> $F/bench_ref_n1.err
python bench.py --no-sweep --no-cpu --no-e2e --no-sustained --steps 20 --warmup 3 > $F/pre_ncu.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $F/launches_c2.csv python bench.py --no-sweep --no-cpu --no-e2e --no-sustained --steps 20 --warmup 3 > $F/ncu_launch.log 2>&1
for b in "1 1 1" "2 2 2" "2 2 4" "4 4 4" "8 8 8" "16 16 16"; do
  tag=$(echo $b | tr -d ' ')
  python tools/profile_sweep.py --blocks $b --iters 3 >> $F/pre_full.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sweep -c 1 -o $F/r01b_sweep_blocks$tag -f python tools/profile_sweep.py --blocks $b --iters 2 > /dev/null 2>&1
done
python tools/profile_sweep.py --dims 32768 32768 1 --blocks 2 4 1 --flags 512 --iters 3 >> $F/pre_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep -c 1 -o $F/r01b_sweep2d_32768sq_odf8 -f python tools/profile_sweep.py --dims 32768 32768 1 --blocks 2 4 1 --flags 512 --iters 2 > /dev/null 2>&1
ls $F >> $F/pre_full.log
