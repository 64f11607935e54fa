F=gpurun_out/final5; mkdir -p $F
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $F/smoke.log 2>&1
python bench.py > $F/bench_c2_n1.json 2> $F/bench_c2_n1.err
python bench.py --config j2d --no-cpu > $F/bench_j2d_n1.json 2> $F/bench_j2d_n1.err
python bench.py --impl reference --steps 3 --warmup 3 > $F/bench_ref_n1.json 2> $F/bench_ref_n1.err
python bench.py --no-sweep --no-cpu --no-e2e --no-sustained --steps 20 --warmup 3 > $F/pre_ncu.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $F/launches_c2.csv python bench.py --no-sweep --no-cpu --no-e2e --no-sustained --steps 20 --warmup 3 > $F/ncu_launch.log 2>&1
