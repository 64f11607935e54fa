F=gpurun_out/final8; mkdir -p $F
python bench.py > $F/bench_c2_n1.json 2> $F/bench_c2_n1.err
python bench.py --config j2d --no-cpu > $F/bench_j2d_n1.json 2> $F/bench_j2d_n1.err
