# ncu launch list of the bench command (one ncu invocation, after the same command ran without it)
python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu --no-e2e --no-sustained > gpurun_out/launch_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_bench_n1.csv \
  python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu --no-e2e --no-sustained > gpurun_out/launch_ncu.log 2>&1
tail -2 gpurun_out/launch_plain.json | cut -c1-200
