for n in 512 768; do
  for i in 0 1; do echo "N=$n INTERIOR=$i"; N=$n INTERIOR=$i python tools/e2e_probe.py | tail -2; done
done
python bench.py --steps 20 --warmup 5 --no-sweep > gpurun_out/r02g_bench_n1.json 2> gpurun_out/r02g_bench_n1.err
python bench.py --config c3 --steps 20 --warmup 5 --no-sweep > gpurun_out/r02g_bench_c3_n1.json 2> gpurun_out/r02g_bench_c3_n1.err
