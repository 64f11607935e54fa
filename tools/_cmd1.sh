F=gpurun_out/promo; mkdir -p $F
ODFS=1,8,64,4096 SETTINGS="JAC_L2PROMO=256;JAC_L2PROMO=128;JAC_L2PROMO=64;JAC_L2PROMO=0;JAC_L2PROMO=256" K=2 timeout 600 python tools/steady_probe.py > $F/steady.log 2>&1
for p in 256 64 0; do
for b in "16 16 16" "4 4 4" "1 1 1"; do
JAC_L2PROMO=$p python tools/profile_sweep.py --blocks $b --iters 3 >> $F/pre.log 2>&1 && \
JAC_L2PROMO=$p ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:sweep -c 1 python tools/profile_sweep.py --blocks $b --iters 2 2>&1 | grep -E "dram|duration" | sed "s/^/promo=$p blocks=$b /" >> $F/ncu.log
done; done
