# timing first (no profiler), then one ncu --set full of the three cases' single profile_sweep launch
set -e
python tools/j2d_wide_probe.py
NO_TIMING=1 ncu --set full --clock-control none -k regex:sweep2d -c 3 -o gpurun_out/r02_ncu_j2d_wide python tools/j2d_wide_probe.py > gpurun_out/ncu_j2d_wide.log 2>&1
tail -3 gpurun_out/ncu_j2d_wide.log
