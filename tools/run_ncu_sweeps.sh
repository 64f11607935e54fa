# the plain run first, then ONE ncu --set full over the same command (2 launches per decomposition)
python tools/ncu_sweeps.py && \
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "jac_profile_sweep/" -c 6 \
  -o gpurun_out/r02_ncu_final_sweeps python tools/ncu_sweeps.py > gpurun_out/ncu_final_sweeps.log 2>&1
grep -v "^==PROF==" gpurun_out/ncu_final_sweeps.log | tail -5
