# x faces through shared memory: parity (whole GPU suite), same-box A/B vs _prev, NVLink bytes of an x split (one ncu)
python -m pytest tests -q -m gpu -x 2>&1 | tail -2
ROOT_B=_prev REPS=3 CASES=512x512x512:1x1x1,512x512x512:2x2x2,512x512x512:4x4x4,512x512x512:8x8x8,512x512x512:16x16x16,1024x1024x1024:32x32x32 python tools/ab_trees.py 2>&1 | tail -6
ROOT_B=_prev REPS=3 AB_GPUS=2 CASES=1024x512x512:2x2x2 python tools/ab_trees.py 2>&1 | tail -1
M=nvltx__bytes_data_user.sum,nvltx__bytes.sum,gpu__time_duration.sum
N=2 GRID=2x1x1 python tools/nvlink_probe.py > gpurun_out/nvlx_plain_smem.txt 2>&1 && \
N=2 GRID=2x1x1 ncu --metrics $M --clock-control none -k regex:sweep_tma -s 4 -c 2 --csv \
    --log-file gpurun_out/nvlx_ncu_smem.csv python tools/nvlink_probe.py > gpurun_out/nvlx_ncu_smem.log 2>&1
tail -3 gpurun_out/nvlx_plain_smem.txt; grep -h nvltx__bytes_data_user gpurun_out/nvlx_ncu_smem.csv | head -4
