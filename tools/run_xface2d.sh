# 2-D x faces through shared memory: parity, same-box A/B vs _prev
python -m pytest tests/test_parity2d_gpu.py tests/test_virtual_remote_gpu.py tests/test_multigpu_gpu.py tests/test_fullsize_gpu.py tests/test_checked_build_gpu.py tests/test_parity_fuzz_gpu.py -q -m gpu -x 2>&1 | tail -2
ROOT_B=_prev REPS=3 CASES=2d32768x32768:1x1,2d32768x32768:2x4,2d32768x32768:8x8,2d8192x8192:16x16 python tools/ab_trees.py 2>&1 | tail -4
ROOT_B=_prev REPS=3 AB_GPUS=2 CASES=2d65536x32768:2x1 python tools/ab_trees.py 2>&1 | tail -1
