F=gpurun_out/resid; mkdir -p $F
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_parity_fuzz_gpu.py tests/test_fullsize_gpu.py -m gpu -q 2>&1 | tail -2 > $F/pytest.log
CASES=64x64x64:2x2x2,128x128x128:2x2x2,512x512x512:1x1x1,512x512x512:2x2x2,512x512x512:2x2x4,512x512x512:4x4x4,512x512x512:8x8x8,512x512x512:16x16x16,768x768x768:2x2x2 REPS=2 timeout 1500 python tools/ab_probe.py > $F/ab.log 2>&1
