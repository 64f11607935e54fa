F=gpurun_out/densefull; mkdir -p $F
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -8 > $F/pytest_gpu.log
CUDA_VISIBLE_DEVICES=0 CASES=64x64x64:2x2x2,512x512x512:16x16x16,512x512x512:8x8x8,512x512x512:2x2x2,1024x1024x1024:32x32x32 REPS=2 timeout 1200 python tools/ab_probe.py > $F/ab.log 2>&1
