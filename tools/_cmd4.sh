F=gpurun_out/pdl; mkdir -p $F
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/pdl_probe.py > $F/probe.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $F/pytest_gpu.log
