set -e
python -m pytest tests/test_parity2d_gpu.py -q -m gpu 2>&1 | tail -3
R=3 python tools/xband_probe.py 2>&1 | tail -6
