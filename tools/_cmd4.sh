F=gpurun_out/final6; mkdir -p $F
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $F/pytest_gpu.log
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $F/smoke.log 2>&1
export CUDA_VISIBLE_DEVICES=0
python tools/profile_sweep.py --blocks 8 8 8 --iters 3 > $F/pre.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep -c 1 -o $F/r01b_sweep_blocks888 -f python tools/profile_sweep.py --blocks 8 8 8 --iters 2 > /dev/null 2>&1
