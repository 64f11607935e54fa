# zero-copy (JAC_DIRECT=1: kernels read / write the pinned host box) vs staged slabs
JAC_EXPERIMENT=1 JAC_DIRECT=1 python -m pytest tests/test_host_transfer_gpu.py -q -m gpu -k pinned 2>&1 | tail -1
for n in 512; do
  echo "N=$n staged"; N=$n python tools/e2e_probe.py | tail -2
  echo "N=$n direct"; JAC_EXPERIMENT=1 JAC_DIRECT=1 N=$n python tools/e2e_probe.py | tail -2
done
echo "C5 direct"; JAC_EXPERIMENT=1 JAC_DIRECT=1 N=1024 BLOCKS=32x32x32 python tools/e2e_probe.py | tail -2
echo "2D-like wide rows direct"; JAC_EXPERIMENT=1 JAC_DIRECT=1 N=512 BLOCKS=1x1x1 python tools/e2e_probe.py | tail -1
