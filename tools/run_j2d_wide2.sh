# wide-row penalty vs tile shape (rows per staged box) and y-chunk length
VARS=5,15,1 R=3 python tools/j2d_wide_probe.py
echo "-- JAC_YCHUNK=2"; JAC_EXPERIMENT=1 JAC_YCHUNK=2 R=3 python tools/j2d_wide_probe.py
echo "-- JAC_YCHUNK=32"; JAC_EXPERIMENT=1 JAC_YCHUNK=32 R=3 python tools/j2d_wide_probe.py
