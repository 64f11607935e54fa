# 4-GPU A/B of the 2-D x-face change on the paper's strong grid at ODF 16 and 1 (A = current, B = _prev)
ROOT_B=_prev REPS=3 AB_GPUS=4 CASES=2d131072x98304:8x8,2d131072x98304:2x2 python tools/ab_trees.py 2>&1 | tail -2
ROOT_B=_prev REPS=3 CASES=2d16384x12288:4x4,2d65536x49152:4x4 python tools/ab_trees.py 2>&1 | tail -2
