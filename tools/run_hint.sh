#!/bin/bash
# mbarrier suspend-time hint A/B: cold (ab_trees) and power-capped steady state, current tree vs _hint/
ROOT_B=$PWD/_hint REPS=3 CASES=512x512x512:1x1x1,512x512x512:2x2x2,512x512x512:4x4x4,512x512x512:16x16x16,2d32768x32768:2x4 python tools/ab_trees.py 2>&1 | tail -5
for r in 1 2; do
  for tree in cur hint; do
    R=""; [ $tree = hint ] && R=$PWD/_hint
    PROBE_ROOT=$R SETTLE=3000 N=500 K=3 ODFS=8 SETTINGS="JAC_AUTOTUNE=1" python tools/steady_probe.py 2>&1 | tail -1 | sed "s/^/$tree /"
  done
done
