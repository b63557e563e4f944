#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for c in c2 c3 c1 c4; do
  python tools/ab_modes.py $c "untiled" 2>&1 | tail -1
  python tools/ab_modes.py $c "tiled:0,0,0" 2>&1 | tail -1
  TCG_L2_ITEM_US=100 python tools/ab_modes.py $c "tiled:0,0,0" 2>&1 | tail -1
done > gpurun_out/ab_l2.log 2>&1
