#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for lm in 0 1 2; do for c in c2 c3; do
 echo "lm $lm"; TCG_L2_LOADS=$lm TCG_L2_ITEM_US=100 python tools/ab_modes.py $c "tiled:0,0,0" 2>&1 | tail -1
 TCG_L2_LOADS=$lm python tools/ab_modes.py $c "tiled:0,0,0" 2>&1 | tail -1
done; done > gpurun_out/lm.log 2>&1
