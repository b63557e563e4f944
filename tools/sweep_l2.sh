#!/bin/bash
# L2-tiled executor: sub-chain length / budget sweep on c3 and c2; c1 host overhead.
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-l2}; mkdir -p $OUT
timeout 300 python tools/ab_modes.py c1 "untiled;windowed;tiled:0,0,0" > $OUT/c1.log 2>&1
for ml in 2 4 8; do for b in 64 88; do
  TCG_L2_MAXLOOPS=$ml TCG_L2_BUDGET_MB=$b AB_STEPS=5 timeout 300 python tools/ab_modes.py c3 "tiled:0,0,0" > $OUT/c3_ml${ml}_b$b.log 2>&1
done; done
AB_STEPS=5 timeout 300 python tools/ab_modes.py c3 "tiled:0,0,0;untiled" > $OUT/c3_default.log 2>&1
for ml in 2 3 4 6; do TCG_L2_MAXLOOPS=$ml timeout 300 python tools/ab_modes.py c2 "tiled:0,0,0" > $OUT/c2_ml$ml.log 2>&1; done
for ml in 2 4 8; do TCG_L2_MAXLOOPS=$ml timeout 300 python tools/ab_modes.py c1 "tiled:0,0,0" > $OUT/c1_ml$ml.log 2>&1; done
