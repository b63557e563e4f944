#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for c in c2 c3; do python tools/ab_modes.py $c "tiled:0,0,0" 2>&1 | tail -1; done > gpurun_out/prof_l2_pre.log 2>&1
for v in 1 6 12; do echo "item_us $v"; TCG_L2_ITEM_US=$v python tools/ab_modes.py c2 "tiled:0,0,0" 2>&1 | tail -1; TCG_L2_ITEM_US=$v python tools/ab_modes.py c3 "tiled:0,0,0" 2>&1 | tail -1; done >> gpurun_out/prof_l2_pre.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_l2tiled -s 8 -c 1 -o gpurun_out/c2_l2 -f \
  python tools/ab_modes.py c2 "tiled:0,0,0" > gpurun_out/ncu_l2.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_l2tiled -s 8 -c 1 -o gpurun_out/c3_l2 -f \
  python tools/ab_modes.py c3 "tiled:0,0,0" > gpurun_out/ncu_l2_c3.log 2>&1; echo "ncu rc=$?"
