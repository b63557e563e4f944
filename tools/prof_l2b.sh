#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TCG_L2_ITEM_US=100 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_l2tiled -s 8 -c 1 -o gpurun_out/c2_l2single -f \
  python tools/ab_modes.py c2 "tiled:0,0,0" > gpurun_out/ncu_l2s.log 2>&1; echo "ncu rc=$?"
