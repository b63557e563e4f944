#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for cfg in 32,8,4 32,4,8 64,4,4 64,2,8 32,8,2 128,2,4 64,4,2 128,2,2 32,8,8 256,1,4; do
  echo "cfg $cfg" 
  TCG_UNTILED_CFG=$cfg timeout 300 python tools/ab_modes.py c2 "untiled;untiled" 2>&1 | tail -1
done > gpurun_out/sweep_untiled.log 2>&1
