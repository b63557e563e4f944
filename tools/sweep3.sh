#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
bash tools/ab_l2.sh
for cfg in 32,8,4 32,8,8 64,4,4 64,4,8 32,4,8 128,2,8 64,2,8 256,1,8; do
  echo "cfg3 $cfg"; TCG_UNTILED_CFG3=$cfg python tools/ab_modes.py c3 untiled 2>&1 | tail -1
done >> gpurun_out/ab_l2.log 2>&1
