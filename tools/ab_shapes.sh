#!/bin/bash
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-sh}; mkdir -p $OUT
for cfg in "64,2,8" "64,2,4" "32,4,4" "32,8,4" "128,2,4" "32,2,4"; do
  TCG_UNTILED_CFG3=$cfg AB_STEPS=2 timeout 300 python tools/ab_modes.py c5 untiled > $OUT/c5_$cfg.log 2>&1
done
for cfg in "256,1,4" "256,1,8" "128,2,4" "256,1,2"; do
  TCG_UNTILED_CFG=$cfg timeout 300 python tools/ab_modes.py c2 untiled > $OUT/c2_$cfg.log 2>&1
done
