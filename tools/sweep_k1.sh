#!/bin/bash
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-k1}; mkdir -p $OUT
TCG_CTAS_PER_SM=1 timeout 300 python tools/ab_modes.py c2 "windowed;windowed:128,8;windowed:192,8;windowed:256,8;windowed:128,16;windowed:96,16" > $OUT/c2_k1.log 2>&1
TCG_CTAS_PER_SM=1 TCG_WIN_MAXLOOPS=6 timeout 300 python tools/ab_modes.py c2 "windowed;windowed:256,8;windowed:384,8;windowed:256,16" > $OUT/c2_k1_ml6.log 2>&1
TCG_CTAS_PER_SM=2 TCG_WIN_MAXLOOPS=6 timeout 300 python tools/ab_modes.py c2 "windowed;windowed:128,8;windowed:192,8" > $OUT/c2_k2_ml6.log 2>&1
TCG_CTAS_PER_SM=1 timeout 300 python tools/ab_modes.py c1 "windowed;windowed:256,8;windowed:128,16;windowed:64,32" > $OUT/c1_k1.log 2>&1
