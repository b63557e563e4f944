#!/bin/bash
# c2 executor sweep: windowed block/stream-tile shapes, prefetch, L2 options.
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-sw}; mkdir -p $OUT
M="untiled;windowed;windowed:128,16;windowed:256,16;windowed:128,32;windowed:64,32;windowed:64,64;windowed:384,8;windowed:192,16;tiled:0,0,0"
timeout 900 python tools/ab_modes.py c2 "$M" > $OUT/win.log 2>&1; echo "win rc=$?"
TCG_PREFETCH=1 timeout 600 python tools/ab_modes.py c2 "windowed;windowed:128,16;windowed:64,32" > $OUT/win_pf.log 2>&1; echo "pf rc=$?"
TCG_L2_DATAFLOW=1 timeout 600 python tools/ab_modes.py c2 "tiled:0,0,0" > $OUT/l2_df.log 2>&1; echo "df rc=$?"
for b in 24 48; do TCG_L2_BUDGET_MB=$b timeout 600 python tools/ab_modes.py c2 "tiled:0,0,0" > $OUT/l2_b$b.log 2>&1; done
timeout 600 python tools/ab_modes.py c1 "untiled;windowed;tiled:0,0,0;auto" > $OUT/c1.log 2>&1; echo "c1 rc=$?"
