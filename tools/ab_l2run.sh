#!/bin/bash
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-lr}; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest.log
timeout 300 python tools/ab_modes.py c1 "untiled;tiled:0,0,0;windowed;untiled;tiled:0,0,0" > $OUT/c1.log 2>&1
timeout 300 python tools/ab_modes.py c2 "untiled;tiled:0,0,0" > $OUT/c2.log 2>&1
TCG_L2_MAXLOOPS=4 AB_STEPS=5 timeout 300 python tools/ab_modes.py c3 "untiled;tiled:0,0,0" > $OUT/c3.log 2>&1
AB_STEPS=10 timeout 300 python tools/ab_modes.py c4 "untiled;tiled:0,0,0" > $OUT/c4.log 2>&1
