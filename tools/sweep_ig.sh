#!/bin/bash
# Item-graph form of the L2-tiled executor.
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-ig}; mkdir -p $OUT
TCG_L2_GRAPH=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest.log
TCG_L2_GRAPH=1 timeout 300 python tools/ab_modes.py c1 "tiled:0,0,0;untiled" > $OUT/c1.log 2>&1
TCG_L2_GRAPH=1 timeout 300 python tools/ab_modes.py c2 "tiled:0,0,0;untiled" > $OUT/c2.log 2>&1
for ml in 4 8; do TCG_L2_GRAPH=1 TCG_L2_MAXLOOPS=$ml timeout 300 python tools/ab_modes.py c2 "tiled:0,0,0" > $OUT/c2_ml$ml.log 2>&1; done
for ml in 2 4 8 16; do for b in 64 88; do
  TCG_L2_GRAPH=1 TCG_L2_MAXLOOPS=$ml TCG_L2_BUDGET_MB=$b AB_STEPS=5 timeout 300 python tools/ab_modes.py c3 "tiled:0,0,0" > $OUT/c3_ml${ml}_b$b.log 2>&1
done; done
TCG_L2_GRAPH=1 AB_STEPS=10 timeout 300 python tools/ab_modes.py c4 "tiled:0,0,0;untiled" > $OUT/c4.log 2>&1
