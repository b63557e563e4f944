#!/bin/bash
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-rn}; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest.log
AB_STEPS=3 timeout 300 python tools/ab_modes.py c5 untiled > $OUT/c5.log 2>&1
AB_STEPS=5 timeout 300 python tools/ab_modes.py c3 untiled > $OUT/c3.log 2>&1
for cfg in "256,1,4" "256,1,8"; do for c in c1 c2 c4; do
  TCG_UNTILED_CFG=$cfg timeout 300 python tools/ab_modes.py $c "untiled;untiled" > $OUT/${c}_$cfg.log 2>&1
done; done
