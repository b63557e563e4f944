#!/bin/bash
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-u2}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest.log
for c in c2 c4 c1; do timeout 300 python tools/ab_modes.py $c "untiled;untiled" > $OUT/$c.log 2>&1; done
AB_STEPS=5 timeout 300 python tools/ab_modes.py c3 "untiled" > $OUT/c3.log 2>&1
