#!/bin/bash
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-cb}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest.log
AB_STEPS=5 timeout 300 python tools/ab_modes.py c3 "untiled;untiled" > $OUT/c3.log 2>&1
AB_STEPS=4 timeout 300 python tools/ab_modes.py c5 "untiled" > $OUT/c5.log 2>&1
timeout 300 python tools/ab_modes.py c2 "untiled" > $OUT/c2.log 2>&1
