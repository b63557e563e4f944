#!/bin/bash
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-ch}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest.log
timeout 300 python tools/host_cost.py > $OUT/host.log 2>&1
for c in c1 c2 c4; do timeout 300 python tools/ab_modes.py $c "untiled;untiled" > $OUT/$c.log 2>&1; done
