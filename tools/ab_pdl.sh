#!/bin/bash
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-pdl}; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest.log
for v in 0 1 0 1; do
  for c in c1 c2 c4; do TCG_PDL=$v timeout 300 python tools/ab_modes.py $c untiled >> $OUT/${c}_pdl$v.log 2>&1; done
done
for v in 0 1; do TCG_PDL=$v AB_STEPS=5 timeout 300 python tools/ab_modes.py c3 untiled >> $OUT/c3_pdl$v.log 2>&1; done
