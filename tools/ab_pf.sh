#!/bin/bash
# A/B: L2 bulk prefetch of the untiled block footprint; GPU parity tests.
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-pf}; mkdir -p $OUT
for c in c2 c3 c4 c1; do
  for pf in 0 1; do TCG_PREFETCH_L2=$pf timeout 300 python tools/ab_modes.py $c "untiled" > $OUT/${c}_pf$pf.log 2>&1; done
done
for pf in 0 1; do TCG_PREFETCH_L2=$pf AB_STEPS=6 timeout 600 python tools/ab_modes.py c5 "untiled" > $OUT/c5_pf$pf.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest.log
