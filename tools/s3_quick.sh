#!/bin/bash
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-s3q}; mkdir -p $OUT
timeout 120 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "Jacobi3DC3 or ns_c5 or random_chains_match" > $OUT/pytest_q.log 2>&1; echo "pytest_q rc=$?" | tee -a $OUT/pytest_q.log
[ "$(tail -1 $OUT/pytest_q.log)" == "pytest_q rc=0" ] || exit 1
timeout 600 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest.log
for d in 1 2 4 6; do
  TCG_S3_D=$d AB_STEPS=5 timeout 120 python tools/ab_modes.py c3 untiled > $OUT/c3_d$d.log 2>&1
  TCG_S3_D=$d AB_STEPS=3 timeout 200 python tools/ab_modes.py c5 untiled > $OUT/c5_d$d.log 2>&1
done
TCG_STAGED3=0 AB_STEPS=5 timeout 120 python tools/ab_modes.py c3 untiled > $OUT/c3_s0.log 2>&1
