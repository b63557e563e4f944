#!/bin/bash
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-s3}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest.log
for v in 0 1; do
  TCG_STAGED3=$v AB_STEPS=5 timeout 300 python tools/ab_modes.py c3 untiled > $OUT/c3_s$v.log 2>&1
  TCG_STAGED3=$v AB_STEPS=3 timeout 300 python tools/ab_modes.py c5 untiled > $OUT/c5_s$v.log 2>&1
done
for zr in 32 128; do :; done
for d in 2 6; do
  TCG_S3_D=$d AB_STEPS=5 timeout 300 python tools/ab_modes.py c3 untiled > $OUT/c3_d$d.log 2>&1
  TCG_S3_D=$d AB_STEPS=3 timeout 300 python tools/ab_modes.py c5 untiled > $OUT/c5_d$d.log 2>&1
done
AB_STEPS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_untiled -s 120 -c 12 --csv --log-file $OUT/c5_launches.csv python tools/ab_modes.py c5 untiled > $OUT/ncu_c5.log 2>&1
