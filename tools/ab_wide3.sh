#!/bin/bash
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-w3}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest.log
for v in 0 1; do TCG_WIDE3=$v AB_STEPS=3 timeout 300 python tools/ab_modes.py c5 untiled > $OUT/c5_w$v.log 2>&1; done
AB_STEPS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_untiled -s 120 -c 8 --csv --log-file $OUT/c5_launches.csv python tools/ab_modes.py c5 untiled > $OUT/ncu_c5.log 2>&1
