#!/bin/bash
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-p5}; mkdir -p $OUT
AB_STEPS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_untiled -s 120 -c 8 --csv --log-file $OUT/c5_launches.csv python tools/ab_modes.py c5 untiled > $OUT/ncu_c5.log 2>&1
AB_STEPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_untiledILi3ELi502" -s 6 -c 1 -o /tmp/c5r -f python tools/ab_modes.py c5 untiled > $OUT/ncu_c5full.log 2>&1
ncu -i /tmp/c5r.ncu-rep --page raw --csv > $OUT/c5r_raw.csv 2>/dev/null
ncu -i /tmp/c5r.ncu-rep --page details --csv > $OUT/c5r_details.csv 2>/dev/null
python tools/ncu_summary.py /tmp/c5r.ncu-rep > $OUT/c5r.md 2>&1
