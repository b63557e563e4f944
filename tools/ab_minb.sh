#!/bin/bash
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-mb}; mkdir -p $OUT
L=paper_1704_00693_b200/_lib
for v in libtcg libtcg_minb4 libtcg_minb6; do
  for c in c2 c4; do TCG_LIB=$PWD/$L/$v.so timeout 300 python tools/ab_modes.py $c untiled > $OUT/${c}_$v.log 2>&1; done
  TCG_LIB=$PWD/$L/$v.so AB_STEPS=5 timeout 300 python tools/ab_modes.py c3 untiled > $OUT/c3_$v.log 2>&1
  TCG_LIB=$PWD/$L/$v.so AB_STEPS=3 timeout 300 python tools/ab_modes.py c5 untiled > $OUT/c5_$v.log 2>&1
done
AB_STEPS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_untiled -s 120 -c 30 --csv --log-file $OUT/c5_launches.csv python tools/ab_modes.py c5 untiled > $OUT/ncu_c5.log 2>&1
