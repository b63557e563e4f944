#!/bin/bash
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-p}; mkdir -p $OUT
cap() {  # name kernel-regex skip count cmd...
  local name=$1 k=$2 s=$3 c=$4; shift 4
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c $c -o /tmp/$name -f "$@" > $OUT/ncu_$name.log 2>&1; echo "ncu $name rc=$?"
  python tools/ncu_summary.py /tmp/$name.ncu-rep > $OUT/$name.md 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > $OUT/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page details --csv > $OUT/${name}_details.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${name}_src.csv 2>/dev/null; gzip -c /tmp/${name}_src.csv > $OUT/${name}_src.csv.gz
}
AB_STEPS=5 cap c1_l2 k_l2tiled 5 1 python tools/ab_modes.py c1 "tiled:0,0,0"
AB_STEPS=5 cap c1_win k_tiled 5 1 python tools/ab_modes.py c1 "windowed"
AB_STEPS=2 cap c3_u k_untiled 40 1 python tools/ab_modes.py c3 "untiled"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/c1_launches.csv python tools/ab_modes.py c1 untiled > /dev/null 2>&1
