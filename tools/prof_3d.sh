#!/bin/bash
# ncu captures of the 3D configs' dominant untiled kernels + c1/c4 launch lists.
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-p3d}; mkdir -p $OUT
cap() {  # name kernel-regex skip count cmd...
  local name=$1 k=$2 s=$3 c=$4; shift 4
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c $c -o /tmp/$name -f "$@" > $OUT/ncu_$name.log 2>&1; echo "ncu $name rc=$?"
  python tools/ncu_summary.py /tmp/$name.ncu-rep > $OUT/$name.md 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > $OUT/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page details --csv > $OUT/${name}_details.csv 2>/dev/null
}
AB_STEPS=2 cap c3_untiled "k_untiled" 40 2 python tools/ab_modes.py c3 untiled
AB_STEPS=1 cap c5_untiled "k_untiled" 140 7 python tools/ab_modes.py c5 untiled
for c in c1 c4; do timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_ --csv --log-file $OUT/launches_$c.csv python tools/ab_modes.py $c untiled > /dev/null 2>&1; done
