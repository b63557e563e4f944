#!/bin/bash
# ncu --set full of generated streaming kernels (one config per capture).
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-ps}; mkdir -p $OUT
export TCG_JIT_CACHE=/tmp/tcg_jit
cap() {  # name skip count env... -- bench args
  local name=$1 s=$2 c=$3 cfg=$4; shift 4
  TCG_STREAM_CFG="$cfg" timeout 900 ncu --set full --clock-control none --import-source on -k regex:tcg_stream -s $s -c $c -o /tmp/$name -f \
    python bench.py "$@" > $OUT/ncu_$name.log 2>&1; echo "ncu $name rc=$?"
  python tools/ncu_summary.py /tmp/$name.ncu-rep > $OUT/$name.md 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > $OUT/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page details --csv > $OUT/${name}_details.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/${name}_src.csv 2>/dev/null
  gzip -c /tmp/${name}_src.csv > $OUT/${name}_src.csv.gz
}
source ${PROF:-tools/prof_list.sh}
