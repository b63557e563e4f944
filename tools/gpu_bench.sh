#!/bin/bash
# Parity tests, bench (default + sharded path on one GPU + per-config lines),
# and the ncu launch list / full captures of the default command. ncu reports
# are exported to CSV on the box (gpurun copies back at most 64 MiB).
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/${TAG:-r}
mkdir -p $OUT
rm -f .tcg_autotune_*
if [ -z "$SKIP_TESTS" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest_gpu.log
fi
timeout 600 python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err; echo "bench rc=$?"
if [ -z "$ONLY_C2" ]; then
  timeout 600 python bench.py --shard --steps 20 --no-cpu-baseline > $OUT/bench_c2_shard.json 2> $OUT/bench_c2_shard.err; echo "bench shard rc=$?"
  for c in c1 c3 c4 c5; do timeout 600 python bench.py --config $c --steps 20 --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "bench $c rc=$?"; done
  timeout 600 python bench.py --impl reference --steps 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"
fi
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_c2.csv \
  python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-untiled > $OUT/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
cap() {  # name kernel-regex skip count bench-args...
  local name=$1 k=$2 s=$3 c=$4; shift 4
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c $c -o /tmp/$name -f \
    python bench.py "$@" > $OUT/ncu_$name.log 2>&1; echo "ncu $name rc=$?"
  python tools/ncu_summary.py /tmp/$name.ncu-rep > $OUT/$name.md 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > $OUT/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page details --csv > $OUT/${name}_details.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/${name}_src.csv 2>/dev/null
  gzip -c /tmp/${name}_src.csv > $OUT/${name}_src.csv.gz
  sz=$(stat -c %s /tmp/$name.ncu-rep 2>/dev/null || echo 0)
  [ "$sz" -lt 12000000 ] && cp /tmp/$name.ncu-rep $OUT/
}
cap c2_untiled k_untiled 200 13 --steps 5 --mode untiled --no-cpu-baseline --no-e2e --no-untiled
cap c2_l2 k_l2tiled 4 1 --steps 3 --mode tiled:0,0,0 --no-cpu-baseline --no-e2e --no-untiled
if [ -z "$ONLY_C2" ]; then
  cap c2_win k_tiled 4 1 --steps 3 --mode windowed --no-cpu-baseline --no-e2e --no-untiled
fi
du -sh $OUT
