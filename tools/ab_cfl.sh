#!/bin/bash
# GPU parity suite + default bench + launch list after the CFL two-pass change.
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/${TAG:-cfl}
mkdir -p $OUT
rm -f .tcg_autotune_*
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.log
timeout 300 python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_untiled -c 400 --csv --log-file $OUT/launches_c2.csv \
  python bench.py --steps 5 --mode untiled --no-cpu-baseline --no-e2e --no-untiled > $OUT/ncu_launch.log 2>&1; echo "ncu rc=$?"
