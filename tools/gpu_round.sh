#!/bin/bash
# One GPU session: parity tests, default bench, per-config benches, ncu.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?"
for c in c1 c4; do timeout 300 python bench.py --config $c --steps 20 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-untiled > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_untiled -s 60 -c 14 -o gpurun_out/c2_untiled -f \
  python bench.py --steps 5 --warmup 3 --mode untiled --no-cpu-baseline --no-e2e --no-untiled > gpurun_out/ncu_full_u.log 2>&1; echo "ncu2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tiled -s 4 -c 2 -o gpurun_out/c2_tiled -f \
  python bench.py --steps 5 --warmup 3 --mode windowed --no-cpu-baseline --no-e2e --no-untiled > gpurun_out/ncu_full_t.log 2>&1; echo "ncu3 rc=$?"
