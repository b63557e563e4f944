#!/bin/bash
# Parity tests, bench (default + sharded path on one GPU + per-config lines),
# and the ncu launch list / full captures of the default command.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
rm -f .tcg_autotune_*
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?"
timeout 600 python bench.py --shard --steps 20 --no-cpu-baseline > gpurun_out/bench_c2_shard.json 2> gpurun_out/bench_c2_shard.err; echo "bench shard rc=$?"
for c in c1 c3 c4; do timeout 600 python bench.py --config $c --steps 20 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"; done
timeout 600 python bench.py --impl reference --steps 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-untiled > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_untiled -s 200 -c 13 -o gpurun_out/c2_untiled -f \
  python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-untiled > gpurun_out/ncu_full_u.log 2>&1; echo "ncu2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_l2tiled -s 4 -c 1 -o gpurun_out/c2_l2 -f \
  python bench.py --steps 3 --mode tiled:0,0,0 --no-cpu-baseline --no-e2e --no-untiled > gpurun_out/ncu_full_l2.log 2>&1; echo "ncu3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tiled -s 4 -c 1 -o gpurun_out/c2_tiled -f \
  python bench.py --steps 3 --mode windowed --no-cpu-baseline --no-e2e --no-untiled > gpurun_out/ncu_full_t.log 2>&1; echo "ncu4 rc=$?"
