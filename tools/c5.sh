#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "ns_c5" > gpurun_out/pytest_c5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c5.log
timeout 1200 python bench.py --config c5 --steps 5 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?"
