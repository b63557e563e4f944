#!/bin/bash
# Stream-executor GPU check: parity tests, then per-config stream vs untiled.
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-st}; mkdir -p $OUT
export TCG_JIT_CACHE=/tmp/tcg_jit
timeout 900 python -m pytest tests/test_gpu_stream.py -q -x ${PYTEST_K:+-k "$PYTEST_K"} > $OUT/pytest_stream.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest_stream.log
for c in ${CONFIGS:-c2 c3 c1}; do
  for m in stream untiled; do
    timeout 300 python bench.py --config $c --mode $m --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e --no-untiled > $OUT/bench_${c}_$m.json 2> $OUT/bench_${c}_$m.err; echo "bench $c $m rc=$?"
  done
done
