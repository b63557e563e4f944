#!/bin/bash
# GPU parity suite + default stream/untiled/auto bench lines per config.
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-gc}; mkdir -p $OUT
export TCG_JIT_CACHE=/tmp/tcg_jit
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q ${PYTEST_ARGS} > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest_gpu.log
for c in ${CONFIGS:-c2 c3 c1}; do
  for m in ${MODES:-stream untiled auto}; do
    timeout 400 python bench.py --config $c --mode $m --steps ${STEPS:-20} --warmup 10 --no-cpu-baseline --no-e2e --no-untiled > $OUT/bench_${c}_$m.json 2> $OUT/bench_${c}_$m.err
    python - $OUT/bench_${c}_$m.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); p=d['detail']['plan']
    print(f"{sys.argv[1].split('/')[-1]:28s} ms/step={d['ms_per_step']:.4f} exec={p['executor']} ctas={p['ctas']} sub={p['subchains']} frac={d['roofline'].get('frac')}")
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
  done
done
