#!/bin/bash
# Sweep streaming-executor shapes per config (bench --mode stream), parity tests first.
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-sw}; mkdir -p $OUT
export TCG_JIT_CACHE=/tmp/tcg_jit
if [ -z "$SKIP_TESTS" ]; then
timeout 900 python -m pytest tests/test_gpu_stream.py -q -x ${PYTEST_K:+-k "$PYTEST_K"} > $OUT/pytest_stream.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest_stream.log
fi
run() { # config tag cfg [env...]
  local c=$1 tag=$2 cfg=$3; shift 3
  env TCG_STREAM_CFG="$cfg" "$@" timeout 300 python bench.py --config $c --mode stream --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e --no-untiled > $OUT/${c}_$tag.json 2> $OUT/${c}_$tag.err
  python - $OUT/${c}_$tag.json "$cfg" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); p=d['detail']['plan']
    print(f"{sys.argv[1].split('/')[-1]:28s} cfg={sys.argv[2]:24s} ms/step={d['ms_per_step']:.4f} ctas={p['ctas']} sub={p['subchains']} tile={p['tile_sizes']} frac={d['roofline'].get('frac')}")
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
}
source ${SWEEP:-tools/sweep_list.sh}
