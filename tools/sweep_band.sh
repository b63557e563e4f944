#!/bin/bash
# Untiled 3D block rasterisation band (TCG_UNTILED_BAND) on c3 / c5.
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-band}; mkdir -p $OUT
export TCG_JIT_CACHE=/tmp/tcg_jit
for c in c5 c3; do
  for b in 0 4 8 16 32 64; do
    TCG_UNTILED_BAND=$b timeout 600 python bench.py --config $c --mode untiled --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e --no-untiled > $OUT/${c}_band$b.json 2> $OUT/${c}_band$b.err
    python - $OUT/${c}_band$b.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"{sys.argv[1].split('/')[-1]:24s} ms/step={d['ms_per_step']:.4f} frac={d['roofline'].get('frac'):.3f}")
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
  done
done
