#!/bin/bash
# Round-2 final capture: GPU suite, smoke, bench lines (default + per config), reference arm,
# ncu launch list of the default command, ncu --set full of the generated c2 / c3 kernels.
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-final}; mkdir -p $OUT
export TCG_JIT_CACHE=/tmp/tcg_jit
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$? $(tail -1 $OUT/pytest_gpu.txt)"
timeout 600 python __graft_entry__.py smoke > $OUT/smoke.txt 2>&1; echo "smoke rc=$? $(tail -1 $OUT/smoke.txt)"
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; echo "bench default rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "bench ref rc=$?"
for c in c1 c3 c4; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-50} --warmup 3 --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "bench $c rc=$?"
done
timeout 1500 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench c5 rc=$?"
timeout 900 python bench.py --config c2 --host python --steps 100 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c2_pyhost.json 2> $OUT/bench_c2_pyhost.err; echo "bench c2 python-host rc=$?"
python - $OUT <<'PY'
import json,sys,glob
for f in sorted(glob.glob(sys.argv[1]+'/bench_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        if d.get('impl')=='reference': print(f.split('/')[-1], 'reference', d['value']); continue
        t=d['detail']
        print(f"{f.split('/')[-1]:26s} value={d['value']:.4g} ms/step={d['ms_per_step']:.4f} exec={t['plan']['executor']} untiled={t['untiled_value'] and round(t['untiled_value']/1e9,1)} stream={t['tiled_value'] and round(t['tiled_value']/1e9,1)} ratio={t['tiled_vs_untiled'] and round(t['tiled_vs_untiled'],3)} e2e={d['e2e'] and d['e2e'].get('value')} frac={d['roofline']['frac'] and round(d['roofline']['frac'],3)}")
    except Exception as e: print(f, 'ERR', e)
PY
# launch list of the default command (after it exited 0 without ncu)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_default.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-untiled > $OUT/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
TAG=${TAG:-final} bash tools/prof_stream.sh
