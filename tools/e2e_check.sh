#!/bin/bash
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-e2e}; mkdir -p $OUT
for c in c2 c4 c1 c3; do timeout 600 python bench.py --config $c --steps 20 --no-cpu-baseline --no-untiled > $OUT/bench_$c.json 2> $OUT/bench_$c.err; done
