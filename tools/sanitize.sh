#!/bin/bash
# compute-sanitizer over the generated streaming kernels (mbarrier-free cp.async
# rings, one CTA barrier per step) and the untiled / periodic kernels on small
# chains: racecheck (shared-memory hazards), synccheck (barrier divergence),
# memcheck (out-of-bounds through the masks). Summaries under $OUT.
# NOTE (round 2): compute-sanitizer is closed on this GPU pool ("runs under it
# have left GPUs needing a reset"): every tool exits 86 with that message
# (profiles/r5/sanitizer.txt). The stand-ins are the reference validators on
# the CTA plans (tests/test_stream_validators.py), the device-side checked
# build (tests/test_gpu_checked.py) and bit-exact parity over shapes that
# force many CTAs, segments and sub-chain boundaries (tests/test_gpu_stream.py).
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-san}; mkdir -p $OUT
export TCG_JIT_CACHE=/tmp/tcg_jit_san
SEL='test_random_chains_2d and narrow or test_random_chains_3d and t8x8 or test_jacobi_app'
for tool in racecheck synccheck memcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_stream.py -q -x -k "$SEL" > $OUT/$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' $OUT/$tool.log | tr '\n' ' ')"
done
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_periodic.py -q -x -k "stream" > $OUT/racecheck_periodic.log 2>&1
echo "racecheck periodic rc=$? $(grep -E 'RACECHECK SUMMARY|passed|failed' $OUT/racecheck_periodic.log | tr '\n' ' ')"
