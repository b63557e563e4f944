#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "tiled or auto or dist" > gpurun_out/pytest_df.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_df.log
for c in c2 c3 c1 c4; do
  python tools/ab_modes.py $c untiled 2>&1 | tail -1
  TCG_L2_DATAFLOW=0 python tools/ab_modes.py $c "tiled:0,0,0" 2>&1 | tail -1
  TCG_L2_DATAFLOW=1 python tools/ab_modes.py $c "tiled:0,0,0" 2>&1 | tail -1
done > gpurun_out/df.log 2>&1
