#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
bash tools/ab_l2.sh
timeout 900 ncu --set full --clock-control none -k regex:k_untiled -s 40 -c 2 -o gpurun_out/c3_untiled -f \
  python tools/ab_modes.py c3 untiled > gpurun_out/ncu_c3u.log 2>&1; echo "ncu rc=$?"
