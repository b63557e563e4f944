#!/bin/bash
# Graph replay A/B + windowed sub-chain length sweep.
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-sw}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest.log
for c in c1 c2 c4; do
  TCG_GRAPHS=0 timeout 300 python tools/ab_modes.py $c "untiled" > $OUT/nograph_$c.log 2>&1
  timeout 300 python tools/ab_modes.py $c "untiled;auto" > $OUT/graph_$c.log 2>&1
done
for n in 2 3 4 6; do TCG_WIN_MAXLOOPS=$n timeout 300 python tools/ab_modes.py c2 "windowed;windowed:128,16;windowed:256,8" > $OUT/win_ml$n.log 2>&1; done
for n in 2 4; do TCG_WIN_MAXLOOPS=$n timeout 300 python tools/ab_modes.py c3 "windowed" > $OUT/c3_win_ml$n.log 2>&1; done
timeout 300 python tools/ab_modes.py c3 "untiled" > $OUT/c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_untiled -s 20 -c 1 -o /tmp/c3u -f python tools/ab_modes.py c3 untiled > $OUT/ncu_c3.log 2>&1
ncu -i /tmp/c3u.ncu-rep --page details --csv > $OUT/c3_untiled_details.csv 2>/dev/null
ncu -i /tmp/c3u.ncu-rep --page raw --csv > $OUT/c3_untiled_raw.csv 2>/dev/null
python tools/ncu_summary.py /tmp/c3u.ncu-rep > $OUT/c3_untiled.md 2>&1
