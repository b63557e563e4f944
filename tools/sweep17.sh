timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest17.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest17.log
for c in "c2 untiled" "c1 untiled" "c3 untiled - 2" "c4 untiled - 20"; do timeout 300 python tools/run_cfg.py $c >> gpurun_out/time17.log 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_untiled -c 13 --csv --log-file gpurun_out/untiled17.csv python tools/run_cfg.py c2 untiled - 1 > gpurun_out/ncu17.log 2>&1
