# default-sizer stream kernels: c2 whole step, c3 first 3-loop kernel
cap c2s 3 1 "" --config c2 --mode stream --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-untiled
cap c3s 18 1 "" --config c3 --mode stream --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-untiled
