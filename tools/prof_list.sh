cap c2s 3 1 "" --config c2 --mode stream --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-untiled
