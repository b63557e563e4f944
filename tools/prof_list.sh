cap c2s 4 1 "" --config c2 --mode stream --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-untiled
cap c3s 4 1 "" --config c3 --mode stream --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-untiled
cap c5h 8 1 "" --config c5 --mode stream --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-untiled
cap c1s 6 2 "" --config c1 --mode stream --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-untiled
