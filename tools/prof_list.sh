export TCG_STREAM_TMA=0 TCG_STREAM_REG_LEAD=2
cap c2w 3 1 "128,1,0,0,0,13,0,0" --config c2 --mode stream --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-untiled
cap c3w 6 1 "256,1,4,32,0,3,0,0" --config c3 --mode stream --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-untiled
