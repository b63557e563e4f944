run c1 base ""
run c1 n64 "64,0,0,0,0,0,0,0"
run c1 n96 "96,0,0,0,0,0,0,0"
run c1 n192 "192,0,0,0,0,0,0,0"
run c1 n256 "256,0,0,0,0,0,0,0"
run c1 h20 "0,0,0,0,0,20,0,0"
run c1 h10 "0,0,0,0,0,10,0,0"
run c1 h7 "0,0,0,0,0,7,0,0"
run c1 n64h20 "64,0,0,0,0,20,0,0"
run c1 n64h10 "64,0,0,0,0,10,0,0"
run c1 s16 "0,0,0,0,16,0,0,0"
run c1 s6 "0,0,0,0,6,0,0,0"
run c1 rmax13 "" TCG_STREAM_RMAX2=1.3
run c1 rmax2 "" TCG_STREAM_RMAX2=2.0
run c1 ob0 "" TCG_STREAM_OWN_BUDGET=0
run c1 ob40 "" TCG_STREAM_OWN_BUDGET=40
