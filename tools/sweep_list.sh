run c1 base ""
run c1 h20 "0,0,0,0,0,20,0,0"
run c1 h10 "0,0,0,0,0,10,0,0"
run c1 h7 "0,0,0,0,0,7,0,0"
run c1 n96 "96,0,0,0,0,0,0,0"
run c1 n96h10 "96,0,0,0,0,10,0,0"
run c1 rmax13 "" TCG_STREAM_RMAX2=1.3
