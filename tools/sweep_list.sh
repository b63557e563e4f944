run c3 s4 ""
run c3 s6 "0,0,0,0,6,0,0,0"
run c3 s8 "0,0,0,0,8,0,0,0"
run c3 s5 "0,0,0,0,5,0,0,0"
run c3 la2 "" TCG_STREAM_LOOKAHEAD=2
run c3 ob "" TCG_STREAM_FAST3=0
