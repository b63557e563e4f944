# cfg: nt,bx,by,ntx,segments,max_loops,minb,prefetch
run c3 base ""
run c3 ns1 "" TCG_STREAM_NSYNC=1
run c3 ns1la2 "" TCG_STREAM_NSYNC=1 TCG_STREAM_LOOKAHEAD=2
run c3 ns1la4 "" TCG_STREAM_NSYNC=1 TCG_STREAM_LOOKAHEAD=4
run c3 ns1by4 "256,1,4,32,0,3,0,0" TCG_STREAM_NSYNC=1
run c3 ns1h4 "0,0,0,0,0,4,0,0" TCG_STREAM_NSYNC=1 TCG_STREAM_RMAX3=3
run c3 ns1f1 "" TCG_STREAM_NSYNC=1 TCG_STREAM_FAST=1
run c2 base ""
run c2 ns1 "" TCG_STREAM_NSYNC=1
run c2 ns1n256 "256,0,0,0,0,0,0,0" TCG_STREAM_NSYNC=1
run c2 ns1n192 "192,0,0,0,0,0,0,0" TCG_STREAM_NSYNC=1
run c1 base ""
run c1 ns1 "" TCG_STREAM_NSYNC=1
run c5 base ""
run c5 ns1 "" TCG_STREAM_NSYNC=1
