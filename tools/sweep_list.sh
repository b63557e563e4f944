run c4 hc ""
run c4 hc4k "" TCG_STREAM_HRED_CTAS=4096
run c4 hc1k "" TCG_STREAM_HRED_CTAS=1184
run c4 h0 "" TCG_STREAM_HORIZ=0
run c5 hc ""
run c5 hc4k "" TCG_STREAM_HRED_CTAS=4096
