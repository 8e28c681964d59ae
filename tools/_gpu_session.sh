# scratch driver (r02 session 7): conv block phase stamps
O=gpurun_out/r02s7; mkdir -p $O
timeout 300 python tools/timeline.py conv_1x1_3x3 conv_c5 x1 counters > $O/timeline_conv_stamps.log 2>&1; echo "rc=$?"
timeout 300 python tools/timeline.py conv_1x1_3x3 x1 counters warm >> $O/timeline_conv_stamps.log 2>&1; echo "rc=$?"
cat $O/timeline_conv_stamps.log
