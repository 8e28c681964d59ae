# scratch driver (r02 session 7): GPT-2s cold vs warm phases
O=gpurun_out/r02s7; mkdir -p $O
timeout 300 python tools/timeline.py gpt2s x0 counters > $O/timeline_gpt2s_coldwarm.log 2>&1
timeout 300 python tools/timeline.py gpt2s x0 counters warm >> $O/timeline_gpt2s_coldwarm.log 2>&1
timeout 300 python tools/timeline.py gpt2s x0 counters variant=0x1 >> $O/timeline_gpt2s_coldwarm.log 2>&1
cat $O/timeline_gpt2s_coldwarm.log
