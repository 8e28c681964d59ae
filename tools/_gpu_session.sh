# scratch driver for one gpurun session (r02, session 4d): l2dsm transport, discard variants, dispatch tables
set -x
O=gpurun_out/r02s4d; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > $O/gpu_tests.log
timeout 300 python tools/timeline.py gpt2s x0 > $O/timeline_gpt2s_x0.log 2>&1
timeout 300 python tools/timeline.py gpt2s x3 > $O/timeline_gpt2s_x3.log 2>&1
timeout 300 python tools/timeline.py gpt2s llama gpt67b x3 > $O/timeline_x3.log 2>&1
for v in 0 0x100 0x80; do timeout 300 python tools/timeline.py gpt67b llama opt variant=$v > $O/timeline_v$v.log 2>&1; done
for w in gpt67b llama1b; do for v in 0 0x100; do
  timeout 300 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file $O/dram_${w}_v$v.csv python tools/dram_bytes.py run $w fused variant=$v > $O/dram_${w}_v$v.log 2>&1
  python tools/dram_bytes.py parse $O/dram_${w}_v$v.csv > $O/dram_${w}_v$v.json 2>>$O/dram_${w}_v$v.log
done; done
timeout 300 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize.py > $O/sanitizer_racecheck.log 2>&1
timeout 900 python -m paper_2512_12949_b200.dispatch > $O/dispatch_build.log 2>&1
mkdir -p $O/dispatch; cp paper_2512_12949_b200/plans/dispatch/*.json $O/dispatch/
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
cat $O/gpu_tests.log | tail -8; grep -h "SUMMARY\|failures" $O/sanitizer_*.log; for f in $O/dram_*.json; do echo $f; grep -o '"dram_total.*' $f; done; grep -h "events\|E_start\|exit" $O/timeline_*.log; cat $O/dispatch_build.log
