# scratch driver for one gpurun session (r02, session 4c): discard, L2 policies for OPT, dispatch tables
set -x
O=gpurun_out/r02s4c; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > $O/gpu_tests.log
for tool in racecheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize.py > $O/sanitizer_$tool.log 2>&1
  echo "rc=$?" >> $O/sanitizer_$tool.log
done
for w in gpt67b llama1b opt13b_m4096; do for v in 0 0x80 0x40 0xC0; do
  timeout 300 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file $O/dram_${w}_v$v.csv python tools/dram_bytes.py run $w fused variant=$v > $O/dram_${w}_v$v.log 2>&1
  python tools/dram_bytes.py parse $O/dram_${w}_v$v.csv > $O/dram_${w}_v$v.json 2>>$O/dram_${w}_v$v.log
done; done
for v in 0 0x80 0x40; do timeout 300 python tools/timeline.py gpt67b llama opt variant=$v > $O/timeline_v$v.log 2>&1; done
timeout 900 python -m paper_2512_12949_b200.dispatch > $O/dispatch_build.log 2>&1
mkdir -p $O/dispatch; cp paper_2512_12949_b200/plans/dispatch/*.json $O/dispatch/
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
cat $O/gpu_tests.log; grep -h "SUMMARY\|failures" $O/sanitizer_*.log; for f in $O/dram_*.json; do echo $f; cut -c1-400 $f | grep -o '"dram_total.*'; done; grep events $O/timeline_*.log; cat $O/dispatch_build.log
