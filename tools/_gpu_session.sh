# scratch driver (r02 session 5c): serpentine unit order A/B (OPT M=4096 DRAM bytes, timelines)
set -x
O=gpurun_out/r02s5c; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_chain.py -m gpu -x -q -k "serpentine or variants" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
for v in 0x0 0x200; do
  timeout 300 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file $O/dram_opt4096_$v.csv python tools/dram_bytes.py run opt13b_m4096 fused variant=$v > /dev/null 2>&1
  python tools/dram_bytes.py parse $O/dram_opt4096_$v.csv > $O/dram_opt4096_$v.json
  cat $O/dram_opt4096_$v.json
  timeout 300 python tools/timeline.py opt opt32k variant=$v > $O/timeline_$v.log 2>&1
  grep "==" $O/timeline_$v.log
done
