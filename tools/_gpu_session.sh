# scratch driver for one gpurun session (r02, session 4f): BK=64 x 6 stages vs BK=128 x 3 stages (pair kernel)
set -x
O=gpurun_out/r02s4f; mkdir -p $O
export B64=paper_2512_12949_b200/libff_chain_bk64.so
FF_CHAIN_LIB=$B64 timeout 900 python -m pytest tests/test_gpu_chain.py -x -q -k "pair or Pair or quad" 2>&1 | tail -5 > $O/gpu_tests_bk64.log
for lib in default bk64; do
  if [ $lib = bk64 ]; then export FF_CHAIN_LIB=$B64; else unset FF_CHAIN_LIB; fi
  timeout 300 python tools/timeline.py gpt67b llama opt opt32k counters > $O/timeline_$lib.log 2>&1
  timeout 300 python tools/timeline.py gpt67b llama opt opt32k counters > $O/timeline_${lib}_2.log 2>&1
done
unset FF_CHAIN_LIB
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum
FF_CHAIN_LIB=$B64 timeout 600 ncu --cache-control none --clock-control none --metrics $M --csv --log-file $O/ncu_opt32k_bk64.csv python tools/dram_bytes.py run opt13b_m32768 fused > $O/ncu_opt32k_bk64.log 2>&1
cat $O/gpu_tests_bk64.log; grep -h "events" $O/timeline_*.log
