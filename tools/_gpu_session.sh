# scratch driver for one gpurun session (r02)
set -x
O=gpurun_out/r02; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > $O/gpu_tests_3.log
python -c "import os; print(sorted((k, v[:80]) for k, v in os.environ.items() if any(s in k for s in ('INJECT','NSIGHT','PROFILER','PRELOAD'))))" > $O/env_noncu.log 2>&1
for v in 0 0x10 0x20 0x30; do timeout 300 python tools/timeline.py gpt67b llama opt variant=$v > $O/timeline_3_v$v.log 2>&1; done
for w in gpt67b llama1b opt13b_m4096; do for impl in fused cublas_eager cublas_fused_epilogue; do
  timeout 300 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file $O/dram_${w}_${impl}.csv python tools/dram_bytes.py run $w $impl > $O/dram_${w}_${impl}.log 2>&1
  python tools/dram_bytes.py parse $O/dram_${w}_${impl}.csv > $O/dram_${w}_${impl}.json 2>>$O/dram_${w}_${impl}.log
done; done
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_3.json 2> $O/bench_3.err
tail -3 $O/gpu_tests_3.log; cat $O/dram_*.json; grep events $O/timeline_3_*.log
