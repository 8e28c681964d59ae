set -x
export FF_NO_COOPERATIVE=1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --cache-control all --clock-control none --csv --log-file gpurun_out/ncu_launches_s2.csv python tests/_profile_run.py llama1b gpt67b gpt2s opt13b_m4096 > gpurun_out/prof_run.log 2>&1
python tests/_ncu_summary.py gpurun_out/ncu_launches_s2.csv llama1b,gpt67b,gpt2s,opt13b_m4096 gpurun_out/ncu_summary.json > /dev/null 2>&1
timeout 600 ncu --set full --cache-control all --clock-control none --import-source on -k regex:ff_chain_pair -s 2 -c 1 -o gpurun_out/prof_pair_llama_s2 python tests/_profile_run.py llama1b > gpurun_out/ncu_full_llama.log 2>&1
timeout 600 ncu --set full --cache-control all --clock-control none --import-source on -k regex:ff_chain_pair -s 2 -c 1 -o gpurun_out/prof_pair_gpt67b_s2 python tests/_profile_run.py gpt67b > gpurun_out/ncu_full_gpt67b.log 2>&1
unset FF_NO_COOPERATIVE
timeout 600 python bench.py > gpurun_out/bench_s2.log 2>&1
ls -la gpurun_out
