# session 5: launch list (4 workloads, fused vs cuBLAS), full captures of the current kernels, final bench line
set -x
export FF_NO_COOPERATIVE=1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --cache-control all --clock-control none --csv --log-file gpurun_out/ncu_launches_s5b.csv python tests/_profile_run.py llama1b gpt67b gpt2s opt13b_m4096 > gpurun_out/prof_run_s5.log 2>&1
python tests/_ncu_summary.py gpurun_out/ncu_launches_s5b.csv llama1b,gpt67b,gpt2s,opt13b_m4096 gpurun_out/ncu_summary.json > gpurun_out/ncu_summary_s5.log 2>&1
timeout 600 ncu --set full --cache-control all --clock-control none --import-source on -k regex:ff_chain_pair -s 2 -c 1 -o gpurun_out/prof_pair_llama_s5b python tests/_profile_run.py llama1b > gpurun_out/ncu_full_llama_s5.log 2>&1
timeout 600 ncu --set full --cache-control all --clock-control none --import-source on -k regex:ff_chain_pair -s 2 -c 1 -o gpurun_out/prof_pair_gpt67b_s5b python tests/_profile_run.py gpt67b > gpurun_out/ncu_full_gpt67b_s5.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu_bench_launches_s5b.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-extra --no-profile-plans > gpurun_out/ncu_bench_stdout_s5.log 2>&1
unset FF_NO_COOPERATIVE
timeout 900 python bench.py > gpurun_out/bench_session5b.log 2>&1
tail -1 gpurun_out/bench_session5b.log > gpurun_out/bench_session5b.json
ls -la gpurun_out
