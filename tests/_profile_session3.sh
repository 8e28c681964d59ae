# ncu launch list of the bench command itself (launch from the dispatch table, no candidate profiling)
export FF_NO_COOPERATIVE=1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu_bench_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-extra --no-profile-plans > gpurun_out/ncu_bench_stdout.log 2>&1
ls -la gpurun_out | tail -3
