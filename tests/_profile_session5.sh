# session 5: full default bench line + ncu launch list of the bench command
set -x
timeout 900 python bench.py > gpurun_out/bench_session5.log 2>&1
tail -1 gpurun_out/bench_session5.log > gpurun_out/bench_session5.json
export FF_NO_COOPERATIVE=1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu_bench_launches_s5.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-extra --no-profile-plans > gpurun_out/ncu_bench_stdout_s5.log 2>&1
ls -la gpurun_out | tail -5
