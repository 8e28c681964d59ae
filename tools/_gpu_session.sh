# scratch driver (r02 session 5m): sustained power / clock, fused vs cuBLAS
set -x
O=gpurun_out/r02s5m; mkdir -p $O
timeout 300 python tools/power_probe.py gpt67b llama1b opt13b_m32768 > $O/power.log 2>&1
cat $O/power.log
