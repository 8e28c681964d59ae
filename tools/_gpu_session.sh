# scratch driver (r02 session 6h): prefetch rule check + GPU suite
set -x
O=gpurun_out/r02s6h; mkdir -p $O
for i in 1 2; do timeout 300 python tools/timeline.py gpt67b llama opt opt32k > $O/t_$i.log 2>&1; grep "==" $O/t_$i.log | sed 's/{.*}//'; done
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -1 $O/gpu_tests.log
