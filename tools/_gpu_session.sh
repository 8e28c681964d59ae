# scratch driver for one gpurun session (r02, session 4): state check
set -x
O=gpurun_out/r02s4; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -40 > $O/gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
tail -3 $O/gpu_tests.log; tail -3 $O/smoke.log; head -c 3000 $O/bench.json
