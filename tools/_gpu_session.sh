# scratch driver (r02 session 5zt): tests after producer trims
set -x
O=gpurun_out/r02s5zt; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -1 $O/gpu_tests.log
timeout 900 python tools/fuzz_chain.py 41 60 > $O/fuzz.log 2>&1; tail -1 $O/fuzz.log
