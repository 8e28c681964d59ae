# scratch driver (r02 session 6m): tail split for gated chains
set -x
O=gpurun_out/r02s6m; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_chain.py -m gpu -x -q -k "tail_split" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -15 $O/tests.log
