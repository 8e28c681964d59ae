# scratch driver (r02 session 7): new GPU tests (reproducible table, CLI --deterministic)
O=gpurun_out/r02s7; mkdir -p $O
timeout 900 python -m pytest tests/test_dispatch.py tests/test_cli.py -m gpu -q > $O/gpu_tests_new.log 2>&1; echo "rc=$?"; tail -3 $O/gpu_tests_new.log
