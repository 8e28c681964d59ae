# scratch driver (r02 session 7): deterministic-mode tests (bf16 + fp16)
O=gpurun_out/r02s7; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_chain.py -m gpu -q -k deterministic > $O/gpu_det2.log 2>&1; echo "rc=$?"; tail -3 $O/gpu_det2.log
