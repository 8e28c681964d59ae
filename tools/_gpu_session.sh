# scratch driver (r02 session 5zn): next-step flag prefetch A/B
set -x
O=gpurun_out/r02s5zp; mkdir -p $O
for i in 1 2; do for lib in libff_nopf libff_chain; do
  FF_CHAIN_LIB=paper_2512_12949_b200/$lib.so timeout 300 python tools/timeline.py gpt67b llama opt opt32k counters > $O/t_${lib}_$i.log 2>&1; echo "## $lib"; grep "==\|prod_w_flag" $O/t_${lib}_$i.log | sed 's/{.*}//'
done; done
timeout 900 python -m pytest tests/test_gpu_chain.py -m gpu -x -q > $O/tests.log 2>&1; echo "tests rc=$?"; tail -1 $O/tests.log
