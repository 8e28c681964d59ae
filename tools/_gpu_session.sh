# scratch driver (r02 session 5zx): validation of the split producer
set -x
O=gpurun_out/r02s5zx; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -1 $O/gpu_tests.log
for seed in 51 52; do FF_CHAIN_LIB=paper_2512_12949_b200/libff_diag.so timeout 900 python tools/fuzz_chain.py $seed 60 > $O/fuzz_$seed.log 2>&1; echo "fuzz $seed rc=$?"; grep "EXPIRED\|FAIL\|ERROR\|fuzz:" $O/fuzz_$seed.log | head -5; done
FF_CHAIN_LIB=paper_2512_12949_b200/libff_diag.so timeout 900 python tools/repro_multi.py iters=2 cases=0,1,2,3,4,5,6,7,8,9 > $O/diag_seq.log 2>&1; echo "diag seq rc=$?"; grep -c expired $O/diag_seq.log
timeout 600 compute-sanitizer --tool synccheck python tools/sanitize.py > $O/synccheck.log 2>&1; echo "synccheck rc=$?"; grep "ERROR SUMMARY\|failures" $O/synccheck.log
timeout 600 compute-sanitizer --tool memcheck python tools/tail_debug.py 11 > $O/memcheck_tail.log 2>&1; echo "memcheck rc=$?"; grep "ERROR SUMMARY" $O/memcheck_tail.log; grep "max err" $O/memcheck_tail.log
