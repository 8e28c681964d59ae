# scratch driver (r02 session 5zb): GPU fuzz with the diagnostic-watchdog build (expired waits reported)
set -x
O=gpurun_out/r02s5zb; mkdir -p $O
for seed in 11 12 13; do FF_CHAIN_LIB=paper_2512_12949_b200/libff_diag.so timeout 900 python tools/fuzz_chain.py $seed 60 > $O/fuzz_$seed.log 2>&1; echo "fuzz $seed rc=$?"; grep "EXPIRED\|FAIL\|ERROR\|fuzz:" $O/fuzz_$seed.log | head -8; done
