# scratch driver (r02 session 4i): A/B builds -- cost of the flag polls and of the weight L2 prefetches
set -x
O=gpurun_out/r02s4i; mkdir -p $O
for lib in libff_chain libff_ab_noflag libff_ab_nopf; do
  export FF_CHAIN_LIB=paper_2512_12949_b200/$lib.so
  timeout 300 python tools/timeline.py gpt67b llama opt opt32k hopsonly counters > $O/timeline_$lib.log 2>&1
done
grep -h "events\|mma_total\|w_full\|prod_w_flag" $O/timeline_*.log
