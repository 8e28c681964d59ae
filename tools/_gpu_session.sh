# scratch driver (r02 session 6j): prefetch distance A/B
set -x
O=gpurun_out/r02s6j; mkdir -p $O
for i in 1 2; do for lib in libff_chain libff_pf1 libff_pf3 libff_pf4; do
  FF_CHAIN_LIB=paper_2512_12949_b200/$lib.so timeout 300 python tools/timeline.py gpt67b llama opt > $O/t_${lib}_$i.log 2>&1; echo "## $lib"; grep "==" $O/t_${lib}_$i.log | sed 's/{.*}//'
done; done
