# scratch driver (r02 session 5t): where the split-N tail goes (A/B builds, results invalid except libff_chain)
set -x
O=gpurun_out/r02s5t; mkdir -p $O
for i in 1 2; do
for lib in libff_chain libff_ab_tail1 libff_ab_tail2 libff_ab_tail3; do
  FF_CHAIN_LIB=paper_2512_12949_b200/$lib.so timeout 300 python tools/timeline.py gpt67b llama > $O/t_${lib}_$i.log 2>&1
  echo "## $lib"; grep -h "==\|E_start\|exit" $O/t_${lib}_$i.log | sed 's/{.*}//'
done
done
