# scratch driver (r02 session 6e): cold-start weight prefetch A/B
set -x
O=gpurun_out/r02s6e; mkdir -p $O
for i in 1 2 3; do for lib in libff_chain libff_cp8 libff_cp16; do
  FF_CHAIN_LIB=paper_2512_12949_b200/$lib.so timeout 300 python tools/timeline.py gpt67b llama > $O/t_${lib}_$i.log 2>&1; echo "## $lib"; grep "==\|cfull0" $O/t_${lib}_$i.log | sed 's/{.*}//'
done; done
