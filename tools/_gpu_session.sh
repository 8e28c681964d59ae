# scratch driver (r02 session 6a): 1-CTA trims: HEAD vs trim-1 vs all
set -x
O=gpurun_out/r02s6a; mkdir -p $O
for i in 1 2 3; do for lib in libff_t0 libff_t1 libff_chain; do
  FF_CHAIN_LIB=paper_2512_12949_b200/$lib.so timeout 300 python tools/timeline.py gpt2s x0 > $O/t_${lib}_$i.log 2>&1; echo "## $lib"; grep "==" $O/t_${lib}_$i.log | sed 's/{.*}//'
done; done
