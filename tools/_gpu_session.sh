# scratch driver (r02 session 7): batched TMEM drains in the 1-CTA kernels vs the 16-column loop (A build)
O=gpurun_out/r02s7; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests_drain.log 2>&1; echo "pytest rc=$?"; tail -2 $O/gpu_tests_drain.log
for r in 1 2; do
 for lib in libff_ab_drain16.so libff_chain.so; do
  echo "== $lib round $r"
  FF_CHAIN_LIB=paper_2512_12949_b200/$lib timeout 600 python tools/ab_variant.py 0x0 0x0 gpt2s llama1b conv_1x1_3x3 conv_c5 steps=200 2>&1 | grep variant
 done
done > $O/ab_drain.log 2>&1
cat $O/ab_drain.log
for lib in libff_ab_drain16.so libff_chain.so; do
  FF_CHAIN_LIB=paper_2512_12949_b200/$lib timeout 300 python tools/timeline.py gpt2s x0 counters 2>&1 | grep -E "==|cfull0|drained0|E_start|E_staged|E_fin"
  FF_CHAIN_LIB=paper_2512_12949_b200/$lib timeout 300 python tools/timeline.py gpt2s x3 cfg=6,4,128,128,3,4,1,1,16,16,96 2>&1 | grep -E "==|cfull0|drained0|E_start|E_staged|E_fin"
done > $O/timeline_drain.log 2>&1
cat $O/timeline_drain.log
