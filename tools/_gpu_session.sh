# scratch driver (r02 session 6n): config sweep with the final kernels (GPT-2s, LLaMA-1B, GPT-6.7B)
set -x
O=gpurun_out/r02s6n; mkdir -p $O
timeout 1800 python tools/sweep_configs.py gpt2s llama1b gpt67b > $O/sweep.log 2>&1; echo "rc=$?"
grep -A8 "==" $O/sweep.log | head -40
