#!/bin/bash
# Headline bench A/B of two kernel variants (GPU box): alternating full bench.py runs (sustained
# 1000-step timed region, as the driver measures), --no-extra --no-cpu.
#   bash tools/bench_ab.sh 0x0 0x4 [rounds=2] > gpurun_out/bench_ab.log
VA=${1:-0x0}; VB=${2:-0x4}; R=${3:-2}
for i in $(seq 1 "$R"); do
  for v in "$VA" "$VB"; do
    FF_BENCH_VARIANT=$v timeout 600 python bench.py --no-extra --no-cpu --rest 0 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('variant $v', d['value'], d['ms_per_step'], \
'vs cublas interleaved', d['fused_vs_cublas']['fused_ms'], d['fused_vs_cublas']['cublas_best_ms'], d['fused_vs_cublas']['speedup'], 'clock', d['clocks'].get('sm_mhz'))"
  done
done
