# scratch driver (r02 session 6x): bench with a rest before every extra config
set -x
O=gpurun_out/r02s6x; mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r02s6x/bench.json').read().strip().splitlines()[-1])
print(d['value'], json.dumps(d['fused_vs_cublas'])[:200])
for k,v in d['extra'].items(): print(k, v.get('fused_ms'), v.get('cublas_best_ms'), v.get('speedup_vs_cublas_best'), v.get('interleaved'))
PY
