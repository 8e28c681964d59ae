# scratch driver (r02 session 7): rebuild the shipped M-bin tables with the reproducible candidates, bench, suite
O=gpurun_out/r02s7; mkdir -p $O
cp -r paper_2512_12949_b200/plans/dispatch $O/dispatch_before
( time timeout 1500 python -m paper_2512_12949_b200.dispatch ) > $O/dispatch_build.log 2>&1; echo "dispatch rc=$?"; tail -6 $O/dispatch_build.log
mkdir -p $O/dispatch_after && cp paper_2512_12949_b200/plans/dispatch/*.json $O/dispatch_after/
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests3.log 2>&1; echo "pytest rc=$?"; tail -2 $O/gpu_tests3.log
timeout 900 python bench.py > $O/bench3.json 2> $O/bench3.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('$O/bench3.json').read().strip().splitlines()[-1])
print(d['value'], d['config']['bit_reproducible'], d['config']['plan'][:80], d['fused_vs_cublas']['speedup'], d['e2e']['value'])
for k,v in d['extra'].items(): print(k, v.get('bit_reproducible'), str(v.get('plan'))[:70], v.get('interleaved'))
"
