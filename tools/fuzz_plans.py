# One-off GPU fuzz of the plan lowering (ff_plan_lower): random valid plans of the
# reference search space (sample_valid_plans, B200 profile) lowered to every transport
# and run against the CPU oracle.  Not in pytest (slow).
import sys, random
import numpy as np
import torch
sys.path.insert(0, '.')
import oracle
from paper_2512_12949_b200 import _native as nat, runtime
from paper_2512_12949_b200 import workload as W
from paper_2512_12949_b200.hardware import b200_profile
from paper_2512_12949_b200.simulator import sample_valid_plans

dev = b200_profile()
rng = random.Random(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
ran = fails = lowered_none = 0
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 12):
    kind = rng.choice(['standard_ffn', 'gated_ffn'])
    m, n, k, l = rng.choice([256, 512, 1024]), 256 * rng.randint(2, 16), 128 * rng.randint(2, 16), 256 * rng.randint(1, 8)
    d = W.DimensionSpec(m, n, k, l, 2)
    g = W.build_gated_ffn(d) if kind == 'gated_ffn' else W.build_standard_ffn(d, 'relu')
    plans = sample_valid_plans(g, dev, 6, seed=i)
    host = {nm: oracle.round_bf16(v) for nm, v in oracle.make_inputs(kind, m, n, k, l, seed=i).items()}
    tens = {nm: torch.from_numpy(v).cuda().bfloat16() for nm, v in host.items()}
    ref = oracle.dense_chain(kind, 'relu' if kind == 'standard_ffn' else 'silu', host)
    for plan in plans:
        for x in ('pair', 'l2', 'dsm'):
            try:
                cfg = runtime.lower(g, plan, 148, x)
            except nat.UnsupportedPlan:
                lowered_none += 1
                continue
            try:
                out = runtime.launch(g, cfg, tens)
                torch.cuda.synchronize()
            except nat.NativeError as e:
                fails += 1
                print('ERROR', kind, (m, n, k, l), plan.describe(), x, cfg.as_dict(), e, flush=True)
                continue
            got = out.float().cpu().numpy()
            err = oracle.max_relative_error(got, ref)
            ran += 1
            if not (np.isfinite(got).all() and err <= 1e-2):
                fails += 1
                print('FAIL', kind, (m, n, k, l), plan.describe(), x, cfg.as_dict(), err, flush=True)
print(f'plan fuzz: {ran} launches, {fails} failures, {lowered_none} unsupported lowerings', flush=True)
