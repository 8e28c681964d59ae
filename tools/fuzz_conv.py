# One-off GPU fuzz of the conv chains: seeded random (batch, h, w, channels, filter sizes)
# within the lowering's constraints, every transport, vs the CPU oracle.  Not in pytest (slow).
import sys, random
import numpy as np
import torch
sys.path.insert(0, '.')
import oracle
from paper_2512_12949_b200 import _native as nat, runtime
from paper_2512_12949_b200.workload import ConvBlockConfig, ConvChainConfig

rng = random.Random(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
n_cases = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ran = fails = 0
for i in range(n_cases):
    block = rng.random() < 0.4
    b = rng.choice([1, 1, 2, 3])
    h, w = rng.randint(3, 40), rng.randint(3, 40)
    if block:  # 1x1 -> act -> k2 x k2
        k1, k2 = 1, rng.choice([3, 5])
        ic = 64 * rng.randint(1, 4)
        oc1 = rng.choice([64, 128]); oc2 = rng.choice([64, 128, 256])
        cfg = ConvBlockConfig(ic, h, w, oc1, oc2, k1, k2)
    else:      # k1 x k1 -> act -> 1x1
        k1, k2 = rng.choice([1, 3, 5]), 1
        ic = 64 * rng.randint(1, 3)
        oc1 = 64 * rng.randint(1, 4); oc2 = 64 * rng.randint(1, 4)
        cfg = ConvChainConfig(ic, h, w, oc1, oc2, k1, k2)
    g = np.random.default_rng(i)
    x = oracle.round_bf16(g.uniform(-1, 1, (b, h, w, ic)).astype(np.float32))
    w1 = oracle.round_bf16(g.uniform(-1, 1, (k1, k1, ic, oc1)).astype(np.float32) / np.sqrt(k1 * k1 * ic))
    w2s = (oc1, oc2) if k2 == 1 else (k2, k2, oc1, oc2)
    w2 = oracle.round_bf16(g.uniform(-1, 1, w2s).astype(np.float32) / np.sqrt(k2 * k2 * oc1))
    ref = oracle.conv_chain(x, w1, w2, 'relu')
    X, W1, W2 = (torch.from_numpy(a).cuda().bfloat16() for a in (x, w1, w2))
    for xch in ('pair', 'l2', 'dsm'):
        try:
            kc = runtime.lower_conv(cfg, b, xch)
        except nat.UnsupportedPlan:
            continue
        try:
            y = runtime.launch_conv(cfg, kc, X, W1, W2)
            torch.cuda.synchronize()
        except (nat.NativeError, ValueError) as e:
            fails += 1
            print('ERROR', cfg, b, xch, kc.as_dict(), e, flush=True)
            continue
        got = y.float().cpu().numpy()
        err = oracle.max_relative_error(got, ref)
        ran += 1
        if not (np.isfinite(got).all() and err <= 1e-2):
            fails += 1
            print('FAIL', cfg, b, xch, kc.as_dict(), err, flush=True)
print(f'conv fuzz: {ran} launches, {fails} failures', flush=True)
