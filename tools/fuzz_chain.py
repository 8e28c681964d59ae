# One-off GPU fuzz: seeded random chains (incl. ragged N / uneven splits, fp16) under every
# transport against the CPU oracle; prints failures.  Not part of the pytest suite (slow).
import sys, random
import numpy as np
import torch
sys.path.insert(0, '.')
import oracle
from paper_2512_12949_b200 import _native as nat, runtime
from paper_2512_12949_b200 import workload as W

def graph(kind, act, m, n, k, l):
    d = W.DimensionSpec(m, n, k, l, 2)
    return W.build_gated_ffn(d) if kind == 'gated_ffn' else W.build_standard_ffn(d, act)

lib = nat.load()
rng = random.Random(int(sys.argv[1]) if len(sys.argv) > 1 else 7)
n_cases, fails, ran = int(sys.argv[2]) if len(sys.argv) > 2 else 60, 0, 0
for i in range(n_cases):
    kind = rng.choice(['standard_ffn', 'gated_ffn'])
    act = 'silu' if kind == 'gated_ffn' else rng.choice(['relu', 'identity', 'silu', 'gelu'])
    m = rng.choice([16, 40, 128, 200, 256, 384, 512, 640, 1000])
    k = 128 * rng.randint(1, 16)
    n = 128 * rng.randint(1, 40)
    l = 256 * rng.randint(1, 10)
    f16 = rng.random() < 0.25
    g = graph(kind, act, m, n, k, l)
    host = {nm: oracle.round_bf16(v) for nm, v in oracle.make_inputs(kind, m, n, k, l, seed=i).items()}
    if f16:
        host = {nm: (v / (np.sqrt(v.shape[0]) if nm != 'A' else 1.0)).astype(np.float16).astype(np.float32)
                for nm, v in host.items()}
    dt = torch.float16 if f16 else torch.bfloat16
    dev = {nm: torch.from_numpy(v).cuda().to(dt) for nm, v in host.items()}
    if kind == 'gated_ffn':
        w = torch.stack([dev['B0'], dev['B1']]); dev['B0'], dev['B1'] = w[0], w[1]
    ref = oracle.dense_chain(kind, act, host)
    for x in ('pair', 'l2', 'dsm'):
        try:
            cfg = runtime.lower(g, None, 148, x)
        except nat.UnsupportedPlan:
            continue
        try:
            out = runtime.launch(g, cfg, dev)
            torch.cuda.synchronize()
        except nat.NativeError as e:
            fails += 1
            print('ERROR', kind, act, (m, n, k, l), 'f16' if f16 else 'bf16', x, cfg.as_dict(), e, flush=True)
            continue
        if hasattr(lib, 'ff_diag_read'):  # diagnostic build (FF_CHAIN_LIB=...libff_diag.so): expired waits
            import ctypes
            d = (ctypes.c_ulonglong * 1025)()
            lib.ff_diag_read(d)
            if d[0]:
                fails += 1
                print('EXPIRED', kind, act, (m, n, k, l), x, cfg.as_dict(), d[0], 'first line', d[1] >> 40,
                      'block', (d[1] >> 20) & 0xFFFFF, 'thread', d[1] & 0xFFFFF, hex(d[2]), flush=True)
        got = out.float().cpu().numpy()
        err = oracle.max_relative_error(got, ref)
        ran += 1
        if not (np.isfinite(got).all() and err <= 1e-2):
            fails += 1
            print('FAIL', kind, act, (m, n, k, l), 'f16' if f16 else 'bf16', x, cfg.as_dict(), err, flush=True)
print(f'fuzz: {ran} launches, {fails} failures', flush=True)
