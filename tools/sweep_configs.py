"""Exhaustive launch-config sweep (exchange, ring, N splits, nb, lb) for the BASELINE chains:
median of cold-L2 launches, checked against cuBLAS; prints the top configs and the auto choice."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_12949_b200 import _native as nat  # noqa: E402
from paper_2512_12949_b200 import runtime  # noqa: E402
from paper_2512_12949_b200 import workload as W  # noqa: E402

flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
WL = {"gpt2s": ("standard_ffn", "gelu", 512, 3072, 768, 768), "llama1b": ("gated_ffn", "silu", 512, 8192, 2048, 2048),
      "gpt67b": ("standard_ffn", "relu", 512, 16384, 4096, 4096), "opt4096": ("standard_ffn", "relu", 4096, 8192, 2048, 2048)}


def timed(fn, iters):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(iters):
        flush.add_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return sorted(ts)[len(ts) // 2]


for name in sys.argv[1:]:
    kind, act, m, n, k, l = WL[name]
    d = W.DimensionSpec(m, n, k, l, 2)
    g = W.build_gated_ffn(d) if kind == "gated_ffn" else W.build_standard_ffn(d, act)
    A = torch.randn(m, k, device="cuda").bfloat16()
    D = (torch.randn(n, l, device="cuda") * 0.02).bfloat16()
    if kind == "gated_ffn":
        w = (torch.randn(2, k, n, device="cuda") * 0.02).bfloat16()
        t = {"A": A, "B0": w[0], "B1": w[1], "D": D}
        ref = (torch.nn.functional.silu(A.float() @ w[0].float()) * (A.float() @ w[1].float())) @ D.float()
    else:
        B = (torch.randn(k, n, device="cuda") * 0.02).bfloat16()
        t = {"A": A, "B": B, "D": D}
        c = A.float() @ B.float()
        c = torch.relu(c) if act == "relu" else torch.nn.functional.gelu(c, approximate="tanh")
        ref = c @ D.float()
    out = torch.empty(m, l, dtype=torch.bfloat16, device="cuda")
    auto = runtime.lower(g, None, 148, "pair")
    res = []
    for x in ("dsm", "l2", "pair", "l2dsm"):
        for lb in (64, 128, 256):
            for nb in (64, 128, 256):
                for ring in range(1, 17):
                    if l % (ring * lb):
                        continue
                    for S in (1, 2, 3, 4, 6, 8, 12, 16):
                        cfg = nat.KernelConfig()
                        cfg.ring, cfg.n_splits, cfg.nb, cfg.lb, cfg.exchange = ring, S, nb, lb, runtime.EXCHANGES[x]
                        try:
                            runtime.launch(g, cfg, t, out=out)
                            torch.cuda.synchronize()
                        except nat.UnsupportedPlan:
                            continue
                        err = ((out.float() - ref).abs().max() / ref.abs().max()).item()
                        us = timed(lambda: runtime.launch(g, cfg, t, out=out), 10)
                        res.append((us, x, ring, S, nb, lb, err))
    res.sort()
    print(f"== {name}: {len(res)} configs; auto {auto.as_dict()}", flush=True)
    for r in res[:12]:
        print("   %7.1f us  %-4s ring %2d S %2d nb %3d lb %3d  err %.1e" % r, flush=True)
    bad = [r for r in res if not r[-1] < 2e-2]
    print("   bad:", bad[:5], flush=True)
