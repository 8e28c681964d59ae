"""Timing probe: ragged pair rings (N chunks not a ring multiple) vs cuBLAS GEMM + act + GEMM."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_12949_b200 import runtime  # noqa: E402
from paper_2512_12949_b200 import workload as W  # noqa: E402

flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")


def timed(fn, iters=50):
    for _ in range(5):
        fn()
    ts = []
    for _ in range(iters):
        flush.add_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return sorted(ts)[len(ts) // 2]


for kind, m, n, k, l in [("gated_ffn", 512, 11008, 4096, 4096), ("gated_ffn", 128, 11008, 4096, 4096),
                         ("gated_ffn", 512, 13824, 5120, 5120), ("standard_ffn", 256, 8960, 1536, 1536),
                         ("gated_ffn", 512, 8192, 2048, 2048)]:
    d = W.DimensionSpec(m, n, k, l, 2)
    g = W.build_gated_ffn(d) if kind == "gated_ffn" else W.build_standard_ffn(d, "relu")
    A = torch.randn(m, k, device="cuda").bfloat16()
    D = (torch.randn(n, l, device="cuda") * 0.02).bfloat16()
    if kind == "gated_ffn":
        w = (torch.randn(2, k, n, device="cuda") * 0.02).bfloat16()
        t = {"A": A, "B0": w[0], "B1": w[1], "D": D}
        ref = lambda: (torch.nn.functional.silu(A @ w[0]) * (A @ w[1])) @ D
    else:
        B = (torch.randn(k, n, device="cuda") * 0.02).bfloat16()
        t = {"A": A, "B": B, "D": D}
        ref = lambda: torch.relu(A @ B) @ D
    cfg = runtime.lower(g, None, 148, "pair")
    out = torch.empty(m, l, dtype=torch.bfloat16, device="cuda")
    us = timed(lambda: runtime.launch(g, cfg, t, out=out))
    err = ((out.float() - ref().float()).abs().max() / ref().float().abs().max()).item()
    print(f"{kind} {m}x{n}x{k}x{l} cfg={cfg.as_dict()} fused={us:.1f}us cublas={timed(ref):.1f}us relerr={err:.2e}",
          flush=True)
