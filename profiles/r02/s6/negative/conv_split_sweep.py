"""Tap-split sweep of a 1x1 -> act -> k2 x k2 conv block (diagnostics, GPU box only).

    python tools/conv_split_sweep.py [splits=1,2,3,4,5,9]

Times the ResNet block of bench.py (256->64->64, 56x56) for each GEMM1 k-block split count,
L2 flushed before every step, and checks each result against the S = 1 launch."""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(argv):
    import bench
    from paper_2512_12949_b200 import runtime, workload as W

    splits = next((a.split("=")[1] for a in argv if a.startswith("splits=")), "1,2,3,4,5,9")
    shape = bench.CONV_WORKLOADS["conv_1x1_3x3"][0]
    ic, h, w, oc1, oc2, k1, k2 = shape
    cfg = W.ConvBlockConfig(*shape)
    g = torch.Generator(device="cpu").manual_seed(11)
    x = (torch.rand(1, h, w, ic, generator=g) * 2 - 1).to(torch.bfloat16).cuda()
    w1 = ((torch.rand(k1, k1, ic, oc1, generator=g) * 2 - 1) / (ic ** 0.5)).to(torch.bfloat16).cuda()
    w2 = ((torch.rand(k2, k2, oc1, oc2, generator=g) * 2 - 1) / (k2 * k2 * oc1) ** 0.5).to(torch.bfloat16).cuda()
    flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def flush():
        flush_buf.add_(1.0)

    base = runtime.lower_conv(cfg, 1, "l2")
    ref = None
    for s in (int(v) for v in splits.split(",")):
        kcfg = runtime.lower_conv(cfg, 1, "l2")
        kcfg.n_splits = s
        y = torch.empty(1, h, w, oc2, dtype=torch.bfloat16, device="cuda")
        fn = lambda: runtime.launch_conv(cfg, kcfg, x, w1, w2, out=y)  # noqa: E731
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        if ref is None:
            ref = y.float().clone()
        err = ((y.float() - ref).abs().max() / ref.abs().max()).item()
        ms = float(np.median(bench.time_steps(fn, 50, flush, torch.cuda.current_stream())))
        print(f"tap splits {s}: {ms * 1e3:6.1f} us  (max rel. diff vs S=1 {err:.2e})  lowered default S={base.n_splits}")


if __name__ == "__main__":
    main(sys.argv[1:])
