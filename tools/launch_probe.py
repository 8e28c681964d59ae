"""Post-flush launch cost probe (diagnostics, GPU box only).

    python tools/launch_probe.py

For each kernel X: flush the L2 (256 MiB write), then time X between CUDA events,
(a) right after the flush and (b) after a 1-element torch op that absorbs any
post-flush cost of the first launch.  Prints the median of 20."""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from bench import make_device_inputs, graph_of, choose_config, cublas_step_fn  # noqa: E402
    from paper_2512_12949_b200 import runtime

    flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    tiny = torch.zeros(1, device="cuda")

    def flush():
        flush_buf.add_(1.0)

    def med(fn, absorb, n=20):
        ts = []
        for _ in range(n):
            flush()
            if absorb:
                tiny.add_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        return float(np.median(ts))

    rows = [("tiny torch op", lambda: tiny.add_(1.0))]
    for name in sys.argv[1:] or ["gpt67b", "llama1b"]:
        from bench import WORKLOADS
        kind, act, m, n, k, l, _ = WORKLOADS[name]
        t = make_device_inputs(kind, m, n, k, l, seed=1, device="cuda")
        g = graph_of(name, m)
        cfg, _, _, _ = choose_config(name, t, profile=False, m=m, flush=flush)
        out = torch.empty((m, l), dtype=torch.bfloat16, device="cuda")
        rows.append((f"{name} fused chain", lambda g=g, cfg=cfg, t=t, out=out: runtime.launch(g, cfg, t, out=out)))
        for v in ("eager", "fused_epilogue"):
            fn, _ = cublas_step_fn(kind, act, t, v)
            rows.append((f"{name} cublas {v}", fn))
        if kind != "gated_ffn":
            a, b = t["A"], t["B"]
            rows.append((f"{name} cublas GEMM1 only", lambda a=a, b=b: torch.matmul(a, b)))
            c = torch.matmul(a, b)
            rows.append((f"{name} cublas GEMM2 only", lambda c=c, d=t["D"]: torch.matmul(c, d)))
        for _ in range(3):
            for _, fn in rows:
                fn()
    torch.cuda.synchronize()
    for label, fn in rows:
        print(f"{label:40s} after flush {med(fn, False):8.1f} us   flush+tiny op first {med(fn, True):8.1f} us")


if __name__ == "__main__":
    main()
