"""Interleaved A/B of two kernel variants (ff_set_variant) on BASELINE chains (diagnostics, GPU box only).

    python tools/ab_variant.py 0x0 0x2 [gpt67b llama1b ...] [steps=200]

Launches alternate A, B, A, B ... through the public runtime, each behind a 256 MiB L2
flush, timed with CUDA events; prints the medians and B / A."""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(argv):
    import bench
    from paper_2512_12949_b200 import _native, runtime

    lib = _native.load()
    va, vb = int(argv[0], 0), int(argv[1], 0)
    steps = next((int(a.split("=")[1]) for a in argv if a.startswith("steps=")), 200)
    names = [a for a in argv[2:] if a in bench.WORKLOADS or a in bench.CONV_WORKLOADS] or ["gpt67b"]
    flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def flush():
        flush_buf.add_(1.0)

    # variants may lay the workspace out differently (the tail split adds exchange regions):
    # one workspace large enough for all of them
    runtime._workspace(1 << 30, torch.device("cuda", 0), torch.cuda.current_stream())
    for name in names:
        if name in bench.CONV_WORKLOADS:  # conv chains: bench.py's shapes, the l2 lowering
            from paper_2512_12949_b200 import workload as W
            ic, h, w, oc1, oc2, k1, k2 = bench.CONV_WORKLOADS[name][0]
            ccfg = W.ConvChainConfig(ic, h, w, oc1, oc2, k1, k2) if k2 == 1 else W.ConvBlockConfig(ic, h, w, oc1, oc2, k1, k2)
            x = (torch.rand(1, h, w, ic, device="cuda") * 2 - 1).bfloat16()
            w1 = ((torch.rand(k1, k1, ic, oc1, device="cuda") * 2 - 1) / (k1 * k1 * ic) ** 0.5).bfloat16()
            w2 = ((torch.rand(*((oc1, oc2) if k2 == 1 else (k2, k2, oc1, oc2)), device="cuda") * 2 - 1) /
                  (k2 * k2 * oc1) ** 0.5).bfloat16()
            y = torch.empty(1, h, w, oc2, dtype=torch.bfloat16, device="cuda")
            kc = runtime.lower_conv(ccfg, 1, "l2")
            run = lambda: runtime.launch_conv(ccfg, kc, x, w1, w2, out=y)  # noqa: E731
        else:
            kind, act, m, n, k, l, _ = bench.WORKLOADS[name]
            t = bench.make_device_inputs(kind, m, n, k, l, seed=1, device="cuda")
            g = bench.graph_of(name, m)
            cfg = bench.choose_config(name, t, profile=False, m=m, flush=flush)[0]
            out = torch.empty((m, l), dtype=torch.bfloat16, device="cuda")
            run = lambda: runtime.launch(g, cfg, t, out=out)  # noqa: E731
        ts = {va: [], vb: []}
        for i in range(steps + 6):
            for v in (va, vb):
                lib.ff_set_variant(v)
                flush()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                run()
                b.record()
                torch.cuda.synchronize()
                if i >= 6:
                    ts[v].append(a.elapsed_time(b) * 1e3)
        lib.ff_set_variant(0)
        ma, mb = float(np.median(ts[va])), float(np.median(ts[vb]))
        # event timestamps are quantised (~1-2 us on these boxes): the trimmed means resolve finer
        ta, tb = (float(np.mean(np.sort(ts[v])[steps // 10: steps - steps // 10])) for v in (va, vb))
        print(f"{name:14s} variant {va:#x}: {ma:8.1f} us (trimmed mean {ta:8.2f})   variant {vb:#x}: {mb:8.1f} us "
              f"(trimmed mean {tb:8.2f})   B/A {tb / ta:.4f}  ({steps} interleaved steps each)")


if __name__ == "__main__":
    main(sys.argv[1:])
