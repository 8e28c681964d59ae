"""Bitwise comparison of two kernel variants' outputs on BASELINE chains (diagnostics, GPU box only).

    python tools/variant_equal.py 0x0 0x1000 [gpt67b gpt2s ...]"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(argv):
    import bench
    from paper_2512_12949_b200 import _native, runtime

    lib = _native.load()
    va, vb = int(argv[0], 0), int(argv[1], 0)
    names = [a for a in argv[2:] if a in bench.WORKLOADS] or ["gpt67b"]
    runtime._workspace(1 << 30, torch.device("cuda", 0), torch.cuda.current_stream())
    for name in names:
        kind, act, m, n, k, l, _ = bench.WORKLOADS[name]
        t = bench.make_device_inputs(kind, m, n, k, l, seed=3, device="cuda")
        g = bench.graph_of(name, m)
        cfg = bench.choose_config(name, t, profile=False, m=m)[0]
        outs = []
        for v in (va, vb, va, vb):
            lib.ff_set_variant(v)
            out = torch.full((m, l), float("nan"), dtype=torch.bfloat16, device="cuda")
            runtime.launch(g, cfg, t, out=out)
            torch.cuda.synchronize()
            outs.append(out)
        lib.ff_set_variant(0)
        same = torch.equal(outs[0], outs[1])
        diff = (outs[0].float() - outs[1].float()).abs().max().item()
        print(f"{name:14s} {va:#x} vs {vb:#x}: bitwise equal {same}  max |diff| {diff:.3g}  "
              f"repeat A {torch.equal(outs[0], outs[2])} repeat B {torch.equal(outs[1], outs[3])}  "
              f"finite {bool(torch.isfinite(outs[1].float()).all())}")


if __name__ == "__main__":
    main(sys.argv[1:])
