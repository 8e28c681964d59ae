"""Run one chain under a sequence of transports, repeatedly, on one stream workspace (diagnostics, GPU box).

    python tools/repro_seq.py standard_ffn relu 17 3328 512 512 dsm,l2,pair,l2dsm [iters=30]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(argv):
    import oracle
    from paper_2512_12949_b200 import _native as nat
    from paper_2512_12949_b200 import runtime
    from paper_2512_12949_b200 import workload as W

    kind, act = argv[0], argv[1]
    m, n, k, l = (int(x) for x in argv[2:6])
    exchanges = argv[6].split(",")
    iters = next((int(a.split("=")[1]) for a in argv if a.startswith("iters=")), 30)
    d = W.DimensionSpec(m, n, k, l)
    graph = W.build_gated_ffn(d) if kind == "gated_ffn" else W.build_standard_ffn(d, act)
    host = oracle.make_inputs(kind, m, n, k, l, seed=3)
    host = {kk: oracle.round_bf16(v) for kk, v in host.items()}
    dev = {kk: torch.from_numpy(v).cuda().to(torch.bfloat16) for kk, v in host.items()}
    ref = oracle.dense_chain(kind, act, host, bf16_intermediate=True)
    cfgs = {}
    for x in exchanges:
        try:
            cfgs[x] = runtime.lower(graph, None, 148, x)
            print(x, cfgs[x].as_dict(), flush=True)
        except nat.UnsupportedPlan:
            print(x, "unsupported", flush=True)
    for i in range(iters):
        for x, cfg in cfgs.items():
            t0 = time.time()
            out = runtime.launch(graph, cfg, dev)
            torch.cuda.synchronize()
            err = oracle.max_relative_error(out.float().cpu().numpy(), ref)
            if not np.isfinite(err) or err > 1e-2 or time.time() - t0 > 1.0:
                print(f"iter {i} {x}: err {err:.3e} {time.time() - t0:.2f} s", flush=True)
    print("done", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
