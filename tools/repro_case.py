"""Repeat one chain launch many times and check every result against the oracle (diagnostics, GPU box).

    python tools/repro_case.py standard_ffn relu 17 3328 512 512 pair [iters=50] [variant=0x..]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))


def main(argv):
    import oracle
    from paper_2512_12949_b200 import _native, runtime
    from paper_2512_12949_b200 import workload as W

    kind, act = argv[0], argv[1]
    m, n, k, l = (int(x) for x in argv[2:6])
    exchange = argv[6]
    iters = next((int(a.split("=")[1]) for a in argv if a.startswith("iters=")), 50)
    var = next((int(a.split("=")[1], 0) for a in argv if a.startswith("variant=")), 0)
    _native.load().ff_set_variant(var)
    d = W.DimensionSpec(m, n, k, l)
    graph = W.build_gated_ffn(d) if kind == "gated_ffn" else W.build_standard_ffn(d, act)
    cfg = runtime.lower(graph, None, 148, exchange)
    print("config", cfg.as_dict(), flush=True)
    host = oracle.make_inputs(kind, m, n, k, l, seed=3)
    host = {kk: oracle.round_bf16(v) for kk, v in host.items()}
    dev = {kk: torch.from_numpy(v).cuda().to(torch.bfloat16) for kk, v in host.items()}
    ref = oracle.dense_chain(kind, act, host, bf16_intermediate=True)
    worst = 0.0
    for i in range(iters):
        out = runtime.launch(graph, cfg, dev)
        torch.cuda.synchronize()
        err = oracle.max_relative_error(out.float().cpu().numpy(), ref)
        worst = max(worst, err)
        if not np.isfinite(err) or err > 1e-2:
            print(f"iter {i}: max rel err {err:.3e}", flush=True)
    print(f"{iters} launches ok, worst max rel err {worst:.3e}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
