"""Run a list of chains x transports in sequence on one stream workspace, repeatedly, checking each result
(diagnostics, GPU box): reproduces order-dependent failures of tests/test_gpu_chain.py.

    python tools/repro_multi.py [iters=20] [cases=0,1,2] [x=dsm,l2,pair,l2dsm]"""
import os
import random
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def cases(n, seed):
    rng = random.Random(seed)
    out = []
    for _ in range(n):
        kind = rng.choice(["standard_ffn", "gated_ffn"])
        act = "silu" if kind == "gated_ffn" else rng.choice(["relu", "identity", "silu", "gelu"])
        m = rng.choice([16, 17, 64, 128, 200, 256, 384, 640])
        k = 128 * rng.randint(1, 12)
        n_ = 256 * rng.randint(1, 16)
        l = 256 * rng.randint(1, 8)
        out.append((kind, act, m, n_, k, l))
    return out


def main(argv):
    import oracle
    from paper_2512_12949_b200 import _native as nat
    from paper_2512_12949_b200 import runtime
    from paper_2512_12949_b200 import workload as W

    lib = nat.load()
    iters = next((int(a.split("=")[1]) for a in argv if a.startswith("iters=")), 20)
    sel = next((a.split("=")[1] for a in argv if a.startswith("cases=")), "0,1,2")
    xs = next((a.split("=")[1] for a in argv if a.startswith("x=")), "dsm,l2,pair,l2dsm").split(",")
    allc = cases(10, 2025)
    if "prealloc" in argv:  # one large workspace up front: no re-allocation between configs
        runtime._workspace(512 << 20, torch.device("cuda", 0), torch.cuda.current_stream())
    work = []
    for ci in (int(c) for c in sel.split(",")):
        kind, act, m, n, k, l = allc[ci]
        d = W.DimensionSpec(m, n, k, l)
        graph = W.build_gated_ffn(d) if kind == "gated_ffn" else W.build_standard_ffn(d, act)
        host = oracle.make_inputs(kind, m, n, k, l, seed=3)
        host = {kk: oracle.round_bf16(v) for kk, v in host.items()}
        dev = {kk: torch.from_numpy(v).cuda().to(torch.bfloat16) for kk, v in host.items()}
        ref = oracle.dense_chain(kind, act, host, bf16_intermediate=True)
        for x in xs:
            try:
                cfg = runtime.lower(graph, None, 148, x)
            except nat.UnsupportedPlan:
                continue
            work.append((ci, x, graph, cfg, dev, ref))
    for i in range(iters):
        for ci, x, graph, cfg, dev, ref in work:
            t0 = time.time()
            if "v" in argv:
                print(f"launch iter {i} case {ci} {x} {cfg.as_dict()}", flush=True)
            out = runtime.launch(graph, cfg, dev)
            torch.cuda.synchronize()
            if hasattr(lib, "ff_diag_read"):  # diagnostic build: which wait expired, if any
                import ctypes
                d3 = (ctypes.c_ulonglong * 1025)()
                lib.ff_diag_read(d3)
                if d3[0]:
                    print(f"iter {i} case {ci} {x} {cfg.as_dict()}: {d3[0]} expired waits", flush=True)
                    groups = {}
                    for j in range(min(512, d3[0])):
                        key, info = d3[1 + 2 * j], d3[2 + 2 * j]
                        line, blk, thr = key >> 40, (key >> 20) & 0xFFFFF, key & 0xFFFFF
                        g = groups.setdefault((line, blk, thr // 32, info), [j, 0, thr])
                        g[1] += 1
                    for (line, blk, w, info), (first, cnt, thr) in sorted(groups.items(), key=lambda kv: kv[1][0]):
                        print(f"    first #{first:3d} line {line} block {blk} warp {w} (thread {thr}) x{cnt} info {info:#x}",
                              flush=True)
            err = oracle.max_relative_error(out.float().cpu().numpy(), ref)
            if not np.isfinite(err) or err > 1e-2 or time.time() - t0 > 1.0:
                print(f"iter {i} case {ci} {x} {cfg.as_dict()}: err {err:.3e} {time.time() - t0:.2f} s", flush=True)
    print("done", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
