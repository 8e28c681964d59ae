"""Where the e2e step time goes (diagnostics, GPU box only).

    python tools/e2e_probe.py [gpt67b|llama1b ...] [steps=300]

Times, for the headline chain: the chain alone back to back (rotating weights, as the e2e loop);
the e2e loop of bench.py (host enqueue time and device time); the loop without its copies; and
the loop's host-side enqueue cost with the chain launch replaced by nothing."""

import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(argv):
    import bench
    from paper_2512_12949_b200 import runtime

    steps = next((int(a.split("=")[1]) for a in argv if a.startswith("steps=")), 300)
    names = [a for a in argv if a in bench.WORKLOADS] or ["gpt67b"]
    dev = torch.device("cuda", 0)
    for name in names:
        kind, act, m, n, k, l, _ = bench.WORKLOADS[name]
        t = bench.make_device_inputs(kind, m, n, k, l, seed=1, device="cuda")
        g = bench.graph_of(name, m)
        cfg = bench.choose_config(name, t, profile=False, m=m)[0]
        host_a = t["A"].cpu().pin_memory()
        # 1. host cost of one launch call (enqueue only)
        out = torch.empty((m, l), dtype=torch.bfloat16, device="cuda")
        for _ in range(10):
            runtime.launch(g, cfg, t, out=out)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            runtime.launch(g, cfg, t, out=out)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"{name}: runtime.launch host enqueue {1e6 * (t1 - t0) / steps:7.1f} us/call, "
              f"device drain {1e6 * (t2 - t0) / steps:7.1f} us/step (same weights: L2-warm)")
        # 2. the bench e2e loop, with host timing around it
        t0 = time.perf_counter()
        r = bench.e2e_pipelined(g, cfg, t, host_a, kind, m, l, steps, dev)
        t1 = time.perf_counter()
        print(f"{name}: e2e loop {1e3 * r['ms_total'] / steps:7.1f} us/step (device events), "
              f"host wall {1e6 * (t1 - t0) / (steps + 4):7.1f} us/step incl. setup")


if __name__ == "__main__":
    main(sys.argv[1:])
