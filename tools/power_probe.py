"""Sustained power / clock of the fused chain vs the unfused cuBLAS path (diagnostics, GPU box only).

    python tools/power_probe.py [gpt67b|llama1b|opt13b_m32768 ...] [variant=0x..] [variant2=0x..] [seconds=2]

For each arm: run (L2 flush + step) back to back for `seconds`, sampling NVML power,
SM clock and throttle reasons every ~5 ms on a side thread; print the mean power, the
median SM clock under load, the median per-step time (CUDA events) and the energy per step
from NVML's total-energy counter (minus a flush-only step's)."""

import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def sample(stop, out):
    import pynvml

    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    while not stop.is_set():
        try:
            out.append((pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
        except Exception:
            pass
        time.sleep(0.005)


def energy_mj():
    import pynvml

    pynvml.nvmlInit()
    return pynvml.nvmlDeviceGetTotalEnergyConsumption(pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device()))


def run_arm(fn, flush, seconds):
    stop, out = threading.Event(), []
    th = threading.Thread(target=sample, args=(stop, out), daemon=True)
    ts = []
    torch.cuda.synchronize()
    e0, w0 = energy_mj(), time.time()
    th.start()
    t_end = time.time() + seconds
    while time.time() < t_end:
        evs = []
        for _ in range(50):
            flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            evs.append((a, b))
        torch.cuda.synchronize()
        ts += [a.elapsed_time(b) * 1e3 for a, b in evs]
    e1, w1 = energy_mj(), time.time()
    stop.set()
    th.join()
    run_arm.last_energy = ((e1 - e0) / len(ts), (e1 - e0) / (w1 - w0))  # mJ per step (incl. flush), mean W
    p = np.array([o[0] for o in out]) if out else np.zeros(1)
    c = np.array([o[1] for o in out]) if out else np.zeros(1)
    return float(np.median(ts)), float(p.mean()), float(np.median(c)), len(ts)


def main(argv):
    import bench
    from paper_2512_12949_b200 import _native, runtime

    var = next((int(a.split("=")[1], 0) for a in argv if a.startswith("variant=")), 0)
    secs = next((float(a.split("=")[1]) for a in argv if a.startswith("seconds=")), 2.0)
    if var:
        _native.load().ff_set_variant(var)
    names = [a for a in argv if a in bench.WORKLOADS] or ["gpt67b"]
    flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def flush():
        flush_buf.add_(1.0)

    idle = torch.zeros(1, device="cuda")
    print(f"idle (flush + 1-element op): step {run_arm(lambda: idle.add_(1), flush, 1.0)}")
    e_idle = run_arm.last_energy[0]
    print(f"   energy per idle step (the flush): {e_idle:.2f} mJ")
    for name in names:
        kind, act, m, n, k, l, _ = bench.WORKLOADS[name]
        t = bench.make_device_inputs(kind, m, n, k, l, seed=1, device="cuda")
        g = bench.graph_of(name, m)
        cfg = bench.choose_config(name, t, profile=False, m=m, flush=flush)[0]
        out = torch.empty((m, l), dtype=torch.bfloat16, device="cuda")
        arms = [("fused", lambda: runtime.launch(g, cfg, t, out=out)),
                ("cublas fused_epilogue_graph", bench._cublas_best_fn(kind, act, t, "fused_epilogue_graph"))]
        var2 = next((int(a.split("=")[1], 0) for a in argv if a.startswith("variant2=")), None)
        if var2 is not None:
            lib = _native.load()

            def fused_v2():
                lib.ff_set_variant(var2)
                runtime.launch(g, cfg, t, out=out)
                lib.ff_set_variant(var)
            arms.append((f"fused variant {var2:#x}", fused_v2))
        for label, fn in arms:
            for _ in range(5):
                fn()
            torch.cuda.synchronize()
            us, watts, mhz, n_steps = run_arm(fn, flush, secs)
            mj, avg_w = run_arm.last_energy
            print(f"{name:14s} {label:28s} step {us:8.1f} us  power {watts:6.0f} W  sm clock {mhz:6.0f} MHz  "
                  f"energy {mj:6.2f} mJ/step, {mj - e_idle:6.2f} above the flush-only step  ({n_steps} steps)")
            time.sleep(1.0)


if __name__ == "__main__":
    main(sys.argv[1:])
