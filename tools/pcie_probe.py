"""Host <-> device copy bandwidth of the GPU box (diagnostics, GPU box only): the bound on bench.py's e2e.

    python tools/pcie_probe.py [mib=4] [n=200]

Pinned host buffers, one copy stream per direction: H2D alone, D2H alone, and both at once
(the e2e loop's pattern), timed with CUDA events."""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(argv):
    mib = next((int(a.split("=")[1]) for a in argv if a.startswith("mib=")), 4)
    n = next((int(a.split("=")[1]) for a in argv if a.startswith("n=")), 200)
    nbytes = mib << 20
    h_in = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(h2d, d2h):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        s1.wait_event(a)
        s2.wait_event(a)
        for _ in range(n):
            if h2d:
                with torch.cuda.stream(s1):
                    d_in.copy_(h_in, non_blocking=True)
            if d2h:
                with torch.cuda.stream(s2):
                    h_out.copy_(d_out, non_blocking=True)
        e1, e2 = torch.cuda.Event(), torch.cuda.Event()
        e1.record(s1)
        e2.record(s2)
        torch.cuda.current_stream().wait_event(e1)
        torch.cuda.current_stream().wait_event(e2)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) * 1e3 / n  # us per copy (pair)

    order = ((True, True, "H2D + D2H"), (False, True, "D2H alone"), (True, False, "H2D alone"),
             (True, True, "H2D + D2H"), (True, False, "H2D alone"))
    for h2d, d2h, label in order:
        timed(h2d, d2h)
        us = timed(h2d, d2h)
        print(f"{label:10s} {mib} MiB: {us:8.1f} us per step, {nbytes / us / 1e3:6.1f} GB/s per direction")


if __name__ == "__main__":
    main(sys.argv[1:])
