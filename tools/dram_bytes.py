"""DRAM bytes of one fused chain vs the unfused cuBLAS path, write-backs included.

Run under ncu on the GPU box (one process per (workload, impl)):

    ncu --cache-control none --clock-control none \
        --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --csv --log-file out.csv python tools/dram_bytes.py run <workload> <fused|cublas_eager|cublas_fused_epilogue>
    python tools/dram_bytes.py parse out.csv        # -> JSON line

Sequence per process: 3 x [flush, step, flush], where flush is a READ of a
512 MiB buffer (torch.sum: it leaves clean lines and evicts everything, so
the dirty lines a step leaves in L2 are written back -- and counted -- in the
flush right after it).  ncu's own cache control is off, so nothing is
flushed outside the measured kernels.  The last repetition is reported:
step read + step write + the following flush's write (= the step's deferred
write-backs)."""

import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(workload, impl):
    import torch

    import bench
    from paper_2512_12949_b200 import runtime

    kind, act, m, n, k, l, _ = bench.WORKLOADS[workload]
    t = bench.make_device_inputs(kind, m, n, k, l, seed=3, device="cuda")
    big = torch.ones(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    sink = torch.empty((), dtype=torch.float32, device="cuda")

    def flush():
        torch.sum(big, dim=0, out=sink)

    if impl == "fused":
        graph = bench.graph_of(workload)
        cfg = bench.choose_config(workload, t, profile=False)[0]
        out = torch.empty((m, l), dtype=torch.bfloat16, device="cuda")

        def step():
            runtime.launch(graph, cfg, t, out=out)
    else:  # cublas_eager | cublas_fused_epilogue
        step = bench.cublas_step_fn(kind, act, t, impl.split("_", 1)[1])[0]
    for _ in range(3):
        flush()
        step()
        flush()
    torch.cuda.synchronize()


def parse(path):
    rows = []
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    for r in csv.DictReader(lines):
        rows.append(r)
    kern = {}
    order = []
    for r in rows:
        key = r["ID"]
        if key not in kern:
            kern[key] = {"name": r["Kernel Name"]}
            order.append(key)
        val = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "usecond": 1e3,
                 "nsecond": 1, "msecond": 1e6}.get(unit, 1)
        kern[key][r["Metric Name"]] = val * scale
    seq = [kern[k] for k in order]
    is_flush = ["reduce_kernel" in s["name"] for s in seq]
    groups, cur = [], []
    for i, s in enumerate(seq):
        if is_flush[i]:
            if cur:
                groups.append((cur, i))
            cur = []
        else:
            cur.append(s)
    ks, after = groups[-1]
    # the flush kernel(s) right after the step: their DRAM writes are the step's write-backs
    wb = 0.0
    j = after
    while j < len(seq) and is_flush[j]:
        wb += seq[j].get("dram__bytes_write.sum", 0.0)
        j += 1
    rd = sum(s.get("dram__bytes_read.sum", 0.0) for s in ks)
    wr = sum(s.get("dram__bytes_write.sum", 0.0) for s in ks)
    ns = sum(s.get("gpu__time_duration.sum", 0.0) for s in ks)
    return {"kernels": [s["name"][:80] for s in ks], "dram_read": int(rd), "dram_write": int(wr),
            "writeback_after": int(wb), "dram_total": int(rd + wr + wb), "kernel_ns": int(ns)}


if __name__ == "__main__":
    if sys.argv[1] == "run":
        # optional variant=0x.. (ff_set_variant: A/B of kernel variants, e.g. 0x80 = no discard)
        var = next((int(a.split("=")[1], 0) for a in sys.argv[4:] if a.startswith("variant=")), 0)
        if var:
            from paper_2512_12949_b200 import _native

            _native.load().ff_set_variant(var)
        run(sys.argv[2], sys.argv[3])
    else:
        print(json.dumps(parse(sys.argv[2])))
