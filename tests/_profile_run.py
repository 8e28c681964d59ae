"""Launch sequence for ncu (no torch flush: ncu's --cache-control all flushes
between kernels).  Per workload: 3 fused launches, then 2 cuBLAS unfused chains
(GEMM -> act(/gate) -> GEMM).  tests/_ncu_summary.py turns the CSV into
profiles/ncu_summary.json.  Run with FF_NO_COOPERATIVE=1 under ncu."""
import sys, torch
sys.path.insert(0, '.')
import bench
from paper_2512_12949_b200 import runtime
names = sys.argv[1:] or ["llama1b"]
for name in names:
    kind, act, m, n, k, l, _ = bench.WORKLOADS[name]
    t = bench.make_device_inputs(kind, m, n, k, l, 3, "cuda")
    g = bench.graph_of(name)
    # the transport bench.py's ProfileBestFromList picks for the workload
    cfg = runtime.lower(g, None, 148, {"gpt2s": "dsm"}.get(name, "auto"))
    out = torch.empty((m, l), dtype=torch.bfloat16, device="cuda")
    for i in range(3):
        runtime.launch(g, cfg, t, out=out)
    torch.cuda.synchronize()
    f = torch.nn.functional
    for i in range(2):
        if kind == "gated_ffn":
            r = (f.silu(t["A"] @ t["B0"]) * (t["A"] @ t["B1"])) @ t["D"]
        elif act == "gelu":
            r = f.gelu(t["A"] @ t["B"], approximate="tanh") @ t["D"]
        else:
            r = torch.relu(t["A"] @ t["B"]) @ t["D"]
    torch.cuda.synchronize()
    print(name, "done", runtime.exchange_name(cfg), flush=True)
