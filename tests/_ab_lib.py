# A/B timing of two builds of the library (FF_CHAIN_LIB selects one per process):
# cold-L2 CUDA-event times, mean and median of 300 launches per chain.
import sys
import torch
sys.path.insert(0, '.')
import bench
import os
from paper_2512_12949_b200 import _native as nat, runtime
if os.environ.get('FF_DBG'):
    nat.load().ff_set_debug_mode(int(os.environ['FF_DBG'], 0))
dev = torch.device('cuda', 0)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
for name in sys.argv[1:]:
    kind, act, m, n, k, l, _ = bench.WORKLOADS[name]
    graph = bench.graph_of(name)
    t = bench.make_device_inputs(kind, m, n, k, l, seed=1, device=dev)
    cfg = runtime.lower(graph, None, 148, 'dsm' if name == 'gpt2s' else 'pair')
    out = torch.empty((m, l), dtype=torch.bfloat16, device=dev)
    for _ in range(5): runtime.launch(graph, cfg, t, out=out)
    ts = []
    for _ in range(300):
        flush.add_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); runtime.launch(graph, cfg, t, out=out); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    print(f"{name:10s} mean {sum(ts)/len(ts):7.2f} us  median {ts[150]:7.2f}  p10 {ts[30]:7.2f}", flush=True)
