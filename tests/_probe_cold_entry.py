# Diagnostics: event time of (a) the chain kernel exiting at entry (debug bit 28) and
# (b) an empty probe kernel of the same launch shape, after a full L2 flush (256 MiB),
# a small flush (2 MiB, L2 stays warm) and no flush: is the entry latency a cold-L2
# (code / parameter fetch) effect?
import sys, ctypes
import torch
sys.path.insert(0, '.')
import bench
from paper_2512_12949_b200 import _native as nat, runtime
lib = nat.load()
dev = torch.device('cuda', 0)
big = torch.empty(64 << 20, dtype=torch.float32, device=dev)
small = torch.empty(512 << 10, dtype=torch.float32, device=dev)
name = 'llama1b'
kind, act, m, n, k, l, _ = bench.WORKLOADS[name]
graph = bench.graph_of(name)
t = bench.make_device_inputs(kind, m, n, k, l, seed=1, device=dev)
cfg = runtime.lower(graph, None, 148, 'pair')
out = torch.empty((m, l), dtype=torch.bfloat16, device=dev)
pst = torch.zeros(4096, dtype=torch.int64, device=dev)
stream = torch.cuda.current_stream().cuda_stream

def chain():
    runtime.launch(graph, cfg, t, out=out)

def probe():
    assert lib.ff_launch_probe(ctypes.c_void_p(pst.data_ptr()), 128, 200 * 1024, 4, 1, ctypes.c_void_p(stream)) == 0

def timed(fn, fl, n=200):
    for _ in range(5): fn()
    ts = []
    for _ in range(n):
        if fl is not None: fl.add_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return sum(ts) / n, ts[n // 2]

for label, mode in [('chain full run', 0), ('chain exit-at-entry', 1 << 28)]:
    lib.ff_set_debug_mode(mode)
    for fl_name, fl in [('full flush', big), ('2 MiB flush', small), ('no flush', None)]:
        print(f"{label:22s} {fl_name:12s} mean %.2f us median %.2f" % timed(chain, fl), flush=True)
lib.ff_set_debug_mode(0)
for fl_name, fl in [('full flush', big), ('2 MiB flush', small), ('no flush', None)]:
    print(f"{'probe kernel':22s} {fl_name:12s} mean %.2f us median %.2f" % timed(probe, fl), flush=True)
