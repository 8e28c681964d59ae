# Diagnostics: host cost of one launch through runtime.launch vs a direct C-ABI call
# with prebuilt descriptors (the GPU runs far behind; 400 calls, perf_counter).
import sys, time, ctypes
import torch
sys.path.insert(0, '.')
import bench
from paper_2512_12949_b200 import _native as nat, runtime
dev = torch.device('cuda', 0)
name = 'llama1b'
kind, act, m, n, k, l, _ = bench.WORKLOADS[name]
graph = bench.graph_of(name)
t = bench.make_device_inputs(kind, m, n, k, l, seed=1, device=dev)
cfg = runtime.lower(graph, None, 148, 'pair')
out = torch.empty((m, l), dtype=torch.bfloat16, device=dev)
lib = nat.load()
s = torch.cuda.current_stream()
runtime.launch(graph, cfg, t, out=out); torch.cuda.synchronize()
ch = runtime.chain_desc(graph, 'bf16')
ws_bytes = lib.ff_chain_workspace_bytes(ctypes.byref(ch), ctypes.byref(cfg))
ws = runtime._workspace(ws_bytes, dev, s)
tp = nat.Tensors(t['A'].data_ptr(), t['B0'].data_ptr(), t['B1'].data_ptr(), t['D'].data_ptr(), out.data_ptr())
args = (ctypes.byref(ch), ctypes.byref(cfg), ctypes.byref(tp), ws.data_ptr(), ws_bytes, s.cuda_stream)
def host_us(fn, n=400):
    torch.cuda.synchronize(); c0 = time.perf_counter()
    for _ in range(n): fn()
    c1 = time.perf_counter(); torch.cuda.synchronize()
    return (c1 - c0) * 1e6 / n
for _ in range(2):
    print('runtime.launch       %.1f us/call' % host_us(lambda: runtime.launch(graph, cfg, t, out=out)))
    print('ff_chain_launch      %.1f us/call' % host_us(lambda: lib.ff_chain_launch(*args)))
    print('torch empty kernel   %.1f us/call' % host_us(lambda: out.zero_()))
