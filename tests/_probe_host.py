# Diagnostics: host cost per launch (Python runtime.launch and the raw C ABI call), GPU kept busy.
import sys, time, ctypes, torch
sys.path.insert(0, '.')
import bench
from paper_2512_12949_b200 import runtime, _native as nat
name = "llama1b"
kind, act, m, n, k, l, _ = bench.WORKLOADS[name]
t = bench.make_device_inputs(kind, m, n, k, l, 3, "cuda")
g = bench.graph_of(name)
cfg = runtime.lower(g, None, 148, "pair")
out = torch.empty((m, l), dtype=torch.bfloat16, device="cuda")
for _ in range(5): runtime.launch(g, cfg, t, out=out)
torch.cuda.synchronize()
hs = []
for i in range(200):
    t0 = time.perf_counter(); runtime.launch(g, cfg, t, out=out); hs.append(time.perf_counter() - t0)
torch.cuda.synchronize()
print(f"runtime.launch host time: median {sorted(hs)[100]*1e6:.1f} us")
lib = nat.load(); ch = runtime.chain_desc(g)
ws_bytes = lib.ff_chain_workspace_bytes(ctypes.byref(ch), ctypes.byref(cfg))
ws = runtime._workspace(ws_bytes, out.device, torch.cuda.current_stream())
tp = nat.Tensors(t["A"].data_ptr(), t["B0"].data_ptr(), t["B1"].data_ptr(), t["D"].data_ptr(), out.data_ptr())
s = torch.cuda.current_stream().cuda_stream
hs = []
for i in range(200):
    t0 = time.perf_counter(); lib.ff_chain_launch(ctypes.byref(ch), ctypes.byref(cfg), ctypes.byref(tp), ws.data_ptr(), ws_bytes, s); hs.append(time.perf_counter() - t0)
torch.cuda.synchronize()
print(f"ff_chain_launch (ctypes) host time: median {sorted(hs)[100]*1e6:.1f} us")
# back-to-back device time per launch
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record()
for i in range(100): lib.ff_chain_launch(ctypes.byref(ch), ctypes.byref(cfg), ctypes.byref(tp), ws.data_ptr(), ws_bytes, s)
b.record(); torch.cuda.synchronize()
print(f"back-to-back: {a.elapsed_time(b)*10:.1f} us per launch (warm L2)")
# CUDA graph of 10 launches
gr = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    runtime.launch(g, cfg, t, out=out)
    torch.cuda.synchronize()
    try:
        with torch.cuda.graph(gr, stream=st):
            for i in range(10): runtime.launch(g, cfg, t, out=out, stream=st)
        ok = True
    except Exception as e:
        ok = False; print("graph capture failed:", repr(e)[:200])
if ok:
    for _ in range(3): gr.replay()
    torch.cuda.synchronize()
    a.record()
    for _ in range(10): gr.replay()
    b.record(); torch.cuda.synchronize()
    print(f"graph replay: {a.elapsed_time(b)*10:.1f} us per launch")
    ref = out.clone(); runtime.launch(g, cfg, t, out=out); torch.cuda.synchronize()
    print("graph output == eager output:", torch.equal(ref, out))
