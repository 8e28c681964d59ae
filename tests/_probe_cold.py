# Diagnostics: kernel time with L2 flushed before every launch (as bench.py), per debug mode.
import sys, ctypes, torch, statistics
sys.path.insert(0, '.')
MODES = [int(x) for x in sys.argv[1:]] or [0]
sys.argv = sys.argv[:1] + ['x']
exec(open('tests/_probe_kernel.py').read().split("for pack in")[0])
flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device='cuda')
def cold(m,n,k,l,act,g,mode,steps=30):
    A,B,B1,D,E,ch,kc,ws,t = setup(m,n,k,l,act,g,None,2)
    lib.ff_set_debug_mode(mode)
    f=lambda: nat.check(lib.ff_chain_launch(ctypes.byref(ch),ctypes.byref(kc),ctypes.byref(t),ws.data_ptr(),ws.numel(),None))
    ts=[]
    for i in range(steps+3):
        flush_buf.add_(1.0)
        s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
        s.record(); f(); e.record(); torch.cuda.synchronize()
        if i >= 3: ts.append(s.elapsed_time(e)*1e3)
    lib.ff_set_debug_mode(0)
    Er, _ = ref(A,B,D,act,B1 if g else None)
    err=((E.float()-Er).abs().max()/Er.abs().max()).item()
    fl = 2.0*m*k*n*(2 if g else 1) + 2.0*m*n*l
    md = statistics.median(ts)
    print(f"m{m} n{n} k{k} l{l} g{int(g)} mode={mode}: cold median {md:7.1f} us  {fl/md/1e6:7.1f} TF/s  err {err:.1e}", flush=True)
for shape in [(512,8192,2048,2048,2,True),(512,16384,4096,4096,1,False),(4096,8192,2048,2048,1,False)]:
    for mode in MODES:
        cold(*shape, mode)
