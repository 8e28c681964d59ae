# Diagnostics: small chains (GPT-2s, conv C5) per exchange, back-to-back and cold.
import sys, ctypes, torch, statistics
sys.path.insert(0, '.')
sys.argv = sys.argv[:1] + ['x']
exec(open('tests/_probe_kernel.py').read().split("for pack in")[0])
flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device='cuda')
def go(m,n,k,l,act,g,x,cfg=None):
    A,B,B1,D,E,ch,kc,ws,t = setup(m,n,k,l,act,g,cfg,x)
    f=lambda: nat.check(lib.ff_chain_launch(ctypes.byref(ch),ctypes.byref(kc),ctypes.byref(t),ws.data_ptr(),ws.numel(),None))
    for _ in range(5): f()
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(20): f()
    e.record(); torch.cuda.synchronize(); b2b=s.elapsed_time(e)/20*1e3
    ts=[]
    for i in range(23):
        flush_buf.add_(1.0); s.record(); f(); e.record(); torch.cuda.synchronize()
        if i>=3: ts.append(s.elapsed_time(e)*1e3)
    Er,_=ref(A,B,D,act,B1 if g else None)
    err=((E.float()-Er).abs().max()/Er.abs().max()).item()
    print(f"m{m} n{n} k{k} l{l} x{x} {kc.as_dict()}: b2b {b2b:6.1f} us cold {statistics.median(ts):6.1f} us err {err:.1e}", flush=True)
for shape in [(512,3072,768,768,3,False),(3136,64,576,256,1,False),(3136,512,640,256,1,False)]:
    for x in (0,1,2):
        try: go(*shape, x)
        except Exception as ex: print("fail", shape, x, ex)
