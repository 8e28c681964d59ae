# Diagnostics: cold-L2 event time of explicit (ring, n_splits, nb, lb) configs per exchange.
import sys, ctypes, torch
sys.path.insert(0, '.')
ARGV = list(sys.argv)
sys.argv = sys.argv[:1] + ['x']
exec(open('tests/_probe_kernel.py').read().split("for pack in")[0])
flush_buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device='cuda')
def timed(shape, cfg, xchg):
    try:
        A,B,B1,D,E,ch,kc,ws,t = setup(*shape,cfg,xchg)
    except Exception as e:
        return None, str(e)[:60]
    f=lambda: nat.check(lib.ff_chain_launch(ctypes.byref(ch),ctypes.byref(kc),ctypes.byref(t),ws.data_ptr(),ws.numel(),None))
    try:
        for _ in range(3): f()
    except Exception as e:
        return None, str(e)[:60]
    ts=[]
    for it in range(11):
        flush_buf.add_(1.0)
        a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b)*1e3)
    Er,_ = ref(A,B,D,shape[4],B1 if shape[5] else None)
    err=((E.float()-Er).abs().max()/Er.abs().max()).item()
    return sorted(ts)[5], f"err {err:.1e} {kc.as_dict()}"
shape = (512,3072,768,768,3,False)
for xchg in (0, 1):
    for cfg in [None, (3,8,128,256), (3,4,128,256), (3,2,128,256), (3,8,64,256), (3,16,64,256), (6,8,64,128), (6,4,128,128), (6,8,128,128), (12,4,64,64), (12,2,128,64), (6,2,128,128)]:
        ms, info = timed(shape, cfg, xchg)
        print(f"x{xchg} cfg {cfg}: {ms if ms is None else round(ms,1)} us {info}", flush=True)
for cfg in [None, (3,4,256,256), (3,2,256,256), (3,1,256,256)]:
    ms, info = timed(shape, cfg, 2)
    print(f"x2 cfg {cfg}: {ms if ms is None else round(ms,1)} us {info}", flush=True)
