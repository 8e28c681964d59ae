# Diagnostics: back-to-back launch time of explicit pair configs / debug modes.
import sys, ctypes, torch
sys.path.insert(0, '.')
sys.argv = sys.argv[:1] + ['x']
exec(open('tests/_probe_kernel.py').read().split("for pack in")[0])
def b2b(m,n,k,l,act,g,cfg,mode=0,iters=20):
    A,B,B1,D,E,ch,kc,ws,t = setup(m,n,k,l,act,g,cfg,2)
    lib.ff_set_debug_mode(mode)
    f=lambda: nat.check(lib.ff_chain_launch(ctypes.byref(ch),ctypes.byref(kc),ctypes.byref(t),ws.data_ptr(),ws.numel(),None))
    for _ in range(5): f()
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(iters): f()
    e.record(); torch.cuda.synchronize()
    us = s.elapsed_time(e)/iters*1e3
    lib.ff_set_debug_mode(0)
    Er, _ = ref(A,B,D,act,B1 if g else None)
    err=((E.float()-Er).abs().max()/Er.abs().max()).item()
    kc2 = nat.KernelConfig(); kc2.ring,kc2.n_splits,kc2.nb,kc2.lb,kc2.exchange = kc.ring,kc.n_splits,kc.nb,kc.lb,2
    fl = 2.0*m*k*n*(2 if g else 1) + 2.0*m*n*l
    print(f"m{m} n{n} k{k} l{l} g{int(g)} cfg={cfg} mode={mode}: {us:7.1f} us  {fl/us/1e6:7.1f} TF/s  err {err:.1e}", flush=True)
LL=(512,8192,2048,2048,2,True); G6=(512,16384,4096,4096,1,False); OPT=(4096,8192,2048,2048,1,False); G2=(512,3072,768,768,3,False)
for cfg in [None,(8,4,128,256),(8,8,128,256),(8,2,128,256)]:
    for mode in ([0, (5<<8)] if cfg is None else [0]):
        b2b(*LL,cfg,mode)
for cfg in [None,(16,2,256,256),(16,4,256,256)]:
    for mode in ([0,(6<<8),(7<<8),(9<<8),(12<<8)] if cfg is None else [0]):
        b2b(*G6,cfg,mode)
for cfg in [None,(8,1,256,256),(8,2,256,256)]:
    b2b(*OPT,cfg,0)
for cfg in [None,(3,4,256,256),(3,8,256,256),(3,16,256,256)]:
    try: b2b(*G2,cfg,0)
    except Exception as ex: print("fail", cfg, ex)
