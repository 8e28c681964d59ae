import sys, time, torch, ctypes
sys.path.insert(0, '.')
from paper_2512_12949_b200 import _native as nat
lib = nat.load()
print(lib.ff_version())
torch.manual_seed(0)
def ref(A,B,D,act,B1=None):
    a=A.float(); c=a@B.float()
    if B1 is not None: c = torch.nn.functional.silu(c)*(a@B1.float())
    elif act==1: c=torch.relu(c)
    elif act==2: c=torch.nn.functional.silu(c)
    elif act==3: c=torch.nn.functional.gelu(c, approximate='tanh')
    cb=c.bfloat16()
    return (cb.float()@D.float()), cb
PACK=[True]
def setup(m,n,k,l,act,gated,cfg,xchg):
    A=(torch.rand(m,k,device='cuda')*2-1).bfloat16()
    if gated and PACK[0]:
        B01=(torch.rand(2,k,n,device='cuda')*2-1).bfloat16(); B, B1 = B01[0], B01[1]
    else:
        B=(torch.rand(k,n,device='cuda')*2-1).bfloat16()
        B1=(torch.rand(k,n,device='cuda')*2-1).bfloat16() if gated else B
    D=(torch.rand(n,l,device='cuda')*2-1).bfloat16()
    E=torch.zeros(m,l,device='cuda',dtype=torch.bfloat16)
    ch=nat.ChainDesc(1 if gated else 0, 2 if gated else act, m,n,k,l,2)
    kc=nat.KernelConfig()
    if cfg is None:
        nat.check(lib.ff_auto_config_ex(ctypes.byref(ch),148,xchg,ctypes.byref(kc)))
    else:
        kc.ring,kc.n_splits,kc.nb,kc.lb=cfg; kc.exchange=xchg
    ws_bytes=lib.ff_chain_workspace_bytes(ctypes.byref(ch),ctypes.byref(kc)) or 256
    ws=torch.zeros(ws_bytes,device='cuda',dtype=torch.uint8)
    t=nat.Tensors(A.data_ptr(),B.data_ptr(),B1.data_ptr(),D.data_ptr(),E.data_ptr())
    return A,B,B1,D,E,ch,kc,ws,t
def run(m,n,k,l,act=1,gated=False,cfg=None,xchg=1):
    A,B,B1,D,E,ch,kc,ws,t = setup(m,n,k,l,act,gated,cfg,xchg)
    Cdbg=torch.zeros(m,n,device='cuda',dtype=torch.bfloat16)
    nat.check(lib.ff_chain_launch_debug(ctypes.byref(ch),ctypes.byref(kc),ctypes.byref(t),ws.data_ptr(),ws.numel(),Cdbg.data_ptr(),None))
    torch.cuda.synchronize()
    Er, Cr = ref(A,B,D,act,B1 if gated else None)
    cerr=((Cdbg.float()-Cr.float()).abs().max()/Cr.float().abs().max()).item()
    eerr=((E.float()-Er).abs().max()/Er.abs().max()).item()
    # second launch (epoch flags / workspace reuse)
    nat.check(lib.ff_chain_launch(ctypes.byref(ch),ctypes.byref(kc),ctypes.byref(t),ws.data_ptr(),ws.numel(),None))
    torch.cuda.synchronize()
    eerr2=((E.float()-Er).abs().max()/Er.abs().max()).item()
    ok = "ok " if max(eerr,eerr2) < 1e-2 else "BAD"
    print(f"{ok} x{xchg} m{m} n{n} k{k} l{l} act{act} g{int(gated)} cfg{cfg} C_err {cerr:.2e} E_err {eerr:.2e} {eerr2:.2e}", flush=True)
cases=[(128,128,64,64,0,False,(1,1,128,64)),(128,256,128,256,1,False,(1,1,128,256)),(128,512,256,512,1,False,(2,1,128,256)),
       (256,1024,256,1024,1,False,(4,1,128,256)),(256,1024,256,1024,1,False,(4,2,128,256)),(200,768,256,768,3,False,None),
       (256,1024,512,512,2,True,(2,1,64,256)),(128,3072,128,2048,1,False,(8,1,128,256)),(128,1536,256,1024,1,False,(4,1,64,256)),
       (3136,64,576,256,1,False,None),(512,3072,768,768,3,False,None),(512,8192,2048,2048,2,True,None),(512,16384,4096,4096,1,False,None),
       (1024,8192,2048,2048,1,False,None)]
pair_cases=[(256,256,128,256,1,False,(1,1,256,256)),(256,512,128,512,1,False,(2,1,256,256)),(512,1024,256,1024,1,False,(4,1,256,256)),
            (512,2048,256,1024,1,False,(4,2,256,256)),(256,512,256,256,2,True,(1,1,128,256)),(256,1024,256,512,2,True,(2,2,128,256)),
            (200,1536,256,768,3,False,(3,2,256,256)),(3136,512,640,256,1,False,None),(512,3072,768,768,3,False,None),
            (512,8192,2048,2048,2,True,None),(512,16384,4096,4096,1,False,None),(1024,8192,2048,2048,1,False,None)]
for pack in (True, False):
    PACK[0]=pack
    for c in pair_cases:
        if not pack and not c[5]: continue
        try:
            run(*c, xchg=2)
        except Exception as e:
            print("FAIL", 2, c, repr(e), flush=True)
PACK[0]=True
for xchg in ([] if len(sys.argv) > 1 else (1,0)):
    for c in cases:
        try:
            run(*c, xchg=xchg)
        except Exception as e:
            print("FAIL", xchg, c, repr(e), flush=True)
def bench(m,n,k,l,g,act,xchg,cfg=None,iters=20):
    A,B,B1,D,E,ch,kc,ws,t = setup(m,n,k,l,act,g,cfg,xchg)
    f=lambda: nat.check(lib.ff_chain_launch(ctypes.byref(ch),ctypes.byref(kc),ctypes.byref(t),ws.data_ptr(),ws.numel(),None))
    for _ in range(3): f()
    torch.cuda.synchronize(); s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): f()
    e.record(); torch.cuda.synchronize(); ms=s.elapsed_time(e)/iters
    fl=2*m*k*n*(2 if g else 1)+2*m*n*l
    return ms, fl, kc
for (m,n,k,l,act,g) in [(512,16384,4096,4096,1,False),(512,8192,2048,2048,2,True),(512,3072,768,768,3,False),(4096,8192,2048,2048,1,False),(3136,64,576,256,1,False)]:
    line=f"TIME m{m} n{n} k{k} l{l} g{int(g)}:"
    for xchg in (2,1,0):
        try:
            ms,fl,kc=bench(m,n,k,l,g,act,xchg)
            line+=f" | x{xchg} {ms*1e3:.1f}us {fl/ms/1e9:.0f}TF/s r{kc.ring} s{kc.n_splits} rings{kc.rings}"
        except Exception as ex:
            line+=f" | x{xchg} ERR {ex}"
    A=(torch.rand(m,k,device='cuda')*2-1).bfloat16(); B=(torch.rand(k,n,device='cuda')*2-1).bfloat16(); D=(torch.rand(n,l,device='cuda')*2-1).bfloat16()
    B1=(torch.rand(k,n,device='cuda')*2-1).bfloat16()
    def cub():
        c=A@B
        c = torch.nn.functional.silu(c)*(A@B1) if g else torch.relu(c)
        return c@D
    for _ in range(3): cub()
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(20): cub()
    e.record(); torch.cuda.synchronize(); ms2=s.elapsed_time(e)/20
    fl=2*m*k*n*(2 if g else 1)+2*m*n*l
    print(line + f" | cublas {ms2*1e3:.1f}us {fl/ms2/1e9:.0f}TF/s", flush=True)
