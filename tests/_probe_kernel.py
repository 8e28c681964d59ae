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
def run(m,n,k,l,act=1,gated=False,cfg=None):
    A=(torch.rand(m,k,device='cuda')*2-1).bfloat16()
    B=(torch.rand(k,n,device='cuda')*2-1).bfloat16()
    B1=(torch.rand(k,n,device='cuda')*2-1).bfloat16() if gated else None
    D=(torch.rand(n,l,device='cuda')*2-1).bfloat16()
    E=torch.zeros(m,l,device='cuda',dtype=torch.bfloat16)
    Cdbg=torch.zeros(m,n,device='cuda',dtype=torch.bfloat16)
    ch=nat.ChainDesc(1 if gated else 0, 2 if gated else act, m,n,k,l,2)
    kc=nat.KernelConfig()
    if cfg is None:
        rc=lib.ff_auto_config(ctypes.byref(ch),148,ctypes.byref(kc)); nat.check(rc)
    else:
        kc.ring,kc.n_splits,kc.nb,kc.lb=cfg
    ws_bytes=lib.ff_chain_workspace_bytes(ctypes.byref(ch),ctypes.byref(kc)) or 16
    ws=torch.empty(ws_bytes//4+4,device='cuda',dtype=torch.float32)
    t=nat.Tensors(A.data_ptr(),B.data_ptr(),B1.data_ptr() if gated else None,D.data_ptr(),E.data_ptr())
    rc=lib.ff_chain_launch_debug(ctypes.byref(ch),ctypes.byref(kc),ctypes.byref(t),ws.data_ptr(),ws.numel()*4,Cdbg.data_ptr(),None)
    nat.check(rc)
    torch.cuda.synchronize()
    Er, Cr = ref(A,B,D,act,B1)
    cerr=((Cdbg.float()-Cr.float()).abs().max()/Cr.float().abs().max()).item()
    eerr=((E.float()-Er).abs().max()/Er.abs().max()).item()
    print(f"m{m} n{n} k{k} l{l} act{act} gated{gated} cfg{kc.as_dict()} C_err {cerr:.3e} E_err {eerr:.3e}", flush=True)
    return cerr, eerr
cases=[(128,128,64,64,0,False,(1,1,128,64)),(128,256,128,256,1,False,(1,1,128,256)),(128,512,256,512,1,False,(2,1,128,256)),
       (256,1024,256,1024,1,False,(4,1,128,256)),(256,1024,256,1024,1,False,(4,2,128,256)),(200,768,256,768,3,False,None),
       (256,1024,512,512,2,True,(2,1,64,256)),(512,3072,768,768,3,False,None),(512,8192,2048,2048,2,True,None),(512,16384,4096,4096,1,False,None)]
for c in cases:
    try:
        run(*c)
    except Exception as e:
        print("FAIL", c, repr(e), flush=True)
# timing
for (m,n,k,l,act,g) in [(512,16384,4096,4096,1,False),(512,8192,2048,2048,2,True),(4096,8192,2048,2048,1,False)]:
    A=(torch.rand(m,k,device='cuda')*2-1).bfloat16(); B=(torch.rand(k,n,device='cuda')*2-1).bfloat16()
    B1=(torch.rand(k,n,device='cuda')*2-1).bfloat16() if g else B
    D=(torch.rand(n,l,device='cuda')*2-1).bfloat16(); E=torch.zeros(m,l,device='cuda',dtype=torch.bfloat16)
    ch=nat.ChainDesc(1 if g else 0, act, m,n,k,l,2); kc=nat.KernelConfig(); nat.check(lib.ff_auto_config(ctypes.byref(ch),148,ctypes.byref(kc)))
    ws=torch.empty(max(1,lib.ff_chain_workspace_bytes(ctypes.byref(ch),ctypes.byref(kc))//4),device='cuda')
    t=nat.Tensors(A.data_ptr(),B.data_ptr(),B1.data_ptr(),D.data_ptr(),E.data_ptr())
    f=lambda: nat.check(lib.ff_chain_launch(ctypes.byref(ch),ctypes.byref(kc),ctypes.byref(t),ws.data_ptr(),ws.numel()*4,None))
    for _ in range(3): f()
    torch.cuda.synchronize(); s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20): f()
    e.record(); torch.cuda.synchronize(); ms=s.elapsed_time(e)/20
    fl=2*m*k*n*(2 if g else 1)+2*m*n*l
    # cublas unfused
    def cub():
        c=A@B
        if g: c=torch.nn.functional.silu(c)*(A@B1)
        else: c=torch.relu(c)
        return c@D
    for _ in range(3): cub()
    torch.cuda.synchronize(); s.record()
    for _ in range(20): cub()
    e.record(); torch.cuda.synchronize(); ms2=s.elapsed_time(e)/20
    print(f"TIME m{m} n{n} k{k} l{l} g{g} cfg {kc.as_dict()} fused {ms*1e3:.1f}us {fl/ms/1e9:.1f} TF/s | cublas {ms2*1e3:.1f}us {fl/ms2/1e9:.1f} TF/s", flush=True)
