import sys, torch, ctypes
sys.path.insert(0, '.')
from paper_2512_12949_b200 import _native as nat
lib = nat.load()
def bench(m,n,k,l,g,cfg=None,iters=20,act=1):
    A=(torch.rand(m,k,device='cuda')*2-1).bfloat16(); B=(torch.rand(k,n,device='cuda')*2-1).bfloat16()
    B1=(torch.rand(k,n,device='cuda')*2-1).bfloat16() if g else B
    D=(torch.rand(n,l,device='cuda')*2-1).bfloat16(); E=torch.zeros(m,l,device='cuda',dtype=torch.bfloat16)
    ch=nat.ChainDesc(1 if g else 0, 2 if g else act, m,n,k,l,2); kc=nat.KernelConfig()
    if cfg is None: nat.check(lib.ff_auto_config(ctypes.byref(ch),148,ctypes.byref(kc)))
    else: kc.ring,kc.n_splits,kc.nb,kc.lb=cfg
    ws=torch.empty(max(4,lib.ff_chain_workspace_bytes(ctypes.byref(ch),ctypes.byref(kc))//4),device='cuda')
    t=nat.Tensors(A.data_ptr(),B.data_ptr(),B1.data_ptr(),D.data_ptr(),E.data_ptr())
    f=lambda: nat.check(lib.ff_chain_launch(ctypes.byref(ch),ctypes.byref(kc),ctypes.byref(t),ws.data_ptr(),ws.numel()*4,None))
    for _ in range(3): f()
    torch.cuda.synchronize(); s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): f()
    e.record(); torch.cuda.synchronize(); ms=s.elapsed_time(e)/iters
    fl=2*m*k*n*(2 if g else 1)+2*m*n*l
    print(f"m{m} n{n} k{k} l{l} g{int(g)} cfg{cfg} ctas {kc.grid_ctas if cfg is None else '-'} {ms*1e3:8.1f}us {fl/ms/1e9:7.1f} TF/s", flush=True)
mode = sys.argv[1] if len(sys.argv)>1 else 'sweep'
if mode == 'one':
    bench(512,16384,4096,4096,False,None,iters=2)
    sys.exit()
# GEMM0-dominated: tiny L, no ring
for cfg in [(1,1,128,256),(1,2,128,256),(1,4,128,256),(1,8,128,256),(1,16,128,256),(1,32,128,256)]:
    bench(512,16384,4096,256,False,cfg)
# ring cost: L = ring*256, K small so GEMM1 dominates
for r in [1,2,4,8,16]:
    bench(512,16384,256,256*r,False,(r,max(1,32//r),128,256))
for cfg in [(16,1,128,256),(16,2,128,256),(16,2,64,256),(8,4,128,256) ]:
    try: bench(512,16384,4096,4096,False,cfg)
    except Exception as ex: print(cfg, ex)
