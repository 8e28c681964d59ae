import sys, torch, ctypes
sys.path.insert(0, '.')
from paper_2512_12949_b200 import _native as nat
lib = nat.load()
torch.manual_seed(0)
def run(m,n,k,l,cfg,gated=False):
    A=(torch.rand(m,k,device='cuda')*2-1).bfloat16(); B=(torch.rand(k,n,device='cuda')*2-1).bfloat16()
    B1=(torch.rand(k,n,device='cuda')*2-1).bfloat16() if gated else B
    D=(torch.rand(n,l,device='cuda')*2-1).bfloat16(); E=torch.zeros(m,l,device='cuda',dtype=torch.bfloat16)
    ch=nat.ChainDesc(1 if gated else 0, 2 if gated else 1, m,n,k,l,2); kc=nat.KernelConfig(); kc.ring,kc.n_splits,kc.nb,kc.lb=cfg
    ws=torch.empty(max(4,lib.ff_chain_workspace_bytes(ctypes.byref(ch),ctypes.byref(kc))//4),device='cuda')
    t=nat.Tensors(A.data_ptr(),B.data_ptr(),B1.data_ptr(),D.data_ptr(),E.data_ptr())
    nat.check(lib.ff_chain_launch(ctypes.byref(ch),ctypes.byref(kc),ctypes.byref(t),ws.data_ptr(),ws.numel()*4,None))
    torch.cuda.synchronize()
    c = A.float()@B.float()
    c = torch.nn.functional.silu(c)*(A.float()@B1.float()) if gated else torch.relu(c)
    Er = c.bfloat16().float()@D.float()
    err=(E.float()-Er).abs()
    scale=Er.abs().max()
    tot=(err.max()/scale).item()
    lb=cfg[3]
    percol=[round((err[:, j*lb:(j+1)*lb].max()/scale).item(),3) for j in range(l//lb)]
    perrow=[round((err[i*128:(i+1)*128].max()/scale).item(),3) for i in range((m+127)//128)]
    print(f"m{m} n{n} k{k} l{l} cfg{cfg} g{int(gated)} err {tot:.3e} per-ring-member {percol} per-mtile {perrow}", flush=True)
for steps in [1,2,3]:
    run(128, 4*128*steps, 256, 1024, (4,1,128,256))
for steps in [1,2,3]:
    run(128, 4*64*steps, 256, 1024, (4,1,64,256))
for steps in [1,2,3]:
    run(128, 4*64*steps, 256, 1024, (4,1,64,256), gated=True)
for G in [2,3,4,5,6,8]:
    run(128, G*128*3, 128, 256*G, (G,1,128,256))
for G in [4,8]:
    run(128, G*128*3, 128, 128*G, (G,1,128,128))
