# Diagnostics: helper-pair state across launches (zone / counters zero after a launch).
import sys, ctypes, torch
sys.path.insert(0, '.')
sys.argv = sys.argv[:1] + ['x']
exec(open('tests/_probe_kernel.py').read().split("for pack in")[0])
from paper_2512_12949_b200 import runtime
for shape in [(512,3072,768,768,3,False),(512,16384,4096,4096,1,False),(512,8192,2048,2048,2,True)]:
    A,B,B1,D,E,ch,kc,ws,t = setup(*shape,None,2)
    f=lambda: nat.check(lib.ff_chain_launch(ctypes.byref(ch),ctypes.byref(kc),ctypes.byref(t),ws.data_ptr(),ws.numel(),None))
    print(shape[:4], kc.as_dict(), flush=True)
    for it in range(3):
        E.zero_(); f(); torch.cuda.synchronize()
        Er, _ = ref(A,B,D,shape[4],B1 if shape[5] else None)
        err=((E.float()-Er).abs().max()/Er.abs().max()).item()
        cnt = ws[(1<<20):(1<<20)+(256<<10)].view(torch.int32)
        zone = ws[(1<<20)+(256<<10):(1<<20)+(256<<10)+(32<<20)].view(torch.float32)
        print(f"  launch {it}: err {err:.2e} nonzero counters {int((cnt!=0).sum())} zone nonzero {int((zone!=0).sum())}", flush=True)
