# Diagnostics: GPU-side gap between two back-to-back launches (globaltimer stamps).
import sys, ctypes, torch
sys.path.insert(0, '.')
sys.argv = sys.argv[:1] + ['x']
exec(open('tests/_probe_kernel.py').read().split("for pack in")[0])
ST = 32
for shape in [(512,8192,2048,2048,2,True),(512,16384,4096,4096,1,False)]:
    A,B,B1,D,E,ch,kc,ws,t = setup(*shape,None,2)
    f=lambda: nat.check(lib.ff_chain_launch(ctypes.byref(ch),ctypes.byref(kc),ctypes.byref(t),ws.data_ptr(),ws.numel(),None))
    bufs=[torch.zeros(kc.grid_ctas*ST+64, dtype=torch.int64, device='cuda') for _ in range(3)]
    for _ in range(3): f()
    torch.cuda.synchronize()
    for b in bufs:
        lib.ff_set_profile_buffer(ctypes.c_void_p(b.data_ptr())); f()
    lib.ff_set_profile_buffer(None)
    torch.cuda.synchronize()
    ent=[b[:kc.grid_ctas*ST].view(-1,ST)[:,16].double() for b in bufs]
    ext=[b[:kc.grid_ctas*ST].view(-1,ST)[:,31].double() for b in bufs]
    for i in range(2):
        print(f"{shape}: kernel span {(ext[i].max()-ent[i].min()).item()/1e3:.1f} us; entry spread {(ent[i].max()-ent[i].min()).item()/1e3:.2f} us; "
              f"gap last-exit -> next first-entry {(ent[i+1].min()-ext[i].max()).item()/1e3:.1f} us", flush=True)
