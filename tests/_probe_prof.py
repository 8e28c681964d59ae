import sys, torch, ctypes
sys.path.insert(0, '.')
sys.argv = sys.argv[:1]
exec(open('tests/_probe_kernel.py').read().split("cases=[")[0])
names = ["prod_total","prod_w_empty","prod_w_flag","mma_total","mma_w_full_g0","mma_w_full_hop","mma_w_cempty","mma_w_ownfull","mma_w_eempty",
         "epi_total","epi_w_cfull","epi_w_ownfree","epi_drainC","epi_store","epi_E"]
def prof(m,n,k,l,act,g,xchg,cfg=None):
    A,B,B1,D,E,ch,kc,ws,t = setup(m,n,k,l,act,g,cfg,xchg)
    buf = torch.zeros(kc.grid_ctas*32 + 4096, dtype=torch.int64, device='cuda')
    f=lambda: nat.check(lib.ff_chain_launch(ctypes.byref(ch),ctypes.byref(kc),ctypes.byref(t),ws.data_ptr(),ws.numel(),None))
    for _ in range(3): f()
    lib.ff_set_profile_buffer(ctypes.c_void_p(buf.data_ptr()))
    f(); torch.cuda.synchronize()
    lib.ff_set_profile_buffer(None)
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record(); f(); e.record(); torch.cuda.synchronize()
    ms=s.elapsed_time(e)
    v = buf[:kc.grid_ctas*32].view(kc.grid_ctas,32)[:, :16].double()/1.9e3  # us at 1.9GHz
    lead = v[0::2] if xchg==2 else v
    print(f"== m{m} n{n} k{k} l{l} g{int(g)} x{xchg} {kc.as_dict()} kernel {ms*1e3:.1f}us")
    for i,nm in enumerate(names):
        col = (lead if nm.startswith("mma") else v)[:, i]
        print(f"   {nm:16s} mean {col.mean().item():8.1f}us  max {col.max().item():8.1f}us")
for (m,n,k,l,act,g) in [(512,16384,4096,4096,1,False),(512,8192,2048,2048,2,True)]:
    for x in (2,1):
        prof(m,n,k,l,act,g,x)
