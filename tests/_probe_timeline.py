# Diagnostics: per-CTA globaltimer timeline of the pair kernel + cuBLAS per-GEMM times.
import sys, torch, ctypes
sys.path.insert(0, '.')
ARGV = list(sys.argv)
sys.argv = sys.argv[:1] + ['x'] + sys.argv[1:]
exec(open('tests/_probe_kernel.py').read().split("PACK[0]=True")[0].split("for pack in")[0])
ST = 32
def timeline(m,n,k,l,act,g,xchg,cfg=None):
    A,B,B1,D,E,ch,kc,ws,t = setup(m,n,k,l,act,g,cfg,xchg)
    buf = torch.zeros(kc.grid_ctas*ST + 4096, dtype=torch.int64, device='cuda')
    f=lambda: nat.check(lib.ff_chain_launch(ctypes.byref(ch),ctypes.byref(kc),ctypes.byref(t),ws.data_ptr(),ws.numel(),None))
    for _ in range(5): f()
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record(); f(); e.record(); torch.cuda.synchronize()
    ms_plain = s.elapsed_time(e)
    import time
    torch.cuda.synchronize(); s.record()
    for _ in range(20): f()
    e.record(); torch.cuda.synchronize()
    ms_b2b = s.elapsed_time(e)/20
    hs=[]
    for _ in range(20):
        t0=time.perf_counter(); f(); hs.append(time.perf_counter()-t0)
    torch.cuda.synchronize()
    print(f"   back-to-back {ms_b2b*1e3:.1f}us/launch; host ff_chain_launch call {sorted(hs)[10]*1e6:.1f}us (median)")
    lib.ff_set_profile_buffer(ctypes.c_void_p(buf.data_ptr()))
    torch.cuda.synchronize(); s.record(); f(); e.record(); torch.cuda.synchronize()
    ms=s.elapsed_time(e)
    lib.ff_set_profile_buffer(None)
    v = buf[:kc.grid_ctas*ST].view(kc.grid_ctas,ST)
    tl = v[:,16:].double()
    t0 = tl[:,0].min()
    rel = (tl - t0)/1e3
    rel[tl==0] = float('nan')
    print(f"== m{m} n{n} k{k} l{l} g{int(g)} x{xchg} {kc.as_dict()} events {ms_plain*1e3:.1f}us (profiled {ms*1e3:.1f}us)")
    names = {0:'entry',1:'setup',6:'E_summed',8:'E_staged',9:'E_slabs_out',10:'E_finished',11:'E_flags_in',12:'E_loaded',13:'E_sum0',14:'E_start',15:'exit'}
    for T in range(1):
        names[2+3*T]=f'cfull{T}'; names[3+3*T]=f'drained{T}'; names[4+3*T]=f'stored{T}'
    for i in range(16):
        col = rel[:,i]; col = col[~torch.isnan(col)]
        if col.numel()==0: continue
        print(f"   {str(names.get(i,i)):10s} min {col.min().item():7.1f} mean {col.mean().item():7.1f} max {col.max().item():7.1f} us")
def cublas(m,n,k,l,g):
    A=torch.randn(m,k,device='cuda').bfloat16(); B=torch.randn(k,(2 if g else 1)*n,device='cuda').bfloat16()
    C=torch.randn(m,n,device='cuda').bfloat16(); D=torch.randn(n,l,device='cuda').bfloat16()
    for name,fn in (("gemm0",lambda: A@B),("gemm1",lambda: C@D)):
        for _ in range(5): fn()
        s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); s.record()
        for _ in range(20): fn()
        e.record(); torch.cuda.synchronize()
        print(f"   cublas {name} {s.elapsed_time(e)/20*1e3:.1f}us (warm L2)")
MODES = [int(x) for x in (sys.argv[2:] if len(sys.argv) > 2 else ["0"])]
for (m,n,k,l,act,g) in [(512,8192,2048,2048,2,True),(512,16384,4096,4096,1,False)]:
    for mode in MODES:
        lib.ff_set_debug_mode(mode)
        print(f"-- debug mode {mode} (bit0 no MMA, bit1 no flag waits)")
        timeline(m,n,k,l,act,g,2)
    lib.ff_set_debug_mode(0)
    cublas(m,n,k,l,g)
