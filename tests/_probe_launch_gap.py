# Diagnostics: where the time between the CUDA events and the kernel's own
# first-entry / last-exit stamps goes.  Sequence per sample (one stream):
#   flush L2 -> stamp0 -> ev_a -> fused chain (per-CTA entry/exit stamps) -> ev_b -> stamp1
# stamp0 -> first CTA entry = launch latency, last exit -> stamp1 = drain tail.
import sys, ctypes, torch
sys.path.insert(0, '.')
ARGV = list(sys.argv)
sys.argv = sys.argv[:1] + ['x']
exec(open('tests/_probe_kernel.py').read().split("for pack in")[0])
ST = 32
flush_buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device='cuda')
stamps = torch.zeros(64, dtype=torch.int64, device='cuda')
stream = torch.cuda.current_stream().cuda_stream
def stamp(i):
    assert lib.ff_stamp_globaltimer(ctypes.c_void_p(stamps.data_ptr() + 8 * i), ctypes.c_void_p(stream)) == 0
NFLUSH = 4 if 'deep' in ARGV else (0 if 'warm' in ARGV else 1)
SHAPES = {"llama": (512,8192,2048,2048,2,True), "gpt67b": (512,16384,4096,4096,1,False),
          "gpt2s": (512,3072,768,768,3,False), "opt": (4096,8192,2048,2048,1,False)}
for name, shape in ([] if 'probe' in ARGV else SHAPES.items() if 'opt' in ARGV else list(SHAPES.items())[:3]):
    for mode, label in (((1 << 28), "empty"), ((1 << 28) | 4, "empty-nocoop")) if 'empty' in ARGV else ((0, "coop"), (4, "no-coop")):
        lib.ff_set_debug_mode(mode)
        A,B,B1,D,E,ch,kc,ws,t = setup(*shape,None,2)
        f=lambda: nat.check(lib.ff_chain_launch(ctypes.byref(ch),ctypes.byref(kc),ctypes.byref(t),ws.data_ptr(),ws.numel(),None))
        buf = torch.zeros(kc.grid_ctas*ST + 64, dtype=torch.int64, device='cuda')
        for _ in range(3): f()
        torch.cuda.synchronize()
        res = []
        for it in range(8):
            ea = torch.cuda.Event(enable_timing=True); eb = torch.cuda.Event(enable_timing=True)
            for _ in range(NFLUSH): flush_buf.add_(1.0)
            if 'spin' in ARGV: lib.ff_spin(ctypes.c_longlong(200000), 148, ctypes.c_void_p(stream))
            stamp(0); ea.record()
            lib.ff_set_profile_buffer(ctypes.c_void_p(buf.data_ptr())); f(); lib.ff_set_profile_buffer(None)
            eb.record(); stamp(1)
            torch.cuda.synchronize()
            v = buf[:kc.grid_ctas*ST].view(-1, ST)
            ent, ext = v[:,16].double(), v[:,31].double()
            s0, s1 = stamps[0].item(), stamps[1].item()
            res.append((ea.elapsed_time(eb)*1e3, (ent.min().item()-s0)/1e3, (ext.max()-ent.min()).item()/1e3,
                        (s1-ext.max().item())/1e3, (ent.max()-ent.min()).item()/1e3))
        res.sort()
        r = res[len(res)//2]
        print(f"{name:7s} {label:8s} grid {kc.grid_ctas:3d}: events {r[0]:6.1f} us | stamp0->first entry {r[1]:5.1f} | "
              f"span {r[2]:6.1f} | last exit->stamp1 {r[3]:5.1f} | entry spread {r[4]:4.1f}", flush=True)
lib.ff_set_debug_mode(0)
# reference points: stamp -> trivial torch kernel -> stamp, and the cuBLAS GEMM
x = torch.zeros(1, device='cuda')
for label, fn in (("torch add", lambda: x.add_(1)),):
    res=[]
    for it in range(8):
        flush_buf.add_(1.0); stamp(0); fn(); stamp(1); torch.cuda.synchronize()
        res.append((stamps[1].item()-stamps[0].item())/1e3)
    print(f"{label}: stamp->kernel->stamp {sorted(res)[4]:.1f} us")
res=[]
for it in range(8):
    flush_buf.add_(1.0); stamp(0); stamp(1); torch.cuda.synchronize()
    res.append((stamps[1].item()-stamps[0].item())/1e3)
print(f"stamp->stamp {sorted(res)[4]:.1f} us")
# launch-shape probe: empty kernel with the chain kernels' launch shape
pst = torch.zeros(4096, dtype=torch.int64, device='cuda')
for ctas, smem, cl, tm in [(128,200*1024,2,6),(128,0,1,6),(128,200*1024,2,4),(128,200*1024,2,5),(128,200*1024,2,3),(128,0,1,3),(128,0,1,2),(128,0,2,2),(1,0,1,0),(128,0,1,0),(128,200*1024,1,0),(128,0,2,0),(128,200*1024,2,0),(128,200*1024,2,1),
                           (128,220*1024,4,1),(148,220*1024,2,1),(96,200*1024,3,1)]:
    res=[]
    for it in range(8):
        flush_buf.add_(1.0); stamp(0)
        assert lib.ff_launch_probe(ctypes.c_void_p(pst.data_ptr()), ctas, smem, cl, tm, ctypes.c_void_p(stream)) == 0
        stamp(1); torch.cuda.synchronize()
        v = pst[:2*ctas].view(-1,2).double()
        s0, s1 = stamps[0].item(), stamps[1].item()
        res.append(((s1-s0)/1e3, (v[:,0].min().item()-s0)/1e3, (v[:,1].max()-v[:,0].min()).item()/1e3, (s1-v[:,1].max().item())/1e3))
    res.sort(); r=res[4]
    print(f"probe ctas {ctas:3d} smem {smem//1024:3d}K cluster {cl} tmem {tm}: stamp->stamp {r[0]:5.1f} | ->entry {r[1]:5.1f} | span {r[2]:5.1f} | exit-> {r[3]:5.1f} us", flush=True)
