# Diagnostics: fused-chain time (cold L2, CUDA events, median of 15) vs helper hops x
# (debug bits 16-19 = x+1; bit 24 = helpers off).
import sys, ctypes, torch
sys.path.insert(0, '.')
ARGV_MODES = sys.argv[1:] or ['0x1000000', '0x20000', '0x30000', '0x40000', '0']
sys.argv = sys.argv[:1] + ['x']
exec(open('tests/_probe_kernel.py').read().split("for pack in")[0])
flush_buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device='cuda')
MODES = [int(x, 0) for x in ARGV_MODES]
SHAPES = {"llama": (512,8192,2048,2048,2,True), "gpt67b": (512,16384,4096,4096,1,False), "gpt2s": (512,3072,768,768,3,False)}
for name, shape in SHAPES.items():
    for mode in MODES:
        lib.ff_set_debug_mode(mode)
        A,B,B1,D,E,ch,kc,ws,t = setup(*shape,None,2)
        f=lambda: nat.check(lib.ff_chain_launch(ctypes.byref(ch),ctypes.byref(kc),ctypes.byref(t),ws.data_ptr(),ws.numel(),None))
        for _ in range(3): f()
        ts=[]
        for it in range(15):
            flush_buf.add_(1.0)
            a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
            a.record(); f(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b)*1e3)
        Er,_ = ref(A,B,D,shape[4],B1 if shape[5] else None)
        err=((E.float()-Er).abs().max()/Er.abs().max()).item()
        print(f"{name:7s} mode {mode:#10x} helpers {kc.helpers:2d} x {kc.helper_x}: {sorted(ts)[7]:6.1f} us err {err:.1e}", flush=True)
lib.ff_set_debug_mode(0)
