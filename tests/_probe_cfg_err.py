# Diagnostics: error of explicit configs for one shape (kernel_config fields ring, n_splits, nb, lb).
import sys, ctypes, torch
sys.path.insert(0, '.')
sys.argv = sys.argv[:1] + ['x']
exec(open('tests/_probe_kernel.py').read().split("for pack in")[0])
shape = (128, 3328, 256, 1792, 2, True)
for xchg in (0, 1):
    for cfg in [(1,4,64,64), (1,1,64,64), (1,4,64,256), (1,1,64,256), (1,2,64,128), (7,1,64,256), (1,13,64,256)]:
        try:
            A,B,B1,D,E,ch,kc,ws,t = setup(*shape, cfg, xchg)
            nat.check(lib.ff_chain_launch(ctypes.byref(ch),ctypes.byref(kc),ctypes.byref(t),ws.data_ptr(),ws.numel(),None))
            torch.cuda.synchronize()
            Er,_ = ref(A,B,D,2,B1)
            err=((E.float()-Er).abs().max()/Er.abs().max()).item()
            print(f"x{xchg} {cfg}: err {err:.2e}", flush=True)
        except Exception as e:
            print(f"x{xchg} {cfg}: {repr(e)[:90]}", flush=True)
