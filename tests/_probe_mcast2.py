# Diagnostics: multicast feed with relaxed (flags 8) vs release (flags 0) remote empty arrives.
import sys, ctypes, torch
sys.path.insert(0, '.')
from paper_2512_12949_b200 import _native as nat
lib = nat.load()
lib.ff_tma_mcast_bench.argtypes=[ctypes.c_void_p]+[ctypes.c_int]*10+[ctypes.POINTER(ctypes.c_float)]
for rows, cols, label in [(2048, 8192, "L2 32MiB"), (8192, 16384, "HBM 256MiB")]:
    mat = torch.randn(rows, cols, device='cuda').bfloat16()
    for csize, ctas in [(1,144),(2,144),(4,144)]:
        for br, bb, stage_kb, stages in [(128,2,64,3),(128,4,64,3),(256,2,64,3)]:
            for flags in ([6] if csize == 1 else [0, 8]):
                ms=ctypes.c_float(); iters=240
                rc=lib.ff_tma_mcast_bench(mat.data_ptr(), rows, cols, stages, iters, br, bb, csize, ctas, stage_kb*1024, flags, ctypes.byref(ms))
                if rc: print("rc", rc, csize, br, bb, flags, flush=True); continue
                tot=ctas*iters*stage_kb*1024
                print(f"{label:10s} cluster {csize} flags {flags} box 64x{br}x{bb} ({64*br*2*bb//1024//csize} KB issued/instr) stage {stage_kb}KB x{stages}: per-SM {tot/ms.value/1e6/ctas:6.1f} GB/s", flush=True)
