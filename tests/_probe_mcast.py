# Diagnostics: per-SM TMA feed vs launch kind, barrier scope, box shape, multicast.
import sys, ctypes, torch
sys.path.insert(0, '.')
from paper_2512_12949_b200 import _native as nat
lib = nat.load()
lib.ff_tma_mcast_bench.argtypes=[ctypes.c_void_p]+[ctypes.c_int]*10+[ctypes.POINTER(ctypes.c_float)]
lib.ff_tma_stream_bench.argtypes=[ctypes.c_void_p]+[ctypes.c_int]*8+[ctypes.POINTER(ctypes.c_float)]
for rows, cols, label in [(2048, 8192, "L2 32MiB"), (4096, 16384, "HBM 128MiB")]:
    mat = torch.randn(rows, cols, device='cuda').bfloat16()
    for br, bb, stage_kb, stages in [(64,4,32,6),(128,2,32,6),(64,8,64,3),(128,4,64,3),(128,2,64,3)]:
        ms=ctypes.c_float(); iters=240
        if stage_kb*1024 == 64*br*2*bb:
            rc=lib.ff_tma_stream_bench(mat.data_ptr(), rows, cols, stages, iters, br | (bb<<16), 144, 1, stage_kb*1024, ctypes.byref(ms))
            tot=144*iters*stage_kb*1024
            print(f"{label:10s} stream-kernel       box 64x{br}x{bb} stage {stage_kb}KB x{stages}: per-SM {tot/ms.value/1e6/144:6.1f} GB/s rc{rc}", flush=True)
        for flags, nm in [(7,"plain+cta-scope"),(6,"cluster1+cta-scope"),(4,"wait.acq.cluster"),(2,"arrive.rel.cluster"),(0,"cluster1+cluster-scope")]:
            rc=lib.ff_tma_mcast_bench(mat.data_ptr(), rows, cols, stages, iters, br, bb, 1, 144, stage_kb*1024, flags, ctypes.byref(ms))
            tot=144*iters*stage_kb*1024
            print(f"{label:10s} {nm:19s} box 64x{br}x{bb} stage {stage_kb}KB x{stages}: per-SM {tot/ms.value/1e6/144:6.1f} GB/s rc{rc}", flush=True)
