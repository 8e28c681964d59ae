import sys, ctypes, torch
sys.path.insert(0, '.')
from paper_2512_12949_b200 import _native as nat
lib = nat.load()
lib.ff_tma_stream_bench.argtypes=[ctypes.c_void_p]+[ctypes.c_int]*8+[ctypes.POINTER(ctypes.c_float)]
rows, cols = 4096, 16384
mat = torch.randn(rows, cols, device='cuda').bfloat16()
for br, bb, stage_kb, stages, prods in [(64,4,32,6,1),(64,4,32,6,2),(64,4,32,6,3),(64,4,32,4,4),(64,2,32,6,2),(64,1,32,6,2),(64,1,32,6,3),
                                        (64,8,64,3,1),(128,4,64,3,1),(64,4,64,3,1),(256,2,64,3,1),(64,8,64,2,2),(128,4,64,2,2),(64,4,64,2,2),(256,4,128,1,1)]:
    ms=ctypes.c_float(); iters=240
    rc=lib.ff_tma_stream_bench(mat.data_ptr(), rows, cols, stages, iters, br | (bb<<16), 148, prods, stage_kb*1024, ctypes.byref(ms))
    tot=148*iters*stage_kb*1024
    kb = 64*br*2*max(bb,1)//1024
    if rc: print("rc", rc, br, bb, stage_kb); continue
    print(f"box 64x{br}x{bb} ({kb} KB/instr) stage {stage_kb}KB x{stages} producers {prods}: {tot/ms.value/1e9:6.2f} TB/s  per-SM {tot/ms.value/1e6/148:6.1f} GB/s", flush=True)
