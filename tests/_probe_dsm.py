import sys, ctypes
sys.path.insert(0, '.')
import torch
from paper_2512_12949_b200 import _native as nat
lib = nat.load()
lib.ff_dsm_push_bench.argtypes=[ctypes.c_int]*5+[ctypes.POINTER(ctypes.c_float)]
lib.ff_max_active_clusters.argtypes=[ctypes.c_int,ctypes.c_int,ctypes.POINTER(ctypes.c_int)]
for cl in [2,4,8,16]:
    n=ctypes.c_int(0); lib.ff_max_active_clusters(cl, 200*1024, ctypes.byref(n))
    print("cluster",cl,"max active clusters", n.value, "SMs", n.value*cl, flush=True)
    for chunk in [4096, 16384, 32768]:
        for depth in [2,4]:
            if 2*depth*chunk > 220*1024: continue
            iters=2000 if chunk<=16384 else 1000
            ms=ctypes.c_float(0)
            rc=lib.ff_dsm_push_bench(cl,chunk,depth,iters,n.value,ctypes.byref(ms))
            if rc: print("err", lib.ff_dsm_last_error()); continue
            total=cl*n.value*chunk*iters
            print(f"  chunk {chunk:6d} depth {depth} : {ms.value*1e3:8.1f} us  aggregate {total/ms.value/1e9:7.2f} TB/s  per-SM {total/ms.value/1e6/(cl*n.value):6.1f} GB/s", flush=True)
