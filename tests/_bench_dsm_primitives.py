# Microbenchmark of the DSM communication primitives: bytes received per CTA per
# primitive call / time, per SM and aggregate (64 KB fp32 tile per CTA).
import ctypes, json, sys
import torch
sys.path.insert(0, '.')
from paper_2512_12949_b200 import _native as nat
lib = nat.load()
lib.ff_dsm_primitive_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
lib.ff_max_active_clusters.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
OPS = {"reduce_scatter": 0, "all_gather": 1, "all_exchange_add": 2, "all_exchange_mul": 3, "shuffle": 4}
N = 16384
rows = []
for G in (2, 4, 8, 16):
    act = ctypes.c_int()
    lib.ff_max_active_clusters(G, 200 * 1024, ctypes.byref(act))
    clusters = max(1, act.value)
    x = torch.rand(clusters * G * N, device="cuda")
    y = torch.empty_like(x)
    for op, code in OPS.items():
        if op == "all_exchange_mul" and G != 2:
            continue
        recv = {"reduce_scatter": (G - 1) * N // G, "all_gather": (G - 1) * N // G,
                "all_exchange_add": 2 * (G - 1) * N // G}.get(op, N) * 4
        ms1, ms2 = ctypes.c_float(), ctypes.c_float()
        assert lib.ff_dsm_primitive_run(code, G, N, clusters, x.data_ptr(), y.data_ptr(), 5, ctypes.byref(ms1)) == 0
        assert lib.ff_dsm_primitive_run(code, G, N, clusters, x.data_ptr(), y.data_ptr(), 105, ctypes.byref(ms2)) == 0
        per_iter_us = (ms2.value - ms1.value) * 1e3 / 100
        gbs_sm = recv / (per_iter_us * 1e-6) / 1e9
        rows.append({"op": op, "cluster": G, "clusters": clusters, "ctas": clusters * G, "bytes_received_per_cta": recv,
                     "us_per_call": round(per_iter_us, 3), "GBps_per_sm": round(gbs_sm, 1),
                     "GBps_aggregate": round(gbs_sm * clusters * G, 1)})
        print(f"G={G:2d} x{clusters:3d} {op:17s} {per_iter_us:7.2f} us/call  {gbs_sm:6.1f} GB/s per SM  "
              f"{gbs_sm * clusters * G / 1e3:6.2f} TB/s aggregate", flush=True)
json.dump(rows, open("gpurun_out/dsm_primitives_bench.json", "w"), indent=1)
