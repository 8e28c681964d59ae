"""DSM fabric bandwidth sweep on the B200 (calibrates dsm.bandwidth[n] of the device
profile, paper Fig. 4 method): ff_dsm_bandwidth over cluster size, chunk size,
outstanding copies and issuing threads for bulk pushes, plus the ld/st.shared::cluster
forms.  Prints one JSON line per point: per-SM and chip-wide GB/s.

    python tools/dsm_sweep.py > profiles/r02/dsm_sweep.jsonl
"""

import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_12949_b200 import _native as nat  # noqa: E402


def point(lib, mode, cluster, chunk, depth, issuers, iters):
    n, ms = ctypes.c_int(0), ctypes.c_float(0)
    rc = lib.ff_dsm_bandwidth(mode, cluster, chunk, depth, issuers, iters, ctypes.byref(n), ctypes.byref(ms))
    if rc:
        return {"mode": mode, "cluster": cluster, "chunk": chunk, "depth": depth, "issuers": issuers,
                "error": lib.ff_dsm_last_error().decode()}
    per_cta = iters * (chunk * issuers if mode == 0 else 128 * 1024)
    ctas = n.value * cluster
    gbs = per_cta * ctas / (ms.value * 1e-3) / 1e9
    return {"mode": ["bulk_push", "ld_pull", "st_push"][mode], "cluster": cluster, "chunk": chunk, "depth": depth,
            "issuers": issuers, "clusters": n.value, "ctas": ctas, "ms": round(ms.value, 4),
            "chip_gbs": round(gbs, 1), "per_sm_gbs": round(gbs / ctas, 2)}


def main():
    lib = nat.load()
    lib.ff_dsm_bandwidth.argtypes = [ctypes.c_int] * 6 + [ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_float)]
    lib.ff_dsm_last_error.restype = ctypes.c_char_p
    for cluster in (2, 4, 8, 16):
        point(lib, 0, cluster, 16384, 4, 1, 16)  # warm-up
        for mode in (1, 2):
            print(json.dumps(point(lib, mode, cluster, 0 + 16, 1, 1, 200)), flush=True)
        for chunk in (4096, 16384, 32768, 65536):
            for issuers in (1, 2, 4):
                for inflight in (64 << 10, 128 << 10, 192 << 10):
                    depth = inflight // (chunk * issuers)
                    if depth < 1:
                        continue
                    iters = max(8, (64 << 20) // (chunk * issuers) // 16)
                    print(json.dumps(point(lib, 0, cluster, chunk, depth, issuers, iters)), flush=True)


if __name__ == "__main__":
    main()
