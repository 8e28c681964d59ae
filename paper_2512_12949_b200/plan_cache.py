"""M-bin plan dispatch table (paper SIV-C3: offline search + on-device
ProfileBestFromList, run-time table lookup by M).

``plans/plan_cache.json`` holds, per chain shape, the top-K plans of this
package's search (bit-exact with the reference) under the B200 profile.  The
runtime lowers them and keeps the fastest on the device.  Regenerate with
``python -m paper_2512_12949_b200.plan_cache``.
"""

from __future__ import annotations

import json
import os

from .workload import DimensionSpec, build_gated_ffn, build_standard_ffn

HERE = os.path.dirname(os.path.abspath(__file__))
CACHE = os.path.join(HERE, "plans", "plan_cache.json")
# searched top-K plans per (dispatch family, M bin): the offline-search leg of the M-bin
# dispatch tables (dispatch.build_table profiles them on the device)
BINS_CACHE = os.path.join(HERE, "plans", "plan_bins.json")

# (kind, activation class, m, n, k, l): the BASELINE.json configurations.
SHAPES = [
    ("gated_ffn", "silu", 512, 8192, 2048, 2048),
    ("standard_ffn", "relu", 512, 16384, 4096, 4096),
    ("standard_ffn", "relu", 512, 3072, 768, 768),
    ("standard_ffn", "relu", 4096, 8192, 2048, 2048),
    ("standard_ffn", "relu", 3136, 64, 576, 256),
]

_cache = None


def _key(kind, act, m, n, k, l) -> str:
    act_class = "silu" if kind == "gated_ffn" else ("identity" if act == "identity" else "nonlinear")
    return f"{kind}/{act_class}/{m}x{n}x{k}x{l}"


def lookup(kind, act, m, n, k, l):
    global _cache
    if _cache is None:
        if not os.path.exists(CACHE):
            _cache = {}
        else:
            with open(CACHE) as fh:
                _cache = json.load(fh)
    return _cache.get(_key(kind, act, m, n, k, l))


def build(shapes=SHAPES, k_top: int = 11, workers: int = 8) -> dict:
    from .hardware import b200_profile
    from .plan import plan_to_dict
    from .search import search

    out = {}
    dev = b200_profile()
    for kind, act, m, n, k, l in shapes:
        dims = DimensionSpec(m, n, k, l, 2)
        g = build_gated_ffn(dims) if kind == "gated_ffn" else build_standard_ffn(dims, act)
        res = search(g, dev, k=k_top, refine_with_simulator=False, workers=workers)
        out[_key(kind, act, m, n, k, l)] = {
            "top": [plan_to_dict(e.plan) for e in res.top],
            "cost_seconds": [e.cost.total for e in res.top],
            "evaluated": res.evaluated,
            "device": dev.name,
        }
    return out


def build_bins(families=None, bins=None, k_top: int = 11, workers: int = 8) -> dict:
    """The reference search's top-K plans (B200 profile) for every dispatch family at
    the upper edge of every M bin (paper SIV-C3: offline search per M bin)."""
    from .dispatch import DEFAULT_BINS, FAMILIES

    families = FAMILIES if families is None else families
    bins = DEFAULT_BINS if bins is None else bins
    shapes = [(kind, act, m, n, k, l) for kind, act, n, k, l in families.values() for m in bins]
    return build(shapes, k_top=k_top, workers=workers)


_bins = None


def plans_by_m(kind, act, n, k, l, bins) -> dict:
    """{M: [FusionPlan, ...]} from plans/plan_bins.json for one dispatch family
    (bins without an entry are left out)."""
    global _bins
    from .plan import plan_from_dict

    if _bins is None:
        _bins = {}
        if os.path.exists(BINS_CACHE):
            with open(BINS_CACHE) as fh:
                _bins = json.load(fh)
    out = {}
    for m in bins:
        e = _bins.get(_key(kind, act, m, n, k, l))
        if e is not None:
            out[m] = [plan_from_dict(p) for p in e["top"]]
    return out


if __name__ == "__main__":
    import sys

    os.makedirs(os.path.dirname(CACHE), exist_ok=True)
    if "bins" in sys.argv[1:]:
        doc = build_bins()
        path = BINS_CACHE
    else:
        doc = build()
        path = CACHE
    with open(path, "w") as fh:
        json.dump(doc, fh, sort_keys=True, indent=1)
    print(f"wrote {path}: {len(doc)} shapes")
