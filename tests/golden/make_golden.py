"""Generate the golden fixtures under tests/golden/ from the REFERENCE planner.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

Everything written here comes from importing /root/reference/pkg/src/fuseplan
read-only; nothing of this repo's package is imported, so the fixtures pin the
reference's behaviour.  The GPU box never reads /root/reference: tests use only
the committed outputs.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

import fuseplan as R  # noqa: E402
from fuseplan import hardware as RH  # noqa: E402
from fuseplan import simulator as RS  # noqa: E402
from fuseplan import workload as RW  # noqa: E402

# Measured B200 profile values (see paper_2512_12949_b200/hardware.py B200_PROFILE_TEXT).
# The reference parser rejects the measured DSM table (DSM < HBM on B200), so the
# DeviceModel is constructed directly -- the search itself does not validate.
B200 = RH.DeviceModel(
    name="b200",
    reg=RH.MemoryLevel("reg", "per-block", 262144, 2.4e15),
    smem=RH.MemoryLevel("smem", "per-block", 232448, 3.6e13),
    dsm_bandwidth_table={2: 5.47e12, 4: 4.35e12, 8: 3.86e12, 16: 3.6e12},
    l2=RH.MemoryLevel("l2", "device", 132120576, 2.0e13),
    global_mem=RH.MemoryLevel("global", "device", None, 6.4522e12),
    max_cluster_blocks=16,
    cluster_dim_options=(1, 2, 4, 8, 16),
    mma_tile=(64, 64, 16),
)

# (name, graph builder, device name)
SEARCH_CASES = [
    ("h100_G1", lambda: R.preset("G1"), "h100"),
    ("h100_G2_desk256", lambda: R.scale_to_desk(R.preset("G2"), 256), "h100"),
    ("h100_S8_desk256", lambda: R.scale_to_desk(R.preset("S8"), 256), "h100"),
    ("h100_C1_desk256", lambda: R.scale_to_desk(R.preset("C1"), 256), "h100"),
    ("h100_G10", lambda: R.preset("G10"), "h100"),
    ("b200_gpt2s", lambda: R.build_standard_ffn(R.DimensionSpec(512, 3072, 768, 768, 2), "relu"), "b200"),
    ("b200_llama1b", lambda: R.build_gated_ffn(R.DimensionSpec(512, 8192, 2048, 2048, 2)), "b200"),
    ("b200_gpt67b", lambda: R.build_standard_ffn(R.DimensionSpec(512, 16384, 4096, 4096, 2), "relu"), "b200"),
    ("b200_conv_c5", lambda: R.preset("C5"), "b200"),
    ("b200_opt13b_m4096", lambda: R.build_standard_ffn(R.DimensionSpec(4096, 8192, 2048, 2048, 2), "relu"), "b200"),
    ("b200_G5", lambda: R.preset("G5"), "b200"),
    ("b200_S3", lambda: R.preset("S3"), "b200"),
]


def device(name):
    return R.default_h100() if name == "h100" else B200


def dumps(doc) -> str:
    return json.dumps(doc, sort_keys=True, indent=1) + "\n"


def write(name, doc):
    with open(os.path.join(HERE, name), "w", encoding="utf-8") as fh:
        fh.write(dumps(doc))


def graph_doc(g) -> dict:
    d = g.dims
    return {"kind": g.kind, "activation": g.activation, "m": d.m, "n": d.n, "k": d.k, "l": d.l,
            "element_size": d.element_size, "logical_m": g.logical_m}


def gen_search():
    out = {}
    for name, build, dev in SEARCH_CASES:
        g = build()
        t0 = time.time()
        res = R.search(g, device(dev), refine_with_simulator=False)
        out[name] = {"graph": graph_doc(g), "device": dev, "result": res.to_dict(),
                     "reference_seconds": round(time.time() - t0, 2)}
        print(f"search {name}: {res.evaluated} survivors, {time.time() - t0:.1f}s, top-1 {res.top[0].plan.describe()}",
              flush=True)
    # default refine (simulator re-rank) on one small chain: ranked_by == "simulator"
    g = R.preset("G1")
    res = R.search(g, R.default_h100())
    out["h100_G1_refined"] = {"graph": graph_doc(g), "device": "h100", "result": res.to_dict()}
    write("search_results.json", out)


def gen_space():
    g = R.build_standard_ffn(R.DimensionSpec(256, 16384, 4096, 4096), "relu")
    doc = {
        "g5_m256_h100": R.count_space(g, R.default_h100()),
        "g5_m256_expansion_h100": R.dsm_space_expansion(g, R.default_h100()),
        "g5_m256_b200": R.count_space(g, B200),
        "schedules": [[sorted(s.spatial), list(s.temporal_order)] for s in R.enumerate_schedules()],
        "s8_h100": R.count_space(R.preset("S8"), R.default_h100()),
        "c3_b200_space": None,
    }
    try:
        R.search(R.preset("C3"), B200)
    except R.EmptySpace as exc:
        doc["c3_b200_space"] = {"empty_stage": exc.stage}
    write("space_counts.json", doc)


def gen_analyzer():
    cases = [
        ("G4", R.scale_to_desk(R.preset("G4"), 256), R.default_h100()),
        ("S8", R.scale_to_desk(R.preset("S8"), 256), R.default_h100()),
        ("C1", R.scale_to_desk(R.preset("C1"), 256), R.default_h100()),
        ("G1", R.preset("G1"), R.default_h100()),
        ("G7_b200", R.scale_to_desk(R.preset("G7"), 512), B200),
    ]
    out = {}
    for name, g, dev in cases:
        plans = RS.sample_valid_plans(g, dev, 20, seed=7)
        rows = []
        cfg = RS.SimConfig(dtype="f64", seed=3)
        inputs = RS.make_inputs(g, cfg)
        ref = RS.oracle(g, inputs)
        for p in plans:
            an = R.analyze(g, dev, p)
            lit = R.analyze(g, dev, p, literal=True)
            e, trace = RS.execute_plan(p, g, inputs, cfg, dev)
            rows.append({
                "plan": R.plan.plan_to_dict(p),
                "report": an.report_dict(),
                "literal_volume": {k: int(v) for k, v in lit.volume.items()},
                "trace": trace.to_dict(),
                "sim_max_rel_error": RS.max_relative_error(e, ref),
                "unfused": RS.unfused_baseline(g, inputs, p)[1].to_dict(),
            })
        out[name] = {"graph": graph_doc(g), "device": "h100" if dev.name == "h100" else "b200", "plans": rows}
        print(f"analyzer {name}: {len(rows)} plans", flush=True)
    write("analyzer_samples.json", out)


def gen_numerics():
    """Reference oracle outputs on seeded inputs (small shapes)."""
    cases = {
        "relu_128x256x128x128": R.build_standard_ffn(R.DimensionSpec(128, 256, 128, 128), "relu"),
        "identity_64x128x64x64": R.build_standard_ffn(R.DimensionSpec(64, 128, 64, 64), "identity"),
        "silu_128x192x64x128": R.build_standard_ffn(R.DimensionSpec(128, 192, 64, 128), "silu"),
        "gated_128x256x128x128": R.build_gated_ffn(R.DimensionSpec(128, 256, 128, 128)),
        "conv_c1_desk": R.scale_to_desk(R.preset("C1"), 128),
    }
    arrays, meta = {}, {}
    for name, g in cases.items():
        for dtype in ("f32", "f64"):
            cfg = RS.SimConfig(dtype=dtype, seed=11)
            inputs = RS.make_inputs(g, cfg)
            e = RS.oracle(g, inputs)
            arrays[f"{name}__{dtype}__E"] = e.astype(np.float64 if dtype == "f64" else np.float32)
            meta[f"{name}__{dtype}"] = {
                "graph": graph_doc(g),
                "seed": 11,
                "input_checksums": {k: float(np.sum(v, dtype=np.float64)) for k, v in inputs.items()},
                "input_first": {k: float(v.flat[0]) for k, v in inputs.items()},
            }
        # plan-faithful replay output for the best plan of the chain
        plan = R.search(g, R.default_h100(), k=1, refine_with_simulator=False).top[0].plan
        cfg = RS.SimConfig(dtype="f64", seed=11)
        e_sim, _ = RS.execute_plan(plan, g, RS.make_inputs(g, cfg), cfg)
        arrays[f"{name}__sim__E"] = e_sim
        meta[f"{name}__sim"] = {"plan": R.plan.plan_to_dict(plan)}
    np.savez_compressed(os.path.join(HERE, "numerics.npz"), **arrays)
    write("numerics_meta.json", meta)


def gen_misc():
    doc = {
        "h100_profile_text": RH.serialize_device_profile(R.default_h100()),
        "presets": {pid: graph_doc(R.preset(pid)) for pid in R.preset_ids()},
        "groups": {str(c): list(R.derive_cluster_groups(*c)) for c in [(2, 4, 2, 4), (2, 4, 2, 8), (1, 1, 1, 1),
                                                                        (1, 16, 1, 8), (1, 8, 2, 8)]},
        "workload_text": RW.serialize_workload(R.build_gated_ffn(R.DimensionSpec(128, 3072, 1024, 1024))),
    }
    write("misc.json", doc)


if __name__ == "__main__":
    which = sys.argv[1:] or ["misc", "space", "analyzer", "numerics", "search"]
    for w in which:
        globals()["gen_" + w]()
