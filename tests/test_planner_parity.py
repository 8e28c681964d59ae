"""Host planner == reference planner, bit for bit, on the committed fixtures
(tests/golden/*.json from tests/golden/make_golden.py)."""

import json
import os

import pytest

import paper_2512_12949_b200 as ff
from paper_2512_12949_b200 import hardware as H
from paper_2512_12949_b200 import plan as P
import importlib

S = importlib.import_module("paper_2512_12949_b200.search")
from paper_2512_12949_b200 import simulator as SIM
from paper_2512_12949_b200 import workload as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


def dumps(doc):
    return json.dumps(doc, sort_keys=True, indent=1)


def graph_from(doc):
    dims = W.DimensionSpec(doc["m"], doc["n"], doc["k"], doc["l"], doc["element_size"])
    if doc["kind"] == W.GATED_FFN:
        return W.build_gated_ffn(dims)
    return W.build_standard_ffn(dims, doc["activation"], logical_m=doc.get("logical_m"))


def device_from(name):
    return H.default_h100() if name == "h100" else H.b200_profile()


# ---------------------------------------------------------------- workload / hardware / plan


def test_presets_match_reference():
    misc = load("misc.json")
    assert sorted(W.preset_ids()) == sorted(misc["presets"]) and len(W.preset_ids()) == 26
    for pid, doc in misc["presets"].items():
        g = W.preset(pid)
        assert (g.kind, g.activation, *g.dims.as_tuple(), g.dims.element_size, g.logical_m) == (
            doc["kind"], doc["activation"], doc["m"], doc["n"], doc["k"], doc["l"], doc["element_size"],
            doc["logical_m"])


def test_profile_text_roundtrip_and_reference_serializer():
    misc = load("misc.json")
    assert H.serialize_device_profile(H.default_h100()) == misc["h100_profile_text"]
    assert H.parse_device_profile(misc["h100_profile_text"]) == H.default_h100()
    b = H.b200_profile()
    assert H.parse_device_profile(H.serialize_device_profile(b), waive=(H.WAIVER_DSM_BELOW_GLOBAL,)) == b
    with pytest.raises(ff.ProfileError):  # the reference rule still applies by default
        H.parse_device_profile(H.B200_PROFILE_TEXT)


def test_profile_validation_errors():
    with pytest.raises(ff.ProfileError):
        H.parse_device_profile("dsm.bandwidth[2] = 1e12\ndsm.bandwidth[4] = 2e12\n")
    with pytest.raises(ff.ProfileError):
        H.parse_device_profile("reg.capacity_bytes = lots\n")
    with pytest.raises(ff.ProfileError):
        H.parse_device_profile("bogus.key = 1\n")
    with pytest.raises(ff.ClusterTooLarge):
        H.dsm_bandwidth(H.default_h100(), 32)
    assert H.dsm_bandwidth(H.default_h100(), 1) == H.default_h100().smem.bandwidth


def test_workload_text_roundtrip():
    misc = load("misc.json")
    g = W.build_gated_ffn(W.DimensionSpec(128, 3072, 1024, 1024))
    assert W.serialize_workload(g) == misc["workload_text"]
    assert W.parse_workload(misc["workload_text"]) == g


def test_schedules_table_iv():
    space = load("space_counts.json")
    got = [[sorted(s.spatial), list(s.temporal_order)] for s in P.enumerate_schedules()]
    assert got == space["schedules"]
    sizes = [len(s.spatial) for s in P.enumerate_schedules()]
    assert [sizes.count(i) for i in (1, 2, 3, 4)] == [24, 12, 4, 1]


def test_cluster_groups_fig7():
    misc = load("misc.json")
    for key, want in misc["groups"].items():
        assert list(P.derive_cluster_groups(*json.loads(key.replace("(", "[").replace(")", "]")))) == want
    with pytest.raises(ff.InfeasibleCluster):
        P.derive_cluster_groups(1, 2, 2, 8)


def test_conv_lowering_and_errors():
    g = W.preset("C4")
    assert g.dims.m == 64 and g.logical_m == 49
    with pytest.raises(ff.UnsupportedConvChain):
        W.ConvChainConfig(64, 56, 56, 64, 64, 1, 3)
    with pytest.raises(ff.InvalidDimension):
        W.conv_chain_to_gemm(W.ConvChainConfig(1, 1, 1, 16, 16, 1, 1))
    with pytest.raises(ff.UnknownPreset):
        W.preset("X9")


def test_plan_json_roundtrip():
    plan = P.make_plan("n", "klm", (64, 1024, 4096, 512), (1, 16, 1, 8)).with_mapping({"C": {"reg": 5}})
    assert P.plan_from_json(P.plan_to_json(plan)) == plan
    with pytest.raises(ff.PlanError):
        P.plan_from_dict({"version": 99})


# ---------------------------------------------------------------- space counting


def test_count_space_table_iii_exact():
    space = load("space_counts.json")
    g = W.build_standard_ffn(W.DimensionSpec(256, 16384, 4096, 4096), "relu")
    got = S.count_space(g, H.default_h100())
    assert dumps(got) == dumps(space["g5_m256_h100"])
    assert got["stages"][0]["count"] == 27_514_634_240_000
    assert got["stages"][1]["count"] == 114_159_375
    assert S.dsm_space_expansion(g, H.default_h100()) == space["g5_m256_expansion_h100"]
    assert dumps(S.count_space(g, H.b200_profile())) == dumps(space["g5_m256_b200"])
    assert dumps(S.count_space(W.preset("S8"), H.default_h100())) == dumps(space["s8_h100"])


def test_empty_space_stage():
    space = load("space_counts.json")
    with pytest.raises(ff.EmptySpace) as info:
        S.search(W.preset("C3"), H.b200_profile())
    assert info.value.stage == space["c3_b200_space"]["empty_stage"]


# ---------------------------------------------------------------- analyzer / replay


@pytest.fixture(scope="module")
def samples():
    return load("analyzer_samples.json")


def test_sample_valid_plans_same_draws(samples):
    for name, case in samples.items():
        g = graph_from(case["graph"])
        plans = SIM.sample_valid_plans(g, device_from(case["device"]), 20, seed=7)
        assert [P.plan_to_dict(p) for p in plans] == [row["plan"] for row in case["plans"]], name


def test_analyzer_reports_match_reference(samples):
    for name, case in samples.items():
        g = graph_from(case["graph"])
        dev = device_from(case["device"])
        for row in case["plans"]:
            plan = P.plan_from_dict(row["plan"])
            rep = ff.analyze(g, dev, plan).report_dict()
            assert dumps(rep) == dumps(row["report"]), (name, row["plan"])
            lit = ff.analyze(g, dev, plan, literal=True).volume
            assert lit == row["literal_volume"]


def test_traffic_replay_matches_reference_simulator(samples):
    """SPEC acceptance 6, across implementations: our replay == reference replay."""
    for name, case in samples.items():
        g = graph_from(case["graph"])
        dev = device_from(case["device"])
        for row in case["plans"][:10]:
            plan = P.plan_from_dict(row["plan"])
            trace = SIM.replay_traffic(plan, g, dev)
            assert dumps(trace.to_dict()) == dumps(row["trace"]), (name, row["plan"])


def test_unfused_baseline_bytes_match_reference(samples):
    for name, case in samples.items():
        g = graph_from(case["graph"])
        for row in case["plans"][:5]:
            plan = P.plan_from_dict(row["plan"])
            _, trace = _unfused_trace(g, plan)
            assert dumps(trace.to_dict()) == dumps(row["unfused"]), name


def _unfused_trace(g, plan):
    # byte model only (no GPU): call the traffic part of unfused_baseline
    import paper_2512_12949_b200.simulator as sim

    orig = sim.oracle
    sim.oracle = lambda graph, inputs: None
    try:
        return sim.unfused_baseline(g, {}, plan)
    finally:
        sim.oracle = orig


# ---------------------------------------------------------------- search


SEARCH_FAST = ["h100_G1", "h100_G2_desk256", "h100_C1_desk256", "h100_G10", "b200_gpt2s", "b200_conv_c5"]
SEARCH_SLOW = ["h100_S8_desk256", "b200_llama1b", "b200_gpt67b", "b200_opt13b_m4096", "b200_G5", "b200_S3"]


@pytest.fixture(scope="module")
def search_gold():
    path = os.path.join(GOLD, "search_results.json")
    if not os.path.exists(path):
        pytest.skip("search goldens not generated")
    return load("search_results.json")


def _check_search(search_gold, name, workers=8):
    case = search_gold[name]
    g = graph_from(case["graph"])
    got = S.search(g, device_from(case["device"]), refine_with_simulator=False, workers=workers)
    assert dumps(got.to_dict()) == dumps(case["result"]), name


@pytest.mark.parametrize("name", SEARCH_FAST)
def test_search_bit_exact(search_gold, name):
    _check_search(search_gold, name)


@pytest.mark.slow
@pytest.mark.parametrize("name", SEARCH_SLOW)
def test_search_bit_exact_large(search_gold, name):
    _check_search(search_gold, name)


def test_search_default_refine_matches(search_gold):
    case = search_gold["h100_G1_refined"]
    got = S.search(graph_from(case["graph"]), H.default_h100(), workers=8)
    assert got.ranked_by == "simulator"
    assert dumps(got.to_dict()) == dumps(case["result"])


def test_search_prefix_and_worker_invariance():
    g = W.scale_to_desk(W.preset("G3"), 256)
    dev = H.default_h100()
    one = S.search(g, dev, k=1, refine_with_simulator=False, workers=1)
    many = S.search(g, dev, k=11, refine_with_simulator=False, workers=4)
    assert dumps(one.top[0].to_dict()) == dumps(many.top[0].to_dict())
    again = S.search(g, dev, k=11, refine_with_simulator=False, workers=1)
    assert dumps(again.to_dict()) == dumps(many.to_dict())
