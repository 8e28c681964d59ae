"""The CPU oracle is pinned against the reference's own outputs (tests/golden/)."""

import json
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def meta():
    with open(os.path.join(GOLD, "numerics_meta.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def arrays():
    return np.load(os.path.join(GOLD, "numerics.npz"))


def _inputs(g, seed, dtype):
    return oracle.make_inputs(g["kind"], g["m"], g["n"], g["k"], g["l"], seed=seed,
                              dtype=np.float64 if dtype == "f64" else np.float32)


def test_make_inputs_reproduces_reference_rng(meta):
    for key, info in meta.items():
        if key.endswith("__sim"):
            continue
        dtype = key.split("__")[1]
        inputs = _inputs(info["graph"], info["seed"], dtype)
        for name, checksum in info["input_checksums"].items():
            assert float(np.sum(inputs[name], dtype=np.float64)) == pytest.approx(checksum, rel=1e-12, abs=1e-9)
            assert float(inputs[name].flat[0]) == info["input_first"][name]


def test_dense_chain_matches_reference_oracle(meta, arrays):
    for key, info in meta.items():
        if key.endswith("__sim"):
            continue
        dtype = key.split("__")[1]
        g = info["graph"]
        got = oracle.dense_chain(g["kind"], g["activation"], _inputs(g, info["seed"], dtype))
        ref = arrays[key + "__E"]
        tol = 1e-12 if dtype == "f64" else 1e-5
        assert oracle.max_relative_error(got, ref) <= tol, key


def test_replay_plan_matches_reference_execute_plan(meta, arrays):
    for key, info in meta.items():
        if not key.endswith("__sim"):
            continue
        name = key[: -len("__sim")]
        g = meta[name + "__f64"]["graph"]
        inputs = _inputs(g, 11, "f64")
        got = oracle.replay_plan(g["kind"], g["activation"], (g["m"], g["n"], g["k"], g["l"]), info["plan"], inputs)
        assert oracle.max_relative_error(got, arrays[key + "__E"]) <= 1e-12, key


def test_replay_plan_equals_dense_on_sampled_plans():
    """SPEC acceptance 5: sampled valid plans reproduce the dense chain (f64)."""
    with open(os.path.join(GOLD, "analyzer_samples.json")) as fh:
        samples = json.load(fh)
    for name, case in samples.items():
        g = case["graph"]
        inputs = oracle.make_inputs(g["kind"], g["m"], g["n"], g["k"], g["l"], seed=3, dtype=np.float64)
        ref = oracle.dense_chain(g["kind"], g["activation"], inputs)
        for row in case["plans"][:6]:
            got = oracle.replay_plan(g["kind"], g["activation"], (g["m"], g["n"], g["k"], g["l"]), row["plan"],
                                     inputs)
            err = oracle.max_relative_error(got, ref)
            assert err <= 1e-10, (name, row["plan"])
            # the reference's own replay error for the same plan is equally small
            assert row["sim_max_rel_error"] <= 1e-10


def test_bf16_rounding_is_round_to_nearest_even():
    x = np.array([1.0, 1.00390625, 1.005859375, -2.5, 3.0e-3, 65504.0], dtype=np.float32)
    import torch

    want = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    np.testing.assert_array_equal(oracle.round_bf16(x), want)


def test_gelu_tanh_matches_torch():
    import torch

    x = np.linspace(-6, 6, 1001).astype(np.float64)
    want = torch.nn.functional.gelu(torch.from_numpy(x), approximate="tanh").numpy()
    np.testing.assert_allclose(oracle.gelu_tanh(x), want, rtol=1e-12, atol=1e-12)
