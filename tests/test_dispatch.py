"""Run-time M-bin dispatch table: bin lookup and table
round trip on CPU; dispatch of ragged M through the shipped tables on the GPU."""

import numpy as np
import pytest

import oracle
from paper_2512_12949_b200 import dispatch


def test_shipped_tables_cover_the_baseline_families():
    for name, (kind, act, n, k, l) in dispatch.FAMILIES.items():
        t = dispatch.shipped(name)
        assert (t.kind, t.activation, t.n, t.k, t.l) == (kind, act, n, k, l)
        assert t.bins == sorted(t.bins) and len(t.configs) == len(t.bins)
        for c in t.configs:
            assert c["exchange"] in (0, 1, 2, 3) and c["ring"] >= 1 and c["n_splits"] >= 1 and c["ms"] > 0


def test_bin_lookup_and_round_trip(tmp_path):
    t = dispatch.shipped("llama1b")
    assert t.bin_of(1) == 0 and t.bin_of(64) == 0 and t.bin_of(65) == 1 and t.bin_of(8192) == len(t.bins) - 1
    with pytest.raises(ValueError):
        t.bin_of(t.bins[-1] + 1)
    p = tmp_path / "t.json"
    t.save(str(p))
    u = dispatch.Dispatcher.load(str(p))
    assert u.to_dict() == t.to_dict()
    cfg = u.config_for(300)
    assert (cfg.ring, cfg.n_splits, cfg.exchange) == tuple(t.configs[t.bin_of(300)][f] for f in ("ring", "n_splits",
                                                                                                   "exchange"))


@pytest.mark.gpu
@pytest.mark.parametrize("name,m", [("llama1b", 300), ("llama1b", 40), ("gpt2s", 777), ("opt13b", 1500)])
def test_dispatch_ragged_m_matches_oracle(name, m):
    import torch

    t = dispatch.shipped(name)
    kind = t.kind
    host = {k: oracle.round_bf16(v) for k, v in oracle.make_inputs(kind, m, t.n, t.k, t.l, seed=9).items()}
    dev = {k: torch.from_numpy(v).cuda().to(torch.bfloat16) for k, v in host.items()}
    out = t.run(dev)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    ref = oracle.dense_chain(kind, t.activation, host, bf16_intermediate=True)
    assert np.isfinite(got).all() and oracle.max_relative_error(got, ref) <= 1e-2


def test_deterministic_candidates_are_reproducible():
    """A reproducible-serving table draws only on bit-reproducible launches (host logic)."""
    from paper_2512_12949_b200 import runtime

    for name, m in (("gpt2s", 512), ("llama1b", 512), ("opt13b", 4096)):
        kind, act, n, k, l = dispatch.FAMILIES[name]
        g = dispatch.family_graph(kind, act, m, n, k, l)
        every = dispatch.candidate_configs(g)
        det = dispatch.candidate_configs(g, deterministic=True)
        assert det and len(det) <= len(every)
        assert all(runtime.is_deterministic(g, c) for c in det)
    g = dispatch.family_graph("standard_ffn", "gelu", 512, 3072, 768, 768)
    assert len(dispatch.candidate_configs(g, deterministic=True)) < len(dispatch.candidate_configs(g))


@pytest.mark.gpu
def test_reproducible_table_build_and_run():
    """build_table(deterministic=True) profiles only bit-reproducible launches; its run() repeats bitwise."""
    import torch

    from paper_2512_12949_b200 import runtime

    t = dispatch.build_table("standard_ffn", "gelu", 3072, 768, 768, bins=(128, 512), iters=3, warmup=1,
                             plans_by_m={}, deterministic=True)
    for b in t.bins:
        assert runtime.is_deterministic(t.graph_for(b), t.config_for(b))
    m = 300
    host = {k: oracle.round_bf16(v) for k, v in oracle.make_inputs("standard_ffn", m, 3072, 768, 768, seed=4).items()}
    dev = {k: torch.from_numpy(v).cuda().to(torch.bfloat16) for k, v in host.items()}
    first = t.run(dev).clone()
    again = t.run(dev)
    torch.cuda.synchronize()
    assert torch.equal(first, again)
    ref = oracle.dense_chain("standard_ffn", "gelu", host, bf16_intermediate=True)
    assert oracle.max_relative_error(first.float().cpu().numpy(), ref) <= 1e-2


def test_pick_reproducible_tie_rule():
    """The fastest launch wins unless a bit-reproducible one is within dispatch.TIE of it (host logic)."""
    from paper_2512_12949_b200 import runtime

    g = dispatch.family_graph("standard_ffn", "gelu", 512, 3072, 768, 768)
    fast = runtime.lower(g, None, 148, "dsm")           # N splits summed by reduce-adds
    det = runtime.explicit_config(g, 6, 4, 128, 128, "l2dsm")
    assert not runtime.is_deterministic(g, fast) and runtime.is_deterministic(g, det)
    assert dispatch.pick_reproducible(g, [(1.000, fast, "a"), (1.005, det, "b")])[1] is det
    assert dispatch.pick_reproducible(g, [(1.000, fast, "a"), (1.050, det, "b")])[1] is fast
    assert dispatch.pick_reproducible(g, [(1.000, det, "b"), (1.001, fast, "a")])[1] is det
