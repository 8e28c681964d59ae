"""GPU parity: the sm_100a fused chain (through the C ABI / public API) against
the CPU oracle on the same seeded inputs.

Tolerance (north star): max-abs relative error <= 1e-2 against the fp32 chain
computed from the bf16-rounded inputs (simulator.py:143-147 metric).  The
oracle also rounds the intermediate C to bf16 (the GPU's dataflow); the
unrounded fp32 oracle is checked too at the same bound."""

import json
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
TOL = 1e-2
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _torch():
    import torch

    return torch


def _graph(kind, act, m, n, k, l):
    from paper_2512_12949_b200 import workload as W

    d = W.DimensionSpec(m, n, k, l, 2)
    return W.build_gated_ffn(d) if kind == "gated_ffn" else W.build_standard_ffn(d, act)


def _inputs(kind, m, n, k, l, seed, packed=True):
    torch = _torch()
    host = {name: oracle.round_bf16(v) for name, v in oracle.make_inputs(kind, m, n, k, l, seed=seed).items()}
    dev = {name: torch.from_numpy(v).cuda().to(torch.bfloat16) for name, v in host.items()}
    if kind == "gated_ffn" and packed:  # gate|up packed [2][K][N]
        w = torch.stack([dev["B0"], dev["B1"]])
        dev["B0"], dev["B1"] = w[0], w[1]
    return host, dev


def _check(kind, act, host, out):
    got = out.float().cpu().numpy()
    ref_b = oracle.dense_chain(kind, act, host, bf16_intermediate=True)
    ref = oracle.dense_chain(kind, act, host)
    err_b = oracle.max_relative_error(got, ref_b)
    err = oracle.max_relative_error(got, ref)
    assert np.isfinite(got).all()
    assert err_b <= TOL and err <= TOL, (err_b, err)
    return err_b


CASES = [
    ("standard_ffn", "relu", 256, 1024, 256, 1024),
    ("standard_ffn", "identity", 128, 512, 128, 256),
    ("standard_ffn", "silu", 256, 2048, 512, 512),
    ("standard_ffn", "gelu", 512, 3072, 768, 768),          # GPT-2 small FFN, full size
    ("gated_ffn", "silu", 256, 1024, 512, 512),
    ("gated_ffn", "silu", 512, 8192, 2048, 2048),           # LLaMA-1B SwiGLU, full size
    ("standard_ffn", "relu", 200, 768, 256, 768),           # ragged M (not a tile multiple)
    ("standard_ffn", "relu", 3136, 64, 576, 256),           # conv C5 implicit GEMM (im2col view)
    ("standard_ffn", "relu", 40, 256, 128, 256),            # M smaller than one tile
]


@pytest.mark.parametrize("exchange", ["dsm", "l2", "pair", "l2dsm"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-{c[1]}-{c[2]}x{c[3]}x{c[4]}x{c[5]}")
def test_fused_chain_matches_oracle(case, exchange):
    from paper_2512_12949_b200 import _native as nat
    from paper_2512_12949_b200 import runtime

    kind, act, m, n, k, l = case
    graph = _graph(kind, act, m, n, k, l)
    try:
        cfg = runtime.lower(graph, None, 148, exchange)
    except nat.UnsupportedPlan:
        pytest.skip(f"{exchange} has no lowering for {case}")
    host, dev = _inputs(kind, m, n, k, l, seed=17)
    out = runtime.launch(graph, cfg, dev)
    _torch().cuda.synchronize()
    _check(kind, act, host, out)
    # relaunch with the same workspace (epoch-stamped flags, reused scratch)
    out2 = runtime.launch(graph, cfg, dev)
    _torch().cuda.synchronize()
    assert _torch().equal(out, out2) or _check(kind, act, host, out2) <= TOL


@pytest.mark.parametrize("ring,splits,nb,lb,exchange", [(1, 1, 128, 256, "l2"), (2, 1, 128, 256, "dsm"),
                                                        (4, 2, 128, 256, "l2"), (8, 1, 128, 128, "dsm"),
                                                        (4, 1, 64, 256, "l2"), (3, 2, 256, 256, "pair"),
                                                        (4, 2, 256, 256, "pair")])
def test_explicit_configs(ring, splits, nb, lb, exchange):
    from paper_2512_12949_b200 import _native as nat
    from paper_2512_12949_b200 import runtime

    m, k = 256, 256
    l = ring * lb
    n = splits * ring * nb * 3
    graph = _graph("standard_ffn", "relu", m, n, k, l)
    cfg = nat.KernelConfig()
    cfg.ring, cfg.n_splits, cfg.nb, cfg.lb, cfg.exchange = ring, splits, nb, lb, runtime.EXCHANGES[exchange]
    host, dev = _inputs("standard_ffn", m, n, k, l, seed=ring * 10 + splits)
    out = runtime.launch(graph, cfg, dev)
    _torch().cuda.synchronize()
    _check("standard_ffn", "relu", host, out)


def test_intermediate_c_matches_oracle():
    """The bf16 intermediate the kernel materialises on chip equals act(A@B)."""
    torch = _torch()
    from paper_2512_12949_b200 import runtime

    graph = _graph("standard_ffn", "gelu", 256, 1024, 256, 512)
    host, dev = _inputs("standard_ffn", 256, 1024, 256, 512, seed=4)
    for exchange in ("dsm", "l2", "pair"):
        cfg = runtime.lower(graph, None, 148, exchange)
        c_dbg = torch.zeros((256, 1024), dtype=torch.bfloat16, device="cuda")
        runtime.launch(graph, cfg, dev, c_debug=c_dbg)
        torch.cuda.synchronize()
        c_ref = oracle.gelu_tanh(host["A"].astype(np.float64) @ host["B"])
        assert oracle.max_relative_error(c_dbg.float().cpu().numpy(), c_ref) <= TOL


def test_reference_plans_execute_through_public_api():
    """Top plans of the reference search (golden, B200 profile) run through
    execute_plan -- the drop-in for simulator.execute_plan -- with the traffic
    trace equal to the analyzer's prediction."""
    import paper_2512_12949_b200 as ff
    from paper_2512_12949_b200 import workload as W
    from paper_2512_12949_b200.hardware import b200_profile
    from paper_2512_12949_b200.plan import plan_from_dict

    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "search_results.json")))
    dev = b200_profile()
    ran = 0
    names = ("b200_gpt2s", "b200_llama1b", "b200_conv_c5", "b200_gpt67b", "b200_opt13b_m4096")
    for name in names:
        g = gold[name]["graph"]
        dims = W.DimensionSpec(g["m"], g["n"], g["k"], g["l"], 2)
        graph = W.build_gated_ffn(dims) if g["kind"] == "gated_ffn" else W.build_standard_ffn(
            dims, g["activation"], logical_m=g.get("logical_m"))
        plan = plan_from_dict(gold[name]["result"]["top"][0]["plan"])
        inputs = ff.make_inputs(graph, ff.SimConfig(seed=2, max_workspace_bytes=8 << 30))
        rounded = {k: oracle.round_bf16(v) for k, v in inputs.items()}
        # the full-size chains exceed execute_plan's default 1 GiB host-tensor guard (simulator.py:198)
        out, trace = ff.execute_plan(plan, graph, rounded, ff.SimConfig(max_workspace_bytes=8 << 30), dev)
        ref = oracle.dense_chain(graph.kind, graph.activation, rounded)
        assert oracle.max_relative_error(out, ref) <= TOL, name
        assert trace.tier_bytes == ff.analyze(graph, dev, plan).volume
        ran += 1
    assert ran == len(names)


def test_verify_report():
    import paper_2512_12949_b200 as ff
    from paper_2512_12949_b200.hardware import b200_profile
    from paper_2512_12949_b200.plan import make_plan

    graph = ff.build_gated_ffn(ff.DimensionSpec(256, 1024, 512, 512))
    plan = make_plan("n", "klm", (64, 128, 1024, 256), (1, 2, 1, 2), "doubled_k")
    rep = ff.verify(plan, graph, ff.SimConfig(seed=9), device=b200_profile())
    assert rep.passed, rep.to_dict()


@pytest.mark.parametrize("name", ["gpt67b", "opt13b_m4096"])
def test_large_baseline_configs(name):
    """Full BASELINE sizes against the CPU oracle (f32 numpy)."""
    import bench
    from paper_2512_12949_b200 import runtime

    kind, act, m, n, k, l, _ = bench.WORKLOADS[name]
    graph = _graph(kind, act, m, n, k, l)
    host, dev = _inputs(kind, m, n, k, l, seed=23)
    out = runtime.run(graph, None, dev)
    _torch().cuda.synchronize()
    _check(kind, act, host, out)


def test_two_streams_and_rejections():
    torch = _torch()
    from paper_2512_12949_b200 import runtime

    graph = _graph("standard_ffn", "relu", 256, 1024, 256, 1024)
    host, dev = _inputs("standard_ffn", 256, 1024, 256, 1024, seed=5)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s1):
        o1 = runtime.run(graph, None, dev, stream=s1, exchange="dsm")
    with torch.cuda.stream(s2):
        o2 = runtime.run(graph, None, dev, stream=s2, exchange="dsm")
    torch.cuda.synchronize()
    _check("standard_ffn", "relu", host, o1)
    _check("standard_ffn", "relu", host, o2)
    with pytest.raises(ValueError):
        bad = dict(dev)
        bad["A"] = dev["A"].float()
        runtime.run(graph, None, bad)
    with pytest.raises(ValueError):
        bad = dict(dev)
        bad["D"] = dev["D"].t()
        runtime.run(graph, None, bad)


@pytest.mark.parametrize("exchange,ring,splits,nb,lb", [("pair", 2, 4, 256, 256), ("l2", 2, 3, 128, 256),
                                                        ("dsm", 2, 2, 128, 128)])
def test_split_reduction_leaves_workspace_zero(exchange, ring, splits, nb, lb):
    """The last of the S contributors of an E tile casts it and re-zeroes the fp32
    tile and its arrival counter, so a workspace zero-filled once stays valid."""
    from paper_2512_12949_b200 import _native as nat
    from paper_2512_12949_b200 import runtime

    torch = _torch()
    m, k = 300, 256
    l = ring * lb
    n = splits * ring * nb * 2
    graph = _graph("standard_ffn", "relu", m, n, k, l)
    cfg = nat.KernelConfig()
    cfg.ring, cfg.n_splits, cfg.nb, cfg.lb = ring, splits, nb, lb
    cfg.exchange = {"dsm": nat.XCHG_DSM, "l2": nat.XCHG_L2, "pair": nat.XCHG_L2_PAIR}[exchange]
    host, dev = _inputs("standard_ffn", m, n, k, l, seed=23)
    for _ in range(3):
        out = runtime.launch(graph, cfg, dev)
        torch.cuda.synchronize()
        assert _check("standard_ffn", "relu", host, out) <= TOL
    stream = torch.cuda.current_stream()
    ws = runtime._workspaces[(torch.cuda.current_device(), int(stream.cuda_stream))]
    lo, hi = 1 << 20, (1 << 20) + (256 << 10) + m * l * 4
    assert int(ws[lo:hi].count_nonzero()) == 0


# pair-kernel variants (ff_set_variant): common GEMM0 k order, plain pair kernel, forced quads
@pytest.mark.parametrize("mode", [0x1, 0x2, 0x4, 0x10, 0x60], ids=["no-krot", "no-quad", "force-quad", "w-evict-first", "w-evict-last-c-normal"])
@pytest.mark.parametrize("case", [("gated_ffn", "silu", 512, 8192, 2048, 2048),
                                  ("standard_ffn", "relu", 512, 16384, 4096, 4096)], ids=["llama1b", "gpt67b"])
def test_pair_kernel_variants_match_oracle_and_repeat_bitwise(case, mode):
    torch = _torch()
    from paper_2512_12949_b200 import _native as nat
    from paper_2512_12949_b200 import runtime

    kind, act, m, n, k, l = case
    graph = _graph(kind, act, m, n, k, l)
    host, dev = _inputs(kind, m, n, k, l, seed=11)
    lib = nat.load()
    lib.ff_set_variant(mode)
    try:
        cfg = runtime.lower(graph, None, 148, "pair")
        out1 = runtime.launch(graph, cfg, dev).clone()
        out2 = runtime.launch(graph, cfg, dev)
        torch.cuda.synchronize()
    finally:
        lib.ff_set_variant(0)
    _check(kind, act, host, out1)
    assert torch.equal(out1, out2), "split-N reductions must be deterministic"


# serpentine n-step order (odd units of a ring walk their n-steps backwards) against the
# common order: both match the oracle (OPT M=4096: 16 units on 9 rings)
@pytest.mark.parametrize("mode", [0x0, 0x200], ids=["serpentine", "no-serp"])
def test_pair_kernel_serpentine_units_match_oracle(mode):
    torch = _torch()
    from paper_2512_12949_b200 import _native as nat
    from paper_2512_12949_b200 import runtime

    kind, act, m, n, k, l = "standard_ffn", "relu", 4096, 8192, 2048, 2048
    graph = _graph(kind, act, m, n, k, l)
    host, dev = _inputs(kind, m, n, k, l, seed=13)
    lib = nat.load()
    lib.ff_set_variant(mode)
    try:
        cfg = runtime.lower(graph, None, 148, "pair")
        assert cfg.units > cfg.rings
        out = runtime.launch(graph, cfg, dev)
        torch.cuda.synchronize()
    finally:
        lib.ff_set_variant(0)
    _check(kind, act, host, out)


# tail split: the last partial wave's units are cut in N across the idle rings and combined by the
# split-N reduce-scatter (11 units of 4 n-steps on 9 rings: 9 whole units + 2 x 4 quarter units),
# against the oracle with and without it, and bitwise repeatable
@pytest.mark.parametrize("mode", [0x0, 0x800], ids=["tail-split", "no-tail-split"])
@pytest.mark.parametrize("case", [("standard_ffn", "relu", 11 * 256, 8192, 512, 2048),   # 2 x 4 quarters of 1 n-step
                                  ("gated_ffn", "silu", 11 * 256, 8192, 512, 2048)],     # 2 x 4 quarters of 2 n-steps
                         ids=["standard", "gated"])
def test_pair_kernel_tail_split_matches_oracle(case, mode):
    torch = _torch()
    from paper_2512_12949_b200 import _native as nat
    from paper_2512_12949_b200 import runtime

    kind, act, m, n, k, l = case
    graph = _graph(kind, act, m, n, k, l)
    host, dev = _inputs(kind, m, n, k, l, seed=17)
    lib = nat.load()
    lib.ff_set_variant(mode)
    try:
        cfg = runtime.lower(graph, None, 148, "pair")
        assert cfg.units == 11 and cfg.rings == 9
        out1 = runtime.launch(graph, cfg, dev).clone()
        out2 = runtime.launch(graph, cfg, dev)
        torch.cuda.synchronize()
    finally:
        lib.ff_set_variant(0)
    _check(kind, act, host, out1)
    assert torch.equal(out1, out2), "the tail split's reduce-scatter must be deterministic"


def _random_cases(n, seed):
    rng = __import__("random").Random(seed)
    cases = []
    for _ in range(n):
        kind = rng.choice(["standard_ffn", "gated_ffn"])
        act = "silu" if kind == "gated_ffn" else rng.choice(["relu", "identity", "silu", "gelu"])
        m = rng.choice([16, 17, 64, 128, 200, 256, 384, 640])
        k = 128 * rng.randint(1, 12)
        n = 256 * rng.randint(1, 16)
        l = 256 * rng.randint(1, 8)
        cases.append((kind, act, m, n, k, l))
    return cases


@pytest.mark.parametrize("exchange", ["dsm", "l2", "pair", "l2dsm"])
@pytest.mark.parametrize("case", _random_cases(10, 2025), ids=lambda c: f"{c[0][:3]}-{c[1]}-{c[2]}x{c[3]}x{c[4]}x{c[5]}")
def test_random_shapes_match_oracle(case, exchange):
    """Seeded random shapes (ragged M down to 16, K in 128s, N/L in 256s) under every transport."""
    from paper_2512_12949_b200 import _native as nat
    from paper_2512_12949_b200 import runtime

    kind, act, m, n, k, l = case
    graph = _graph(kind, act, m, n, k, l)
    try:
        cfg = runtime.lower(graph, None, 148, exchange)
    except nat.UnsupportedPlan:
        pytest.skip(f"{exchange} has no lowering for {case}")
    host, dev = _inputs(kind, m, n, k, l, seed=3)
    out = runtime.launch(graph, cfg, dev)
    _torch().cuda.synchronize()
    _check(kind, act, host, out)


# ragged n-steps of the pair kernel: ceil(chunks / S) chunks per N split, so the last
# n-step (and the last split) may be short; `total` = N / nb chunks
@pytest.mark.parametrize("kind,ring,splits,total", [("standard_ffn", 4, 1, 5), ("standard_ffn", 4, 2, 6),
                                                    ("standard_ffn", 3, 2, 7), ("standard_ffn", 6, 1, 1),
                                                    ("standard_ffn", 2, 4, 11), ("gated_ffn", 4, 2, 9),
                                                    ("gated_ffn", 3, 4, 13)])
def test_pair_ragged_steps_match_oracle(kind, ring, splits, total):
    torch = _torch()
    from paper_2512_12949_b200 import _native as nat
    from paper_2512_12949_b200 import runtime

    act = "silu" if kind == "gated_ffn" else "gelu"
    nb = 128 if kind == "gated_ffn" else 256
    m, k, lb = 384, 256, 256
    l, n = ring * lb, total * nb
    graph = _graph(kind, act, m, n, k, l)
    cfg = nat.KernelConfig()
    cfg.ring, cfg.n_splits, cfg.nb, cfg.lb, cfg.exchange = ring, splits, nb, lb, runtime.EXCHANGES["pair"]
    host, dev = _inputs(kind, m, n, k, l, seed=ring + 7 * total)
    out1 = runtime.launch(graph, cfg, dev).clone()
    out2 = runtime.launch(graph, cfg, dev)
    torch.cuda.synchronize()
    _check(kind, act, host, out1)
    assert torch.equal(out1, out2)


@pytest.mark.parametrize("case", [("gated_ffn", "silu", 512, 11008, 4096, 4096),     # LLaMA-7B (reference preset S3)
                                  ("standard_ffn", "relu", 256, 8960, 1536, 1536)], ids=["llama7b", "ragged-std"])
def test_auto_lowering_with_ragged_ring(case):
    """Shapes whose chunks do not fill the widest ring lower to a ragged pair ring."""
    from paper_2512_12949_b200 import runtime

    kind, act, m, n, k, l = case
    graph = _graph(kind, act, m, n, k, l)
    cfg = runtime.lower(graph, None, 148, "pair")
    assert n != cfg.n_splits * cfg.steps * cfg.ring * cfg.nb and cfg.l_clusters == 1
    host, dev = _inputs(kind, m, n, k, l, seed=5)
    out = runtime.launch(graph, cfg, dev)
    _torch().cuda.synchronize()
    _check(kind, act, host, out)


def test_pair_many_splits_small_m():
    """Tiny M with a wide N lowers to 32 N splits of a ring of one pair; the tail's
    exchange-region maps (unused beyond 8 splits) once got an illegal zero-row box
    (found by tests/_fuzz_gpu.py)."""
    from paper_2512_12949_b200 import runtime

    kind, act, m, n, k, l = "gated_ffn", "silu", 40, 4096, 768, 256
    graph = _graph(kind, act, m, n, k, l)
    cfg = runtime.lower(graph, None, 148, "pair")
    assert cfg.n_splits > 8
    host, dev = _inputs(kind, m, n, k, l, seed=31)
    out = runtime.launch(graph, cfg, dev)
    _torch().cuda.synchronize()
    _check(kind, act, host, out)


def test_workspace_zero_invariant_across_configs():
    """The split counters and the fp32 E zone of the shared per-stream workspace
    are zero after every launch (configs reuse one workspace; a config whose
    regions overlapped the zone once corrupted the next split chain)."""
    torch = _torch()
    from paper_2512_12949_b200 import _native as nat
    from paper_2512_12949_b200 import runtime

    seq = [("gated_ffn", "silu", 128, 3328, 256, 1792), ("standard_ffn", "relu", 200, 768, 256, 768),
           ("gated_ffn", "silu", 384, 768, 1536, 1792), ("standard_ffn", "gelu", 512, 3072, 768, 768)]
    for case in seq:
        for exchange in ("pair", "l2", "dsm", "l2dsm"):
            graph = _graph(*case)
            try:
                cfg = runtime.lower(graph, None, 148, exchange)
            except nat.UnsupportedPlan:
                continue
            host, dev = _inputs(case[0], *case[2:], seed=5)
            out = runtime.launch(graph, cfg, dev)
            torch.cuda.synchronize()
            _check(case[0], case[1], host, out)
            for ws in runtime._workspaces.values():
                cnt = ws[(1 << 20):(1 << 20) + (256 << 10)]
                zone = ws[(1 << 20) + (256 << 10):(1 << 20) + (256 << 10) + (32 << 20)]
                assert int((cnt != 0).sum()) == 0 and int((zone != 0).sum()) == 0, (case, exchange, cfg.as_dict())


F16_CASES = [
    ("gated_ffn", "silu", 512, 8192, 2048, 2048),      # LLaMA-1B shape
    ("standard_ffn", "relu", 512, 16384, 4096, 4096),  # GPT-6.7B shape
    ("standard_ffn", "gelu", 200, 768, 256, 768),
]


@pytest.mark.parametrize("exchange", ["dsm", "l2", "pair", "l2dsm"])
@pytest.mark.parametrize("case", F16_CASES, ids=lambda c: f"{c[0][:3]}-{c[1]}-{c[2]}x{c[3]}x{c[4]}x{c[5]}")
def test_fp16_chain_matches_oracle(case, exchange):
    """fp16 storage (north star: bf16/fp16 with fp32 accumulation).  Weights are
    scaled by 1/sqrt(fan-in) so C and E stay inside the fp16 range."""
    torch = _torch()
    from paper_2512_12949_b200 import _native as nat
    from paper_2512_12949_b200 import runtime

    kind, act, m, n, k, l = case
    graph = _graph(kind, act, m, n, k, l)
    try:
        cfg = runtime.lower(graph, None, 148, exchange)
    except nat.UnsupportedPlan:
        pytest.skip(f"{exchange} has no lowering for {case}")
    raw = oracle.make_inputs(kind, m, n, k, l, seed=4)
    scale = {"A": 1.0, "B": k ** -0.5, "B0": k ** -0.5, "B1": k ** -0.5, "D": n ** -0.5}
    host = {name: oracle.round_f16(v * scale[name]) for name, v in raw.items()}
    dev = {name: torch.from_numpy(v).cuda().to(torch.float16) for name, v in host.items()}
    out = runtime.launch(graph, cfg, dev)
    torch.cuda.synchronize()
    assert out.dtype == torch.float16
    got = out.float().cpu().numpy()
    ref_h = oracle.dense_chain(kind, act, host, f16_intermediate=True)
    ref = oracle.dense_chain(kind, act, host)
    assert np.isfinite(got).all()
    assert oracle.max_relative_error(got, ref_h) <= TOL and oracle.max_relative_error(got, ref) <= TOL


@pytest.mark.parametrize("exchange", ["dsm", "l2"])
@pytest.mark.parametrize("case", [("standard_ffn", "gelu", 512, 3072, 768, 768), ("gated_ffn", "silu", 256, 1024, 512, 512)],
                         ids=["gpt2s", "gated-small"])
def test_one_cta_region_finish_matches_oracle_and_repeats_bitwise(case, exchange):
    """1-CTA kernels' opt-in split-N reduce-scatter through exchange regions (FF_VARIANT_FINISH_REGIONS)."""
    torch = _torch()
    from paper_2512_12949_b200 import _native as nat
    from paper_2512_12949_b200 import runtime

    kind, act, m, n, k, l = case
    graph = _graph(kind, act, m, n, k, l)
    cfg = runtime.lower(graph, None, 148, exchange)
    assert cfg.n_splits > 1
    host, dev = _inputs(kind, m, n, k, l, seed=12)
    lib = nat.load()
    lib.ff_set_variant(0x8)
    try:
        out1 = runtime.launch(graph, cfg, dev).clone()
        out2 = runtime.launch(graph, cfg, dev)
        torch.cuda.synchronize()
    finally:
        lib.ff_set_variant(0)
    _check(kind, act, host, out1)
    assert torch.equal(out1, out2)


@pytest.mark.parametrize("splits", [2, 4, 8])
@pytest.mark.parametrize("case", [("standard_ffn", "gelu", 512, 3072, 768, 768), ("gated_ffn", "silu", 256, 1024, 512, 512),
                                  ("standard_ffn", "relu", 200, 2048, 256, 512)],
                         ids=["gpt2s", "gated-small", "ragged-m"])
def test_dsm_reduce_scatter_matches_oracle_and_repeats_bitwise(case, splits):
    """FF_XCHG_L2_DSMR: the N splits of an E tile form one thread-block cluster and sum
    their fp32 partials by a DSM reduce-scatter (st.shared::cluster into the owner's
    drained stages, split-order sum): matches the oracle and is bit-reproducible."""
    torch = _torch()
    from paper_2512_12949_b200 import _native as nat
    from paper_2512_12949_b200 import runtime

    kind, act, m, n, k, l = case
    graph = _graph(kind, act, m, n, k, l)
    cfg = runtime.lower(graph, None, 148, "l2dsm")
    cfg.n_splits = splits
    host, dev = _inputs(kind, m, n, k, l, seed=13)
    try:
        out1 = runtime.launch(graph, cfg, dev).clone()
    except nat.UnsupportedPlan as exc:
        pytest.skip(f"{splits} splits do not tile {case}: {exc}")
    out2 = runtime.launch(graph, cfg, dev)
    torch.cuda.synchronize()
    _check(kind, act, host, out1)
    assert torch.equal(out1, out2)


@pytest.mark.parametrize("exchange,case", [("pair", ("gated_ffn", "silu", 512, 8192, 2048, 2048)),
                                           ("l2", ("gated_ffn", "silu", 512, 8192, 2048, 2048)),
                                           ("dsm", ("gated_ffn", "silu", 512, 8192, 2048, 2048)),
                                           # multi-unit rings (16 units on 9 rings): unit-boundary reorder
                                           ("pair", ("standard_ffn", "relu", 4096, 2048, 512, 2048)),
                                           # ragged ring (N = 11 chunks on a ring of 4 pairs)
                                           ("pair", ("standard_ffn", "gelu", 384, 2816, 256, 1024))],
                         ids=["pair", "l2", "dsm", "pair-multi-unit", "pair-ragged"])
def test_cuda_graph_capture_replays_the_chain(exchange, case):
    """Stream capture of runtime.launch (no host sync, caller-owned workspace per
    stream).  Every replay must see a fresh launch epoch (kept on the device): the
    inputs change between replays, so a stale ready flag would leak the previous
    replay's intermediate into the result."""
    torch = _torch()
    from paper_2512_12949_b200 import runtime

    kind, act, m, n, k, l = case
    graph = _graph(kind, act, m, n, k, l)
    cfg = runtime.lower(graph, None, 148, exchange)
    host, dev = _inputs(kind, m, n, k, l, seed=21)
    out = torch.empty((m, l), dtype=torch.bfloat16, device="cuda")
    a_static = dev["A"]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        runtime.launch(graph, cfg, dev, out=out, stream=st)  # workspace for this stream exists before capture
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            runtime.launch(graph, cfg, dev, out=out, stream=st)
        for seed in (31, 32, 33):
            new_a = oracle.round_bf16(oracle.make_inputs(kind, m, n, k, l, seed=seed)["A"])
            a_static.copy_(torch.from_numpy(new_a).to(torch.bfloat16))
            g.replay()
            st.synchronize()
            _check(kind, act, dict(host, A=new_a), out)


# deterministic mode (runtime.lower(..., deterministic=True), ff_config_deterministic): the
# selected launch matches the oracle and writes a bit-identical E on repeated runs, also when
# other launches (the reduce-add lowerings) run in between and perturb the timing
@pytest.mark.parametrize("case", [("standard_ffn", "gelu", 512, 3072, 768, 768),
                                  ("gated_ffn", "silu", 512, 8192, 2048, 2048),
                                  ("standard_ffn", "relu", 1024, 4096, 1024, 1024),
                                  ("standard_ffn", "relu", 200, 768, 256, 768)],
                         ids=["gpt2s", "llama1b", "std-1024", "ragged-m"])
@pytest.mark.parametrize("exchange", ["auto", "l2dsm"])
def test_deterministic_mode_matches_oracle_and_repeats_bitwise(case, exchange):
    torch = _torch()
    from paper_2512_12949_b200 import _native as nat
    from paper_2512_12949_b200 import runtime

    kind, act, m, n, k, l = case
    graph = _graph(kind, act, m, n, k, l)
    host, dev = _inputs(kind, m, n, k, l, seed=23)
    try:
        cfg = runtime.lower(graph, None, 148, exchange, deterministic=True)
    except nat.UnsupportedPlan:
        pytest.skip(f"no bit-reproducible {exchange} lowering for this shape")
    assert runtime.is_deterministic(graph, cfg)
    first = runtime.launch(graph, cfg, dev).clone()
    _check(kind, act, host, first)
    other = runtime.lower(graph, None, 148, "l2")
    for _ in range(4):
        runtime.launch(graph, other, dev)  # a reduce-add lowering in between
        again = runtime.launch(graph, cfg, dev)
        torch.cuda.synchronize()
        assert torch.equal(first, again), "deterministic launch changed its result"


@pytest.mark.parametrize("case", [("standard_ffn", "gelu", 512, 3072, 768, 768),
                                  ("gated_ffn", "silu", 256, 2048, 512, 512)], ids=["gpt2s", "gated-small"])
def test_deterministic_mode_fp16_repeats_bitwise(case):
    """fp16 storage through the reproducible launches: the oracle bound and bitwise repeats."""
    torch = _torch()
    from paper_2512_12949_b200 import runtime

    kind, act, m, n, k, l = case
    graph = _graph(kind, act, m, n, k, l)
    raw = oracle.make_inputs(kind, m, n, k, l, seed=8)
    scale = {"A": 1.0, "B": k ** -0.5, "B0": k ** -0.5, "B1": k ** -0.5, "D": n ** -0.5}
    host = {name: oracle.round_f16(v * scale[name]) for name, v in raw.items()}
    dev = {name: torch.from_numpy(v).cuda().to(torch.float16) for name, v in host.items()}
    for cfg in runtime.reproducible_configs(graph)[:3] + [runtime.lower(graph, None, 148, "auto", deterministic=True)]:
        assert runtime.is_deterministic(graph, cfg)
        first = runtime.launch(graph, cfg, dev).clone()
        again = runtime.launch(graph, cfg, dev)
        torch.cuda.synchronize()
        assert first.dtype == torch.float16 and torch.equal(first, again), cfg.as_dict()
        got = first.float().cpu().numpy()
        assert oracle.max_relative_error(got, oracle.dense_chain(kind, act, host, f16_intermediate=True)) <= TOL
