"""Conv chains (ConvChainConfig, workload.py:168-199): conv(k1 x k1, same) ->
ReLU -> conv(1 x 1) executed as an implicit GEMM (im2col TMA) by the fused
sm_100a kernel, checked against the CPU oracle: the reference's GEMM-chain
view of the conv (dense_chain over the im2col matrix, simulator.py:126-134).

The im2col restatement itself has no reference counterpart (the reference
feeds a random im2col matrix), so it is pinned against torch's direct
convolution (fp32, CPU) instead.  Tolerance: 1e-2 max-abs relative error."""

import numpy as np
import pytest

import oracle

TOL = 1e-2

# reference presets (workload.py:207-240) and small shapes: (ic, h, w, oc1, oc2, k1, k2, batch)
GPU_CASES = [
    ("C5", (64, 56, 56, 64, 256, 3, 1), 1),
    ("C6", (128, 28, 28, 128, 512, 3, 1), 1),
    ("C7", (256, 14, 14, 256, 1024, 3, 1), 1),
    ("C8", (512, 7, 7, 512, 2048, 3, 1), 1),
    ("C1", (64, 56, 56, 256, 64, 1, 1), 1),
    ("C4", (512, 7, 7, 2048, 512, 1, 1), 1),
    ("b2-5x5", (64, 9, 13, 128, 256, 5, 1), 2),
    ("b3-ragged", (128, 11, 10, 64, 128, 3, 1), 3),
]


def _conv_inputs(ic, h, w, oc1, oc2, k1, batch, seed=0, k2=1):
    rng = np.random.default_rng(seed)
    x = oracle.round_bf16(rng.uniform(-1, 1, (batch, h, w, ic)).astype(np.float32))
    w1 = oracle.round_bf16((rng.uniform(-1, 1, (k1, k1, ic, oc1)) / np.sqrt(k1 * k1 * ic)).astype(np.float32))
    w2_shape = (oc1, oc2) if k2 == 1 else (k2, k2, oc1, oc2)
    w2 = oracle.round_bf16((rng.uniform(-1, 1, w2_shape) / np.sqrt(k2 * k2 * oc1)).astype(np.float32))
    return x, w1, w2


# extension: 1x1 conv -> ReLU -> k2 x k2 conv (ResNet bottleneck order, BASELINE.json configs[3])
BLOCK_CASES = [
    ("resnet-c2x-56", (256, 56, 56, 64, 64, 1, 3), 1),
    ("resnet-c3x-28", (512, 28, 28, 128, 128, 1, 3), 1),
    ("b2-5x5-ragged", (128, 9, 11, 64, 256, 1, 5), 2),
    ("b1-3x3-tiny", (64, 5, 6, 128, 64, 1, 3), 1),
]


@pytest.mark.parametrize("k2", [3, 5])
def test_block_oracle_matches_direct_conv(k2):
    torch = pytest.importorskip("torch")
    x, w1, w2 = _conv_inputs(16, 7, 9, 24, 8, 1, 2, seed=k2, k2=k2)
    got = oracle.conv_chain(x, w1, w2, "relu")
    xt = torch.from_numpy(x).permute(0, 3, 1, 2).double()
    c = torch.nn.functional.conv2d(xt, torch.from_numpy(w1).permute(3, 2, 0, 1).double()).relu()
    y = torch.nn.functional.conv2d(c, torch.from_numpy(w2).permute(3, 2, 0, 1).double(), padding=k2 // 2)
    assert oracle.max_relative_error(got, y.permute(0, 2, 3, 1).numpy()) < 1e-5


def test_block_config_rules():
    from paper_2512_12949_b200 import runtime, workload as W
    from paper_2512_12949_b200 import _native as nat
    from paper_2512_12949_b200.errors import UnsupportedConvChain

    with pytest.raises(UnsupportedConvChain):  # the reference's class keeps its k2 == 1 rule
        W.ConvChainConfig(64, 8, 8, 64, 64, 1, 3)
    with pytest.raises(UnsupportedConvChain):
        W.ConvBlockConfig(64, 8, 8, 64, 64, 3, 3)
    cfg = runtime.lower_conv(W.ConvBlockConfig(256, 56, 56, 64, 64, 1, 3), exchange="l2")
    assert (cfg.ring, cfg.n_splits, cfg.nb, cfg.lb, cfg.units) == (1, 1, 64, 64, 25)
    for exchange in ("dsm", "pair"):
        with pytest.raises(nat.UnsupportedPlan):
            runtime.lower_conv(W.ConvBlockConfig(256, 56, 56, 64, 64, 1, 3), exchange=exchange)
    from paper_2512_12949_b200.errors import CapacityExceeded

    with pytest.raises(CapacityExceeded) as info:  # the whole intermediate of a tile: oc1 <= 128
        runtime.lower_conv(W.ConvBlockConfig(256, 14, 14, 256, 64, 1, 3), exchange="l2")
    assert (info.value.tensor, info.value.floor, info.value.unplaced) == ("C", "smem", 128 * 128 * 2)


@pytest.mark.parametrize("k1", [1, 3, 5])
def test_im2col_oracle_matches_direct_conv(k1):
    torch = pytest.importorskip("torch")
    x, w1, w2 = _conv_inputs(16, 7, 9, 24, 8, k1, 2, seed=k1)
    got = oracle.conv_chain(x, w1, w2, "relu")
    xt = torch.from_numpy(x).permute(0, 3, 1, 2).double()
    c = torch.nn.functional.conv2d(xt, torch.from_numpy(w1).permute(3, 2, 0, 1).double(), padding=k1 // 2).relu()
    y = torch.nn.functional.conv2d(c, torch.from_numpy(w2).t().double()[:, :, None, None])
    ref = y.permute(0, 2, 3, 1).numpy()
    assert oracle.max_relative_error(got, ref) < 1e-5


def test_conv_lowering_matches_reference_gemm_view():
    """ff_conv_chain_desc gives the reference's conv_chain_to_gemm dims (unpadded m)."""
    import ctypes

    from paper_2512_12949_b200 import _native as nat
    from paper_2512_12949_b200 import runtime, workload as W

    lib = nat.load()
    for pid in ("C5", "C6", "C7", "C8", "C1"):
        g = W.preset(pid)
        cfg = W.ConvChainConfig(*W._PRESETS_CONV[pid])
        ch = nat.ChainDesc()
        nat.check(lib.ff_conv_chain_desc(ctypes.byref(runtime.conv_desc(cfg)), ctypes.byref(ch)))
        assert (ch.n, ch.k, ch.l) == (g.dims.n, g.dims.k, g.dims.l)
        assert ch.m == cfg.h * cfg.w and g.dims.m == -(-ch.m // 16) * 16
    with pytest.raises(nat.UnsupportedPlan):  # implicit GEMM needs 64-channel blocks
        runtime.lower_conv(W.ConvChainConfig(48, 8, 8, 64, 64, 3, 1), exchange="dsm")
    with pytest.raises(nat.UnsupportedPlan):  # im2col runs on the 1-CTA kernels only
        runtime.lower_conv(W.ConvChainConfig(64, 8, 8, 64, 256, 3, 1), exchange="pair")


@pytest.mark.gpu
@pytest.mark.parametrize("exchange", ["dsm", "l2", "pair"])
@pytest.mark.parametrize("case", GPU_CASES, ids=lambda c: c[0])
def test_conv_chain_matches_oracle(case, exchange):
    import torch

    from paper_2512_12949_b200 import _native as nat
    from paper_2512_12949_b200 import runtime, workload as W

    name, shape, batch = case
    cfg = W.ConvChainConfig(*shape)
    ic, h, w, oc1, oc2, k1, _ = shape
    try:
        kcfg = runtime.lower_conv(cfg, batch, exchange)
    except nat.UnsupportedPlan:
        pytest.skip(f"{exchange} has no lowering for {name}")
    x, w1, w2 = _conv_inputs(ic, h, w, oc1, oc2, k1, batch, seed=7)
    dev = [torch.from_numpy(a).cuda().to(torch.bfloat16).contiguous() for a in (x, w1, w2)]
    for _ in range(2):  # second launch: workspace / epoch reuse
        y = runtime.launch_conv(cfg, kcfg, *dev)
        torch.cuda.synchronize()
        got = y.float().cpu().numpy()
        ref_b = oracle.conv_chain(x, w1, w2, "relu", bf16_intermediate=True)
        ref = oracle.conv_chain(x, w1, w2, "relu")
        assert np.isfinite(got).all()
        err_b, err = oracle.max_relative_error(got, ref_b), oracle.max_relative_error(got, ref)
        assert err_b <= TOL and err <= TOL, (name, exchange, kcfg.as_dict(), err_b, err)


@pytest.mark.gpu
@pytest.mark.parametrize("case", BLOCK_CASES, ids=lambda c: c[0])
def test_conv_block_matches_oracle(case):
    """1x1 -> ReLU -> k2 x k2: GEMM1 reads im2col boxes of the L2-resident
    intermediate after the halo tiles are published (parity unpinned: no
    reference counterpart; the oracle is pinned to torch's direct conv above)."""
    import torch

    from paper_2512_12949_b200 import runtime, workload as W

    name, shape, batch = case
    cfg = W.ConvBlockConfig(*shape)
    ic, h, w, oc1, oc2, k1, k2 = shape
    x, w1, w2 = _conv_inputs(ic, h, w, oc1, oc2, k1, batch, seed=3, k2=k2)
    dev = [torch.from_numpy(a).cuda().to(torch.bfloat16).contiguous() for a in (x, w1, w2)]
    kcfg = runtime.lower_conv(cfg, batch, "l2")
    for _ in range(2):
        y = runtime.launch_conv(cfg, kcfg, *dev)
        torch.cuda.synchronize()
        got = y.float().cpu().numpy()
        ref_b = oracle.conv_chain(x, w1, w2, "relu", bf16_intermediate=True)
        ref = oracle.conv_chain(x, w1, w2, "relu")
        err_b, err = oracle.max_relative_error(got, ref_b), oracle.max_relative_error(got, ref)
        assert np.isfinite(got).all()
        assert err_b <= TOL and err <= TOL, (name, kcfg.as_dict(), err_b, err)


@pytest.mark.gpu
@pytest.mark.parametrize("case", [("C5", (64, 56, 56, 64, 256, 3, 1), 1), ("block-3x3", (256, 14, 14, 64, 64, 1, 3), 2)],
                         ids=lambda c: c[0])
def test_conv_chain_fp16(case):
    """fp16 storage through the implicit-GEMM conv paths (im2col TMA maps of FLOAT16)."""
    import torch

    from paper_2512_12949_b200 import runtime, workload as W

    name, shape, batch = case
    ic, h, w, oc1, oc2, k1, k2 = shape
    cfg = W.ConvChainConfig(*shape) if k2 == 1 else W.ConvBlockConfig(*shape)
    x, w1, w2 = (oracle.round_f16(a) for a in _conv_inputs(ic, h, w, oc1, oc2, k1, batch, seed=13, k2=k2))
    dev = [torch.from_numpy(a).cuda().to(torch.float16).contiguous() for a in (x, w1, w2)]
    y = runtime.run_conv(cfg, *dev, exchange="l2")
    torch.cuda.synchronize()
    assert y.dtype == torch.float16
    got = y.float().cpu().numpy()
    ref = oracle.conv_chain(x, w1, w2, "relu")
    assert np.isfinite(got).all() and oracle.max_relative_error(got, ref) <= TOL
