"""FlashFuser's DSM communication primitives (paper SIII-B; the reference models
their bytes in analyzer.py:331-354) executed over sm_100a distributed shared
memory (csrc/dsm_primitives.cuh) and checked against numpy: reduce-scatter and
all-exchange (Add) sum in cluster-rank order, so fp32 results are exact."""

import ctypes

import numpy as np
import pytest

from paper_2512_12949_b200 import _native as nat

OPS = {"reduce_scatter": 0, "all_gather": 1, "all_exchange_add": 2, "all_exchange_mul": 3, "shuffle": 4}


def _lib():
    lib = nat.load()
    lib.ff_dsm_primitive_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
    lib.ff_dsm_last_error.restype = ctypes.c_char_p
    return lib


def test_primitive_entry_point_rejects_bad_shapes():
    lib = _lib()
    ms = ctypes.c_float()
    assert lib.ff_dsm_primitive_run(0, 3, 100, 1, None, None, 1, ctypes.byref(ms)) == 3   # 100 % 12
    assert lib.ff_dsm_primitive_run(3, 3, 120, 1, None, None, 1, ctypes.byref(ms)) == 3   # mul needs pairs
    assert lib.ff_dsm_primitive_run(9, 2, 64, 1, None, None, 1, ctypes.byref(ms)) == 5


def expected(op, x):
    """x: [clusters, G, N] -> expected per-CTA output [clusters, G, N]."""
    c, g, n = x.shape
    out = x.copy()
    acc = x[:, 0].copy()
    for r in range(1, g):
        acc = acc + x[:, r]  # rank order, fp32
    if op == "all_exchange_add":
        out[:] = acc[:, None]
    elif op == "reduce_scatter":
        s = n // g
        for r in range(g):
            out[:, r, r * s:(r + 1) * s] = acc[:, r * s:(r + 1) * s]
    elif op == "all_gather":
        s = n // g
        for r in range(g):
            out[:, :, r * s:(r + 1) * s] = x[:, r:r + 1, r * s:(r + 1) * s]
    elif op == "all_exchange_mul":
        gate, up = x[:, 0::2], x[:, 1::2]
        prod = (gate / (1.0 + np.exp(-gate))) * up
        out[:, 0::2] = prod
        out[:, 1::2] = prod
    elif op == "shuffle":
        out = np.roll(x, 1, axis=1)
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 4, 8, 16])
@pytest.mark.parametrize("op", list(OPS))
def test_dsm_primitive_matches_numpy(op, G):
    import torch

    if op == "all_exchange_mul" and G != 2:
        pytest.skip("the SwiGLU all-exchange pairs CTAs")
    N, clusters = 64 * G * 4, 3
    rng = np.random.default_rng(G)
    x = rng.uniform(-1, 1, (clusters, G, N)).astype(np.float32)
    dx = torch.from_numpy(x).cuda().contiguous()
    dy = torch.empty_like(dx)
    ms = ctypes.c_float()
    rc = _lib().ff_dsm_primitive_run(OPS[op], G, N, clusters, dx.data_ptr(), dy.data_ptr(), 1, ctypes.byref(ms))
    assert rc == 0, _lib().ff_dsm_last_error()
    got = dy.cpu().numpy()
    want = expected(op, x)
    if op == "reduce_scatter":  # only each CTA's own slice is defined after a reduce-scatter
        s = N // G
        for r in range(G):
            np.testing.assert_array_equal(got[:, r, r * s:(r + 1) * s], want[:, r, r * s:(r + 1) * s])
    elif op == "all_exchange_mul":
        np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-6)
    else:
        np.testing.assert_array_equal(got, want)
