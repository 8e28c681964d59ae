"""numpy restatement of the reference chain semantics (TEST INFRASTRUCTURE).

Parity: pinned against reference outputs in tests/golden/ (numerics.npz,
analyzer_samples.json); GELU (tanh form) is an extension the reference lacks
(workload.py:29-32) -- parity unpinned for that activation alone.
"""

from __future__ import annotations

import itertools

import numpy as np

DIMS = ("m", "n", "k", "l")


def relu(x):
    return np.maximum(x, 0)


def silu(x):
    # simulator.py:107-108
    return x / (1.0 + np.exp(-x))


def gelu_tanh(x):
    # GPT-2 "gelu_new": 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3)))
    return 0.5 * x * (1.0 + np.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


_ACT = {"identity": lambda x: x, "relu": relu, "silu": silu, "gelu": gelu_tanh}


def make_inputs(kind: str, m: int, n: int, k: int, l: int, seed: int = 0, dtype=np.float32) -> dict:
    """simulator.py:112-123: U[-1,1] from default_rng(seed), drawn in sorted name order."""
    rng = np.random.default_rng(seed)
    shapes = {"A": (m, k), "D": (n, l)}
    for w in (("B0", "B1") if kind == "gated_ffn" else ("B",)):
        shapes[w] = (k, n)
    return {name: rng.uniform(-1.0, 1.0, shapes[name]).astype(dtype) for name in sorted(shapes)}


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float32 (what the GPU sees)."""
    bits = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    bits = (bits + 0x7FFF + ((bits >> 16) & 1)) & 0xFFFF0000
    return bits.astype(np.uint32).view(np.float32)


def round_f16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to IEEE half, returned as float32."""
    return np.asarray(x, dtype=np.float32).astype(np.float16).astype(np.float32)


def dense_chain(kind: str, activation: str, inputs: dict, bf16_intermediate: bool = False,
                f16_intermediate: bool = False) -> np.ndarray:
    """simulator.py:126-134: E = act(A@B)@D or (silu(A@B0) * (A@B1))@D, dense, no tiling.
    ``bf16_intermediate`` / ``f16_intermediate`` round C to the GPU's 2-byte storage type
    before the second GEMM (the GPU dataflow)."""
    a = inputs["A"]
    if kind == "gated_ffn":
        c = silu(a @ inputs["B0"]) * (a @ inputs["B1"])
    else:
        c = _ACT[activation](a @ inputs["B"])
    if bf16_intermediate:
        c = round_bf16(c)
    if f16_intermediate:
        c = round_f16(c)
    return c @ inputs["D"]


def max_relative_error(result, reference) -> float:
    """simulator.py:143-147."""
    result = np.asarray(result, dtype=np.float64)
    reference = np.asarray(reference, dtype=np.float64)
    scale = float(np.max(np.abs(reference)))
    diff = float(np.max(np.abs(result - reference)))
    return diff if scale == 0.0 else diff / scale


def replay_plan(kind: str, activation: str, dims: tuple, plan: dict, inputs: dict) -> np.ndarray:
    """Numeric part of simulator.execute_plan (simulator.py:204-422): replay the
    plan's loop nest at cluster-cover granularity.

    ``plan`` is the reference JSON plan dict (plan.py:337-355).  GEMM0 batches
    accumulate split-K slices per block tile (:302-340, both gated lowerings),
    the combine applies when the reduction completes (completion mode) or per
    increment (:342-345, :395-405), GEMM1 fires accumulate E partials
    (:347-362) and completed tiles are added into E (:363-371; "+=" is the
    inter-cluster reduction).  Traffic counting is the analyzer's job and is
    not restated here.
    """
    m, n, k, l = dims
    spatial = set(plan["schedule"]["spatial"])
    order = list(plan["schedule"]["temporal"])
    blk = plan["tiles"]["block"]
    cls = plan["tiles"]["cluster"]
    low = plan.get("gated_lowering", "n/a")
    gated = kind == "gated_ffn"
    eff = {"m": m, "n": n, "k": 2 * k if low == "doubled_k" else k, "l": l}
    split = dict(cls)
    if low == "spatial_split":
        split["k"] = cls["k"] // 2
    cover = {d: split[d] * blk[d] for d in DIMS}
    steps = {d: eff[d] // cover[d] for d in DIMS}
    trips = {d: (1 if d in spatial else steps[d]) for d in DIMS}
    grid = {d: (steps[d] if d in spatial else 1) for d in DIMS}
    level = {d: i + 1 for i, d in enumerate(order)}
    completion = "k" not in level or level["k"] == max(level[d] for d in "mnk" if d in level)
    act = _ACT[activation]
    a_mat, d_mat = inputs["A"], inputs["D"]
    e_out = np.zeros((m, l), dtype=a_mat.dtype)
    pos = {d: i for i, d in enumerate(order)}

    def tr(leaf, d):
        return leaf[pos[d]] if d in pos else 0

    def gemm0(base, leaf):
        m0 = base["m"] + tr(leaf, "m") * cover["m"]
        n0 = base["n"] + tr(leaf, "n") * cover["n"]
        k0 = base["k"] + tr(leaf, "k") * cover["k"]
        rows, cols = slice(m0, m0 + cover["m"]), slice(n0, n0 + cover["n"])
        acc0 = np.zeros((cover["m"], cover["n"]), dtype=a_mat.dtype)
        acc1 = np.zeros_like(acc0) if gated else None
        for j in range(split["k"]):
            ks = k0 + j * blk["k"]
            if gated and low == "spatial_split":
                a_sl = a_mat[rows, ks:ks + blk["k"]]
                acc0 += a_sl @ inputs["B0"][ks:ks + blk["k"], cols]
                acc1 += a_sl @ inputs["B1"][ks:ks + blk["k"], cols]
            elif gated:
                lo, hi = ks, ks + blk["k"]          # virtual range in the stacked 2K reduction
                if lo < k:                           # branch 0 part
                    t = min(hi, k)
                    acc0 += a_mat[rows, lo:t] @ inputs["B0"][lo:t, cols]
                if hi > k:                           # branch 1 part
                    s = max(lo, k)
                    acc1 += a_mat[rows, s - k:hi - k] @ inputs["B1"][s - k:hi - k, cols]
            else:
                acc0 += a_mat[rows, ks:ks + blk["k"]] @ inputs["B"][ks:ks + blk["k"], cols]
        return acc0, acc1

    def combine(acc0, acc1):
        return silu(acc0) * acc1 if gated else act(acc0)

    need = trips["n"] * (1 if completion else trips["k"])
    inc_depth = max((level[d] for d in "mnk" if d in level), default=0)
    g1_depth = max((level[d] for d in "mnl" if d in level), default=0)
    inc_pos = [i for i, d in enumerate(order) if level[d] <= inc_depth]
    g1_pos = [i for i, d in enumerate(order) if level[d] <= g1_depth]
    grid_dims = [d for d in DIMS if d in spatial]
    for cell in itertools.product(*(range(grid[d]) for d in grid_dims)):
        base = {d: 0 for d in DIMS}
        for d, g in zip(grid_dims, cell):
            base[d] = g * cover[d]
        partial, ready, e_acc, count = {}, {}, {}, {}
        done0, done1 = set(), set()
        last_inc = last_g1 = None

        def fire(region, leaf):
            tm, tl = tr(leaf, "m"), tr(leaf, "l")
            n0 = base["n"] + tr(leaf, "n") * cover["n"]
            l0 = base["l"] + tl * cover["l"]
            contrib = region @ d_mat[n0:n0 + cover["n"], l0:l0 + cover["l"]]
            e_acc[(tm, tl)] = e_acc[(tm, tl)] + contrib if (tm, tl) in e_acc else contrib
            count[(tm, tl)] = count.get((tm, tl), 0) + 1
            if count[(tm, tl)] == need:
                m0 = base["m"] + tm * cover["m"]
                e_out[m0:m0 + cover["m"], l0:l0 + cover["l"]] += e_acc.pop((tm, tl))

        for leaf in itertools.product(*(range(trips[d]) for d in order)):
            tm, tn, tk, tl = (tr(leaf, d) for d in DIMS)
            if completion:
                if (tm, tn, tk) not in done0:
                    done0.add((tm, tn, tk))
                    acc = gemm0(base, leaf)
                    if (tm, tn) in partial:
                        p0, p1 = partial[(tm, tn)]
                        acc = (p0 + acc[0], p1 + acc[1] if gated else None)
                    partial[(tm, tn)] = acc
                    if tk == trips["k"] - 1:
                        ready[(tm, tn)] = combine(*partial.pop((tm, tn)))
                if (tm, tn) in ready and (tm, tn, tl) not in done1:
                    done1.add((tm, tn, tl))
                    fire(ready[(tm, tn)], leaf)
            else:
                key = tuple(leaf[i] for i in inc_pos)
                if key != last_inc:
                    last_inc = key
                    ready["inc"] = combine(*gemm0(base, leaf))
                key = tuple(leaf[i] for i in g1_pos)
                if key != last_g1:
                    last_g1 = key
                    fire(ready["inc"], leaf)
    return e_out


def im2col_nhwc(x: np.ndarray, k1: int) -> np.ndarray:
    """The reference's conv lowering made explicit (conv_chain_to_gemm,
    workload.py:191-199: m = h*w, k = ic*k1^2): x [batch, h, w, ic] NHWC ->
    A [batch*h*w, k1*k1*ic] with K ordered (tap r, tap s, channel), stride 1,
    same padding (zeros outside the image)."""
    b, h, w, c = x.shape
    pad = k1 // 2
    xp = np.zeros((b, h + 2 * pad, w + 2 * pad, c), dtype=x.dtype)
    xp[:, pad:pad + h, pad:pad + w, :] = x
    cols = [xp[:, r:r + h, s:s + w, :] for r in range(k1) for s in range(k1)]
    return np.concatenate(cols, axis=-1).reshape(b * h * w, k1 * k1 * c)


def conv_chain(x: np.ndarray, w1: np.ndarray, w2: np.ndarray, activation: str = "relu",
               bf16_intermediate: bool = False) -> np.ndarray:
    """conv(k1 x k1, same) -> act -> conv(1x1) as the GEMM chain the reference
    executes on a conv preset (dense_chain over the im2col matrix).
    x [b, h, w, ic], w1 [k1, k1, ic, oc1] (HWIO), w2 [oc1, oc2] -> y [b, h, w, oc2].
    Extension (no reference counterpart): w2 [k2, k2, oc1, oc2] applies a k2 x k2
    second convolution to the intermediate (im2col of C, same padding)."""
    b, h, w, _ = x.shape
    k1 = w1.shape[0]
    if w2.ndim == 4:
        c = _ACT[activation](im2col_nhwc(x, k1) @ w1.reshape(-1, w1.shape[-1]))
        if bf16_intermediate:
            c = round_bf16(c)
        c = c.reshape(b, h, w, w1.shape[-1])
        y = im2col_nhwc(c, w2.shape[0]) @ w2.reshape(-1, w2.shape[-1])
        return y.reshape(b, h, w, w2.shape[-1])
    inputs = {"A": im2col_nhwc(x, k1), "B": w1.reshape(-1, w1.shape[-1]), "D": w2}
    y = dense_chain("standard_ffn", activation, inputs, bf16_intermediate=bf16_intermediate)
    return y.reshape(b, h, w, w2.shape[1])
