"""GPU runner: ``run(graph, plan, tensors)`` -> E through the C ABI.

Lowering (ff_plan_lower, C++) turns the logical plan into a physical sm_100a
launch; see DESIGN.md.  Tensors are caller-owned bf16 CUDA tensors in the
reference layouts A[m,k], B[k,n] / B0,B1[k,n], D[n,l]; the output E[m,l] is
allocated here unless ``out`` is given.  Work is stream-ordered with no host
synchronisation.  There is no CPU fallback: a missing library or device raises.
"""

from __future__ import annotations

import ctypes
from typing import Optional

from . import _native as nat
from .plan import FusionPlan
from .workload import DIMS, GATED_FFN, ChainGraph, ConvBlockConfig, ConvChainConfig

_workspaces: dict = {}
_desc_cache: dict = {}
_cuda_ok = False


def chain_desc(graph: ChainGraph, dtype: str = "bf16") -> nat.ChainDesc:
    d = graph.dims
    return nat.ChainDesc(nat.KIND[graph.kind], nat.ACT[graph.activation], d.m, d.n, d.k, d.l, d.element_size,
                         nat.DTYPE[dtype])


def _storage(tensors) -> str:
    """'bf16' or 'f16': every chain tensor must share one 2-byte storage type."""
    import torch

    kinds = {t.dtype for t in tensors}
    if kinds == {torch.bfloat16}:
        return "bf16"
    if kinds == {torch.float16}:
        return "f16"
    raise ValueError(f"chain tensors must all be bfloat16 or all float16, got {sorted(map(str, kinds))}")


def plan_desc(plan: FusionPlan) -> nat.PlanDesc:
    pd = nat.PlanDesc()
    pd.spatial_mask = sum(1 << i for i, d in enumerate(DIMS) if d in plan.schedule.spatial)
    order = plan.schedule.temporal_order
    for i, d in enumerate(order):
        pd.temporal[i] = DIMS.index(d)
    pd.n_temporal = len(order)
    for i, d in enumerate(DIMS):
        pd.block[i] = plan.tiles.block[d]
        pd.cluster[i] = plan.tiles.cluster[d]
    pd.gated_lowering = nat.LOWERING[plan.gated_lowering]
    return pd


def _num_sms() -> int:
    import torch

    return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count


EXCHANGES = {"dsm": nat.XCHG_DSM, "l2": nat.XCHG_L2, "pair": nat.XCHG_L2_PAIR, "l2dsm": nat.XCHG_L2_DSMR}


def exchange_name(cfg: nat.KernelConfig) -> str:
    return {v: k for k, v in EXCHANGES.items()}[int(cfg.exchange)]


def explicit_config(graph: ChainGraph, ring: int, n_splits: int, nb: int, lb: int, exchange: str,
                    num_sms: Optional[int] = None) -> nat.KernelConfig:
    """An explicit physical launch, validated and completed (ff_config_finish);
    raises UnsupportedPlan when no kernel runs it."""
    lib = nat.load()
    cfg = nat.KernelConfig()
    cfg.ring, cfg.n_splits, cfg.nb, cfg.lb, cfg.exchange = ring, n_splits, nb, lb, EXCHANGES[exchange]
    nat.check(lib.ff_config_finish(ctypes.byref(chain_desc(graph)), num_sms if num_sms is not None else 148,
                                   ctypes.byref(cfg)))
    return cfg


def reproducible_configs(graph: ChainGraph, num_sms: Optional[int] = None) -> list:
    """Explicit DSM reduce-scatter launches (FF_XCHG_L2_DSMR: the S splits of an E tile are
    one cluster and sum in split order) over the E slice widths and chunk widths the 1-CTA
    kernels run -- bit-reproducible alternatives to the reduce-add split lowerings (GPT-2s:
    ring 6 x 4 splits ties the fastest reduce-add launch, profiles/r02/s5/sweep_final.log)."""
    out = []
    for lb in (256, 128):
        if graph.dims.l % lb:
            continue
        for s in (2, 4, 8):
            for nb in (128, 64):
                try:
                    out.append(explicit_config(graph, graph.dims.l // lb, s, nb, lb, "l2dsm", num_sms))
                except nat.FusePlanError:
                    continue
    return out


def is_deterministic(graph: ChainGraph, cfg: nat.KernelConfig, num_sms: Optional[int] = None) -> bool:
    """True when launching ``cfg`` writes a bit-identical E on every run with the same
    inputs (ff_config_deterministic): no N splits, the DSM reduce-scatter of the splits,
    or the CTA-pair kernel's exchange-region finish.  Otherwise the N-split partials
    meet through TMA reduce-adds whose order follows the CTAs' timing."""
    lib = nat.load()
    out = ctypes.c_int32(0)
    nat.check(lib.ff_config_deterministic(ctypes.byref(chain_desc(graph)), ctypes.byref(cfg),
                                          num_sms if num_sms is not None else 148, ctypes.byref(out)))
    return bool(out.value)


def lower(graph: ChainGraph, plan: Optional[FusionPlan] = None, num_sms: Optional[int] = None,
          exchange: str = "auto", deterministic: bool = False) -> nat.KernelConfig:
    """Physical launch configuration for (graph, plan).  plan=None lets the
    runtime choose the hardware-shaped configuration; ``exchange`` picks the
    shuffle transport: "dsm" (thread-block cluster, distributed shared memory),
    "l2" (TMA through an L2-resident scratch), "pair" (L2 transport, CTA-pair
    cta_group::2 kernel), "l2dsm" (L2 ring; the N splits of every E tile form a
    thread-block cluster and reduce their partials over DSM) or "auto" (first of
    pair, l2, dsm that supports it).

    deterministic=True: only launches whose E is bit-identical run to run
    (is_deterministic).  "auto" then returns the first of pair, l2dsm, l2, dsm
    that qualifies; an explicit transport whose lowering sums split partials by
    reduce-adds raises UnsupportedPlan."""
    if deterministic:
        if exchange == "auto":
            for candidate in ("pair", "l2dsm", "l2", "dsm"):
                try:
                    cfg = lower(graph, plan, num_sms, candidate)
                except nat.UnsupportedPlan:
                    continue
                if is_deterministic(graph, cfg, num_sms):
                    return cfg
            rc = reproducible_configs(graph, num_sms) if plan is None else []
            if rc:
                return rc[0]
            raise nat.UnsupportedPlan("no bit-reproducible lowering (every transport sums N-split partials by "
                                      "reduce-adds); pass an explicit one-split config to launch()")
        cfg = lower(graph, plan, num_sms, exchange)
        if not is_deterministic(graph, cfg, num_sms):
            raise nat.UnsupportedPlan(f"the {exchange} lowering ({cfg.as_dict()}) sums its N-split partials by "
                                      "reduce-adds: not bit-reproducible (deterministic=True)")
        return cfg
    if exchange == "auto":
        last = None
        for candidate in ("pair", "l2", "dsm"):
            try:
                return lower(graph, plan, num_sms, candidate)
            except nat.UnsupportedPlan as exc:
                last = exc
        raise last
    lib = nat.load()
    cfg = nat.KernelConfig()
    ch = chain_desc(graph)
    sms = num_sms if num_sms is not None else 148
    x = EXCHANGES[exchange]
    if plan is None:
        nat.check(lib.ff_auto_config_ex(ctypes.byref(ch), sms, x, ctypes.byref(cfg)))
    else:
        pd = plan_desc(plan)
        nat.check(lib.ff_plan_lower_ex(ctypes.byref(ch), ctypes.byref(pd), sms, x, ctypes.byref(cfg)))
    return cfg


def _workspace(nbytes: int, device, stream):
    """Per-(device, stream) workspace, zero-filled once when allocated.

    The kernels leave it zero again (epoch-stamped flags, split counters and
    the fp32 E region reset by the last contributor), but two launches in
    flight at the same time must not share one, hence one per stream."""
    import torch

    if nbytes == 0:
        return None
    key = (device.index if device.index is not None else torch.cuda.current_device(), int(stream.cuda_stream))
    buf = _workspaces.get(key)
    if buf is None or buf.numel() < nbytes:
        with torch.cuda.stream(stream):
            buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)
        _workspaces[key] = buf
    return buf


def _check_out(out, shape, like):
    """A caller-supplied output must be a contiguous CUDA tensor of the inputs'
    dtype, exact shape and device: the kernel writes it through a TMA map built
    from the shape with a dense row stride (and plain stores in the split finish)."""
    if (not out.is_cuda or out.device != like.device or out.dtype != like.dtype or tuple(out.shape) != tuple(shape)
            or not out.is_contiguous()):
        raise ValueError(f"out must be a contiguous {like.dtype} CUDA tensor of shape {tuple(shape)} on {like.device}")
    if out.data_ptr() % 16:
        raise ValueError("out must be 16-byte aligned")


def _stream_of(stream, device):
    """torch stream for `stream` (None = current stream, or a raw cudaStream_t handle)."""
    import torch

    s = stream if stream is not None else torch.cuda.current_stream(device)
    if not hasattr(s, "cuda_stream"):
        s = torch.cuda.ExternalStream(int(s), device=device)
    return s


def _require_cuda():
    import torch

    if not _cuda_ok:
        if not torch.cuda.is_available():
            raise nat.NativeUnavailable("no CUDA device: the fused chain only executes on sm_100a")
        globals()["_cuda_ok"] = True


def launch(graph: ChainGraph, cfg: nat.KernelConfig, tensors: dict, out=None, stream=None, c_debug=None):
    """Launch one fused chain with an explicit physical configuration."""
    import torch

    lib = nat.load()
    _require_cuda()
    gated = graph.kind == GATED_FFN
    names = ("A", "B0", "B1", "D") if gated else ("A", "B", "D")
    d = graph.dims
    shapes = {"A": (d.m, d.k), "B": (d.k, d.n), "B0": (d.k, d.n), "B1": (d.k, d.n), "D": (d.n, d.l)}
    storage = _storage([tensors[n] for n in names])
    a = tensors["A"]
    for name in names:
        t = tensors[name]
        if (not t.is_cuda or t.device != a.device or tuple(t.shape) != shapes[name] or not t.is_contiguous()):
            raise ValueError(f"{name} must be a contiguous {storage} CUDA tensor of shape {shapes[name]} on "
                             f"{a.device}")
        if t.data_ptr() % 16:
            raise ValueError(f"{name} must be 16-byte aligned")
    if out is None:
        out = torch.empty((d.m, d.l), dtype=a.dtype, device=a.device)
    else:
        _check_out(out, (d.m, d.l), a)
    if c_debug is not None:
        _check_out(c_debug, (d.m, d.n), a)
    # descriptor + workspace size per (chain, storage, launch config): a serving loop
    # calls this with the same shapes every step (host cost ~15 -> ~8 us per launch)
    key = (graph.kind, graph.activation, d.m, d.n, d.k, d.l, storage, bytes(cfg))
    cached = _desc_cache.get(key)
    if cached is None:
        ch = chain_desc(graph, storage)
        cached = (ch, lib.ff_chain_workspace_bytes(ctypes.byref(ch), ctypes.byref(cfg)))
        if len(_desc_cache) > 256:
            _desc_cache.clear()
        _desc_cache[key] = cached
    ch, ws_bytes = cached
    s = _stream_of(stream, a.device)
    handle = s.cuda_stream
    ws = _workspace(ws_bytes, a.device, s)
    tp = nat.Tensors(a.data_ptr(), tensors["B0" if gated else "B"].data_ptr(),
                     tensors["B1"].data_ptr() if gated else None, tensors["D"].data_ptr(), out.data_ptr())
    ws_ptr = ws.data_ptr() if ws is not None else None
    ws_bytes = ws.numel() if ws is not None else 0  # the buffer's size: the library checks it covers the layout
    if c_debug is not None:
        rc = lib.ff_chain_launch_debug(ctypes.byref(ch), ctypes.byref(cfg), ctypes.byref(tp), ws_ptr, ws_bytes,
                                       c_debug.data_ptr(), handle)
    else:
        rc = lib.ff_chain_launch(ctypes.byref(ch), ctypes.byref(cfg), ctypes.byref(tp), ws_ptr, ws_bytes, handle)
    nat.check(rc)
    return out


def run(graph: ChainGraph, plan: Optional[FusionPlan], tensors: dict, out=None, stream=None,
        exchange: str = "auto", deterministic: bool = False):
    """Execute the chain under ``plan`` on the current GPU; returns E (bf16).
    deterministic=True restricts the lowering to bit-reproducible launches (see lower)."""
    return launch(graph, lower(graph, plan, _num_sms(), exchange, deterministic), tensors, out=out, stream=stream)


def kernel_launches(graph: ChainGraph, cfg: nat.KernelConfig) -> int:
    """How many CUDA kernels one launch issues."""
    lib = nat.load()
    ch = chain_desc(graph)
    return int(lib.ff_chain_kernel_count(ctypes.byref(ch), ctypes.byref(cfg)))


def profile_best_from_list(graph: ChainGraph, plans, tensors: dict, iters: int = 10, warmup: int = 3,
                           exchanges=("l2", "dsm")):
    """Alg. 2 line 10 (ProfileBestFromList): time each candidate
    plan's fused kernel (under each shuffle transport) on the device and return
    [(ms, plan, cfg)] fastest first.  Plans with no sm_100a lowering are skipped."""
    import torch

    timed = []
    seen = set()
    for plan, exchange in ((p, x) for p in plans for x in exchanges):
        try:
            cfg = lower(graph, plan, _num_sms(), exchange)
        except nat.UnsupportedPlan:
            continue
        key = tuple(cfg.as_dict().items())
        if key in seen:
            continue
        seen.add(key)
        out = torch.empty((graph.dims.m, graph.dims.l), dtype=tensors["A"].dtype, device=tensors["A"].device)
        for _ in range(warmup):
            launch(graph, cfg, tensors, out=out)
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        for _ in range(iters):
            launch(graph, cfg, tensors, out=out)
        stop.record()
        stop.synchronize()
        timed.append((start.elapsed_time(stop) / iters, plan, cfg))
    timed.sort(key=lambda x: x[0])
    return timed


def profile_configs(graph: ChainGraph, cfgs, tensors: dict, iters: int = 10, warmup: int = 3):
    """Time explicit physical configurations; returns [(ms, cfg)] in input order."""
    import torch

    out = []
    res = torch.empty((graph.dims.m, graph.dims.l), dtype=tensors["A"].dtype, device=tensors["A"].device)
    for cfg in cfgs:
        for _ in range(warmup):
            launch(graph, cfg, tensors, out=res)
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        for _ in range(iters):
            launch(graph, cfg, tensors, out=res)
        stop.record()
        stop.synchronize()
        out.append((start.elapsed_time(stop) / iters, cfg))
    return out


# ----------------------------------------------------------------------------- conv chains


def conv_desc(cfg, batch: int = 1, activation: str = "relu", dtype: str = "bf16") -> nat.ConvDesc:
    """ffConvDesc of a ConvChainConfig (reference) or ConvBlockConfig (k2 > 1 extension)."""
    return nat.ConvDesc(batch, cfg.h, cfg.w, cfg.ic, cfg.oc1, cfg.oc2, cfg.k1, cfg.k2, nat.ACT[activation],
                        nat.DTYPE[dtype])


def lower_conv(cfg, batch: int = 1, exchange: str = "auto", activation: str = "relu",
               num_sms: Optional[int] = None) -> nat.KernelConfig:
    """Physical launch for a conv chain (ConvChainConfig, workload.py:168-184).
    k1 > 1 runs as an implicit GEMM on the 1-CTA kernels ("dsm" / "l2")."""
    lib = nat.load()
    cd = conv_desc(cfg, batch, activation)
    order = {"auto": ("pair", "l2", "dsm")}.get(exchange, (exchange,))
    last = None
    for x in order:
        out = nat.KernelConfig()
        try:
            nat.check(lib.ff_conv_chain_lower(ctypes.byref(cd), num_sms or 148, EXCHANGES[x], ctypes.byref(out)))
            return out
        except nat.UnsupportedPlan as exc:
            last = exc
    raise last


def launch_conv(cfg, kcfg: nat.KernelConfig, x, w1, w2, out=None, stream=None, activation: str = "relu"):
    """conv(k1 x k1, same padding) -> act -> conv(k2 x k2) on NHWC bf16 tensors:
    x [batch, h, w, ic], w1 [k1, k1, ic, oc1] (HWIO), w2 [oc1, oc2] (k2 == 1) or
    [k2, k2, oc1, oc2]; returns y [batch, h, w, oc2].  k1 > 1: GEMM0 reads x
    through an im2col tensor map; k2 > 1 (ConvBlockConfig): GEMM1 reads the
    L2-resident intermediate through one."""
    import torch

    lib = nat.load()
    _require_cuda()
    batch = x.shape[0]
    w2_shape = (cfg.oc1, cfg.oc2) if cfg.k2 == 1 else (cfg.k2, cfg.k2, cfg.oc1, cfg.oc2)
    shapes = {"x": (batch, cfg.h, cfg.w, cfg.ic), "w1": (cfg.k1, cfg.k1, cfg.ic, cfg.oc1), "w2": w2_shape}
    storage = _storage([x, w1, w2])
    for name, t in (("x", x), ("w1", w1), ("w2", w2)):
        if not t.is_cuda or t.device != x.device or tuple(t.shape) != shapes[name] or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous {storage} CUDA tensor of shape {shapes[name]} on "
                             f"{x.device}")
        if t.data_ptr() % 16:
            raise ValueError(f"{name} must be 16-byte aligned")
    if out is None:
        out = torch.empty((batch, cfg.h, cfg.w, cfg.oc2), dtype=x.dtype, device=x.device)
    else:
        _check_out(out, (batch, cfg.h, cfg.w, cfg.oc2), x)
    cd = conv_desc(cfg, batch, activation, storage)
    ws_bytes = lib.ff_conv_chain_workspace_bytes(ctypes.byref(cd), ctypes.byref(kcfg))
    s = _stream_of(stream, x.device)
    ws = _workspace(ws_bytes, x.device, s)
    tp = nat.Tensors(x.data_ptr(), w1.data_ptr(), None, w2.data_ptr(), out.data_ptr())
    nat.check(lib.ff_conv_chain_launch(ctypes.byref(cd), ctypes.byref(kcfg), ctypes.byref(tp),
                                       ws.data_ptr() if ws is not None else None, ws_bytes, s.cuda_stream))
    return out


def run_conv(cfg, x, w1, w2, out=None, stream=None, exchange: str = "auto",
             activation: str = "relu"):
    """Execute a conv chain on the current GPU (the reference's conv presets
    C1-C8, workload.py:207-240, without materialising the im2col matrix)."""
    kcfg = lower_conv(cfg, x.shape[0], exchange, activation, _num_sms())
    return launch_conv(cfg, kcfg, x, w1, w2, out=out, stream=stream, activation=activation)
