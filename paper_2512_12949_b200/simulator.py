"""Plan execution API (fuseplan/simulator.py) backed by the sm_100a kernels.

The reference executes a plan with a numpy tile replay that also counts the
bytes crossing each memory tier (simulator.py:177-424).  Here the numerics run
on the GPU through the C ABI (:mod:`runtime`), and the byte trace comes from
:func:`replay_traffic`, a loop-nest replay of the same plan that counts tile
events without touching matrices -- an independent re-derivation of the
analyzer's closed forms (their equality is tested on sampled plans).

There is no CPU execution path: :func:`execute_plan` raises if the CUDA
extension or device is unavailable.
"""

from __future__ import annotations

import itertools
import random
from dataclasses import dataclass, field
from math import prod
from typing import Optional

import numpy as np

from .analyzer import DEFAULT_ACC_SIZE, analyze, live_tile_counts, slot_tier_bytes
from .errors import PlanError
from .hardware import DeviceModel, b200_profile
from .plan import LOWERING_DOUBLED_K, LOWERING_SPATIAL_SPLIT, FusionPlan, TileSizes, plan_geometry, \
    structural_violations, enumerate_schedules
from .workload import DIMS, GATED_FFN, ChainGraph

DEFAULT_WORKSPACE_BYTES = 1 << 30


@dataclass(frozen=True)
class SimConfig:
    """simulator.py:45-62.  dtype is the host precision of generated inputs and
    returned outputs; the GPU computes in bf16 with fp32 accumulation, so the
    default tolerance is the north-star bound 1e-2."""

    dtype: str = "f32"
    seed: int = 0
    tolerance: Optional[float] = None
    enforce_rules: bool = True
    acc_size: int = DEFAULT_ACC_SIZE
    max_workspace_bytes: int = DEFAULT_WORKSPACE_BYTES

    @property
    def np_dtype(self):
        return np.float64 if self.dtype == "f64" else np.float32

    @property
    def effective_tolerance(self) -> float:
        return 1e-2 if self.tolerance is None else self.tolerance


@dataclass
class TrafficTrace:
    """Per-tier, per-primitive and per-tensor byte counters (simulator.py:65-99)."""

    tier_bytes: dict = field(default_factory=lambda: dict.fromkeys(("reg", "smem", "dsm", "l2", "global"), 0))
    primitives: dict = field(default_factory=lambda: dict.fromkeys(
        ("all_exchange", "shuffle", "reduce_scatter", "inter_cluster_reduce"), 0))
    per_tensor: dict = field(default_factory=dict)

    def _bump(self, tensor, kind, nbytes):
        slot = self.per_tensor.setdefault(tensor, {})
        slot[kind] = slot.get(kind, 0) + nbytes

    def add_load(self, tensor: str, nbytes: int) -> None:
        self.tier_bytes["global"] += nbytes
        self.tier_bytes["smem"] += nbytes
        self._bump(tensor, "loads", nbytes)

    def add_store(self, tensor: str, nbytes: int) -> None:
        self.tier_bytes["global"] += nbytes
        self._bump(tensor, "stores", nbytes)

    def add_primitive(self, name: str, nbytes: int) -> None:
        if nbytes:
            self.primitives[name] += nbytes
            self.tier_bytes["dsm"] += nbytes

    def charge_region(self, split: dict, copies: int, touches: int = 1) -> None:
        for tier, nbytes in split.items():
            self.tier_bytes["global" if tier == "l2" else tier] += nbytes * copies * touches

    def to_dict(self) -> dict:
        return {"tier_bytes": {k: int(v) for k, v in self.tier_bytes.items()},
                "primitives_bytes": {k: int(v) for k, v in sorted(self.primitives.items())},
                "per_tensor": {k: dict(v) for k, v in sorted(self.per_tensor.items())}}


def fits_execution_budget(graph: ChainGraph, budget: int = DEFAULT_WORKSPACE_BYTES) -> bool:
    """simulator.py:137-140 (kept: the search's refine default depends on it)."""
    return 2 * 8 * sum(graph.tensor_elements(t.name) for t in graph.tensors) <= budget


def max_relative_error(result, reference) -> float:
    """max|E - Eref| / max|Eref| (simulator.py:143-147)."""
    result = np.asarray(result, dtype=np.float64)
    reference = np.asarray(reference, dtype=np.float64)
    scale = float(np.max(np.abs(reference)))
    diff = float(np.max(np.abs(result - reference)))
    return diff if scale == 0.0 else diff / scale


def make_inputs(graph: ChainGraph, config: SimConfig = SimConfig()) -> dict:
    """Seeded U[-1,1] inputs in sorted-name order (simulator.py:112-123)."""
    rng = np.random.default_rng(config.seed)
    d = graph.dims
    shapes = {"A": (d.m, d.k), "D": (d.n, d.l)}
    for name in (("B0", "B1") if graph.kind == GATED_FFN else ("B",)):
        shapes[name] = (d.k, d.n)
    return {name: rng.uniform(-1.0, 1.0, shapes[name]).astype(config.np_dtype) for name in sorted(shapes)}


# ---------------------------------------------------------------------------
# traffic replay (no numerics)
# ---------------------------------------------------------------------------

def _check_plan(plan: FusionPlan, graph: ChainGraph, device: DeviceModel, enforce_rules: bool) -> None:
    problems = structural_violations(plan, graph, device)
    if problems:
        raise PlanError("; ".join(problems))
    if enforce_rules:
        from .search import rule3_activation, rule4_dependency

        if not rule4_dependency(plan.schedule):
            raise PlanError("output-column dimension is grid-spatial")
        if not rule3_activation(plan.schedule, graph, plan.tiles.cluster, plan.tiles.block, plan.gated_lowering):
            raise PlanError("combine would consume incomplete reduction sums")


def replay_traffic(plan: FusionPlan, graph: ChainGraph, device: Optional[DeviceModel] = None,
                   acc_size: int = DEFAULT_ACC_SIZE) -> TrafficTrace:
    """Walk the plan's loop nest cluster by cluster and count every tile event
    exactly as the reference replay does (simulator.py:204-422), without
    the matrix arithmetic."""
    device = device or b200_profile()
    mapping = analyze(graph, device, plan, acc_size).mapping
    geom = plan_geometry(graph, plan)
    order = plan.schedule.temporal_order
    levels = geom.levels
    cl = geom.cluster
    blk = geom.block
    elt = graph.dims.element_size
    nblk = geom.blocks
    gated = graph.kind == GATED_FFN
    low = plan.gated_lowering
    completion = geom.completion_mode
    f_a, f_b, f_d = blk["m"] * blk["k"] * elt, blk["k"] * blk["n"] * elt, blk["n"] * blk["l"] * elt
    f_c, f_e = blk["m"] * blk["n"] * acc_size, blk["m"] * blk["l"] * acc_size
    payload = 2 * f_c if low == LOWERING_DOUBLED_K and cl.cls_k > 1 else f_c
    live = live_tile_counts(graph, plan, geom)
    c_slots = slot_tier_bytes(mapping["C"], live["C"]["m"] * live["C"]["n"], f_c)
    e_slots = slot_tier_bytes(mapping["E"], live["E"]["m"] * live["E"]["l"], f_e)
    pos = {d: i for i, d in enumerate(order)}
    trips = [geom.trips[d] for d in order]
    need = geom.trips["n"] * (1 if completion else geom.trips["k"])

    def prefix_positions(index_dims, phase):
        depth = max((levels[d] for d in index_dims if d in levels), default=0)
        allowed = phase if completion else set(DIMS)
        return [i for i, d in enumerate(order) if levels[d] <= depth and d in allowed]

    a_pos = prefix_positions(("m", "k"), {"m", "n", "k"})
    b_pos = prefix_positions(("k", "n"), {"m", "n", "k"})
    d_pos = prefix_positions(("n", "l"), {"m", "n", "l"})
    depth0 = max((levels[d] for d in "mnk" if d in levels), default=0)
    depth1 = max((levels[d] for d in "mnl" if d in levels), default=0)
    inc_pos = [i for i, d in enumerate(order) if levels[d] <= depth0]
    g1_pos = [i for i, d in enumerate(order) if levels[d] <= depth1]

    trace = TrafficTrace()
    weight_stream = 0
    for _cell in range(geom.num_clusters):
        last = {"a": None, "b": None, "d": None, "inc": None, "g1": None}
        produced, consumed_pairs, ready = set(), set(), set()
        consumed = {}

        def changed(tag, leaf, positions):
            key = tuple(leaf[i] for i in positions)
            if key != last[tag]:
                last[tag] = key
                return True
            return False

        def t(leaf, d):
            return leaf[pos[d]] if d in pos else 0

        def gemm0_loads(leaf):
            nonlocal weight_stream
            if changed("a", leaf, a_pos):
                trace.add_load("A", nblk * f_a)
            if changed("b", leaf, b_pos):
                if gated and low == LOWERING_SPATIAL_SPLIT:
                    trace.add_load("B0", (nblk // 2) * f_b)
                    trace.add_load("B1", (nblk // 2) * f_b)
                elif gated:
                    trace.tier_bytes["global"] += nblk * f_b
                    trace.tier_bytes["smem"] += nblk * f_b
                    weight_stream += nblk * f_b
                else:
                    trace.add_load("B", nblk * f_b)

        def fire(leaf):
            tm, tn, tl = t(leaf, "m"), t(leaf, "n"), t(leaf, "l")
            trace.add_primitive("shuffle", nblk * (cl.cls_shuffle - 1) * f_c)
            if changed("d", leaf, d_pos):
                trace.add_load("D", nblk * cl.cls_shuffle * f_d)
            if completion:
                trace.charge_region(c_slots[(tm % live["C"]["m"]) * live["C"]["n"] + tn % live["C"]["n"]], nblk)
            e_slot = e_slots[(tm % live["E"]["m"]) * live["E"]["l"] + tl % live["E"]["l"]]
            trace.charge_region(e_slot, nblk, touches=2)
            consumed[(tm, tl)] = consumed.get((tm, tl), 0) + 1
            if consumed[(tm, tl)] == need:
                trace.add_primitive("reduce_scatter", cl.cls_m * cl.cls_l * (cl.cls_reduce - 1) * f_e)
                trace.charge_region(e_slot, nblk)
                trace.add_store("E", geom.cover["m"] * geom.cover["l"] * elt)

        for leaf in itertools.product(*(range(n) for n in trips)):
            tm, tn, tk, tl = (t(leaf, d) for d in DIMS)
            if completion:
                if (tm, tn, tk) not in produced:
                    produced.add((tm, tn, tk))
                    gemm0_loads(leaf)
                    if tk == geom.trips["k"] - 1:
                        trace.add_primitive("all_exchange", nblk * (cl.cls_k - 1) * payload)
                        trace.charge_region(c_slots[(tm % live["C"]["m"]) * live["C"]["n"] + tn % live["C"]["n"]],
                                            nblk)
                        ready.add((tm, tn))
                if (tm, tn) in ready and (tm, tn, tl) not in consumed_pairs:
                    consumed_pairs.add((tm, tn, tl))
                    fire(leaf)
            else:
                if changed("inc", leaf, inc_pos):
                    gemm0_loads(leaf)
                    trace.add_primitive("all_exchange", nblk * (cl.cls_k - 1) * payload)
                if changed("g1", leaf, g1_pos):
                    fire(leaf)
    if weight_stream:
        trace.per_tensor["B0"] = {"loads": weight_stream // 2}
        trace.per_tensor["B1"] = {"loads": weight_stream // 2}
    reducers = geom.grid["n"] * geom.grid["k"]
    if reducers > 1 and "E" in trace.per_tensor:
        stores = trace.per_tensor["E"]["stores"]
        trace.primitives["inter_cluster_reduce"] = stores - stores // reducers
    return trace


# ---------------------------------------------------------------------------
# execution on the GPU
# ---------------------------------------------------------------------------

def _to_device(x):
    import torch

    if isinstance(x, torch.Tensor):
        return x if x.is_cuda else x.cuda()
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def execute_plan(plan: FusionPlan, graph: ChainGraph, inputs: dict, config: SimConfig = SimConfig(),
                 device: Optional[DeviceModel] = None):
    """Execute the plan with the fused sm_100a kernel; returns (E, TrafficTrace).

    Drop-in for simulator.execute_plan (simulator.py:177-424): same checks
    (structural, Rules 3/4, workspace budget), same return shape.  numpy inputs
    give a numpy E in ``config.dtype``; torch inputs give a bf16 CUDA tensor.
    """
    from . import runtime

    device = device or b200_profile()
    _check_plan(plan, graph, device, config.enforce_rules)
    if not fits_execution_budget(graph, config.max_workspace_bytes):
        raise PlanError("full tensors exceed the execution workspace budget; use analyzer-only mode")
    import torch

    host = not any(isinstance(v, torch.Tensor) for v in inputs.values())
    dev_inputs = {k: _to_device(v).to(torch.bfloat16).contiguous() for k, v in inputs.items()}
    out = runtime.run(graph, plan, dev_inputs)
    trace = replay_traffic(plan, graph, device, config.acc_size)
    if host:
        out = out.float().cpu().numpy().astype(config.np_dtype)
    return out, trace


def oracle(graph: ChainGraph, inputs: dict):
    """Dense chain reference in fp32 with plain PyTorch (no tiling), evaluated
    on the inputs' device (simulator.py:126-134).  Test/verification helper."""
    import torch

    t = {k: (v if isinstance(v, torch.Tensor) else torch.from_numpy(np.asarray(v))).float() for k, v in inputs.items()}
    a = t["A"]
    if graph.kind == GATED_FFN:
        c = torch.nn.functional.silu(a @ t["B0"]) * (a @ t["B1"])
    else:
        h = a @ t["B"]
        act = graph.activation
        c = {"identity": lambda x: x, "relu": torch.relu, "silu": torch.nn.functional.silu,
             "gelu": lambda x: torch.nn.functional.gelu(x, approximate="tanh")}[act](h)
    return c @ t["D"]


@dataclass
class VerifyReport:
    """simulator.py:432-458."""

    max_rel_error: float
    tolerance: float
    numerics_pass: bool
    parity: Optional[dict]
    parity_pass: Optional[bool]
    literal_mode: bool = False

    @property
    def passed(self) -> bool:
        return self.numerics_pass and (self.parity_pass is None or self.parity_pass)

    def to_dict(self) -> dict:
        return {"max_rel_error": self.max_rel_error, "tolerance": self.tolerance,
                "numerics_pass": self.numerics_pass, "parity_delta_bytes": self.parity,
                "parity_pass": self.parity_pass, "literal_mode": self.literal_mode, "pass": self.passed}


def verify(plan: FusionPlan, graph: ChainGraph, config: SimConfig = SimConfig(), check_parity: bool = True,
           device: Optional[DeviceModel] = None, literal: bool = False) -> VerifyReport:
    """Run on the GPU, compare with the fp32 dense reference computed from the
    same bf16-rounded inputs, and check replay == analyzer (simulator.py:461-487)."""
    import torch

    device = device or b200_profile()
    inputs = make_inputs(graph, config)
    dev = {k: torch.from_numpy(v).cuda().to(torch.bfloat16) for k, v in inputs.items()}
    result, trace = execute_plan(plan, graph, dev, config, device)
    reference = oracle(graph, dev)
    err = max_relative_error(result.float().cpu().numpy(), reference.cpu().numpy())
    parity = parity_pass = None
    if check_parity:
        vol = analyze(graph, device, plan, config.acc_size, literal=literal).volume
        parity = {t: trace.tier_bytes[t] - vol[t] for t in trace.tier_bytes}
        parity_pass = None if literal else all(v == 0 for v in parity.values())
    tol = config.effective_tolerance
    return VerifyReport(err, tol, err <= tol, parity, parity_pass, literal)


def unfused_baseline(graph: ChainGraph, inputs: dict, plan: FusionPlan):
    """Byte model of the two-kernel path, intermediate round-tripping global
    memory (simulator.py:495-556); E computed by two cuBLAS GEMMs + act."""
    trace = unfused_traffic(graph, plan)
    return oracle(graph, {k: _to_device(v) for k, v in inputs.items()}), trace


def unfused_traffic(graph: ChainGraph, plan: FusionPlan) -> TrafficTrace:
    """The byte trace of unfused_baseline alone (no inputs, no execution):
    tile loads replayed with singleton clusters, C stored in full and read once."""
    d = graph.dims
    elt = d.element_size
    blk = plan.tiles.block
    sched = plan.schedule
    trace = TrafficTrace()

    def kernel_loads(phase, tensors):
        spatial = [x for x in phase if x in sched.spatial]
        temporal = [x for x in sched.temporal_order if x in phase]
        trips = {x: d.size(x) // blk[x] for x in temporal}
        grid = prod(d.size(x) // blk[x] for x in spatial) if spatial else 1
        lv = {x: i + 1 for i, x in enumerate(temporal)}
        keys = {}
        for name, idx, _ in tensors:
            depth = max((lv[x] for x in idx if x in lv), default=0)
            keys[name] = [i for i, x in enumerate(temporal) if lv[x] <= depth]
        last = dict.fromkeys(keys)
        for leaf in itertools.product(*(range(trips[x]) for x in temporal)):
            for name, _, nbytes in tensors:
                key = tuple(leaf[i] for i in keys[name])
                if key != last[name]:
                    last[name] = key
                    trace.add_load(name, nbytes * grid)

    weights = ("B0", "B1") if graph.kind == GATED_FFN else ("B",)
    kernel_loads(("m", "n", "k"), [("A", ("m", "k"), blk["m"] * blk["k"] * elt)]
                 + [(w, ("k", "n"), blk["k"] * blk["n"] * elt) for w in weights])
    c_bytes = d.m * d.n * elt
    trace.add_store("C", c_bytes * ((d.k // blk["k"]) if "k" in sched.spatial else 1))
    trace.add_load("C", c_bytes)
    kernel_loads(("m", "n", "l"), [("D", ("n", "l"), blk["n"] * blk["l"] * elt)])
    trace.add_store("E", d.m * d.l * elt * ((d.n // blk["n"]) if "n" in sched.spatial else 1))
    return trace


def sample_valid_plans(graph: ChainGraph, device: DeviceModel, count: int, seed: int = 0,
                       acc_size: int = DEFAULT_ACC_SIZE, max_attempts: int = 200000) -> list:
    """Seeded random draws that pass every pruning rule (simulator.py:564-619);
    the same seed yields the same plans as the reference."""
    from .search import _k_choices, _rule2_clusters, _streams, rule4_dependency, rule5_capacity

    rng = random.Random(seed)
    streams = _streams(graph, device)
    clusters_of = {s.lowering: _rule2_clusters(s, device) for s in streams}
    schedules = enumerate_schedules(DIMS)
    out, seen = [], set()
    for _ in range(max_attempts):
        if len(out) >= count:
            break
        stream = streams[rng.randrange(len(streams))]
        schedule = schedules[rng.randrange(len(schedules))]
        if not rule4_dependency(schedule):
            continue
        options = clusters_of[stream.lowering]
        cluster = options[rng.randrange(len(options))]
        k_opts = _k_choices(stream, schedule, cluster, graph, False, stream.tiles_divisible["k"])
        if not k_opts:
            continue
        div = stream.tiles_divisible
        block = {"m": rng.choice(div["m"]), "n": rng.choice(div["n"]), "k": rng.choice(k_opts),
                 "l": rng.choice(div["l"])}
        plan = FusionPlan(schedule, TileSizes(block, dict(cluster)), stream.lowering)
        if structural_violations(plan, graph, device) or not rule5_capacity(plan, graph, device, acc_size):
            continue
        if plan.key in seen:
            continue
        seen.add(plan.key)
        out.append(plan)
    if len(out) < count:
        raise PlanError(f"could only sample {len(out)} of {count} valid plans")
    return out
