"""Dataflow analyzer (paper Alg. 1; fuseplan/analyzer.py): closed-form per-tier
byte volumes and the greedy resource mapping of the reused tensors.

Conventions (normative, analyzer.py:1-28): inputs stream global -> smem and a
tile reloads whenever a temporal loop at or outside its innermost indexing
loop advances; the intermediate C is materialised once per region in
completion mode and streamed in increment mode; C and the E accumulator are
placed greedily reg -> smem -> dsm (-> l2 -> global for E) with l2 charges
accounted to global; DSM primitive bytes are received bytes.

Every integer produced here must equal the reference bit for bit -- the
search ranks on it.  ``_volume_core`` is the single implementation; the full
:func:`analyze` report and the search's ranking fast path both call it.
"""

from __future__ import annotations

from dataclasses import dataclass
from math import prod
from typing import Optional

from .errors import CapacityExceeded, WrongTensorClass
from .hardware import DeviceModel
from .plan import LOWERING_DOUBLED_K, FusionPlan, PlanGeometry, plan_geometry
from .workload import DIMS, GATED_FFN, ROLE_INTERMEDIATE, ROLE_OUTPUT, ChainGraph

TIERS = ("reg", "smem", "dsm", "l2", "global")   # analyzer.py:47
DEFAULT_ACC_SIZE = 4                             # analyzer.py:48
_FIRST_GEMM = frozenset("mnk")
_SECOND_GEMM = frozenset("mnl")
_ALL = frozenset(DIMS)


def tile_footprint(tensor, block: dict, element_size: int) -> int:
    """Bytes of one block tile (analyzer.py:51-57)."""
    return prod(block[d] for d in DIMS if tensor.indexed_by(d)) * element_size


@dataclass(frozen=True)
class EventCounts:
    """Per-block load multipliers and per-cluster firing counts (analyzer.py:65-74)."""

    a_loads: int
    b_loads: int
    d_loads: int
    exchanges: int
    gemm1_fires: int
    stores: int


def _event_counts(geom: PlanGeometry, levels: dict) -> EventCounts:
    """analyzer.py:77-110."""
    nest = sorted((depth, d) for d, depth in levels.items())
    trips = geom.trips

    def innermost(dims) -> int:
        return max((depth for depth, d in nest if d in dims), default=0)

    def trips_through(depth: int, allowed) -> int:
        out = 1
        for lvl, d in nest:
            if lvl <= depth and d in allowed:
                out *= trips[d]
        return out

    def trips_of(dims) -> int:
        return prod(trips[d] for d in dims if d in levels)

    scope0, scope1 = (_FIRST_GEMM, _SECOND_GEMM) if geom.completion_mode else (_ALL, _ALL)
    a = trips_through(innermost("mk"), scope0)
    b = trips_through(innermost("kn"), scope0)
    d = trips_through(innermost("nl"), scope1)
    if geom.completion_mode:
        exchanges, fires = trips_of("mn"), trips_of("mnl")
    else:
        exchanges = trips_through(innermost("mnk"), _ALL)
        fires = trips_through(innermost("mnl"), _ALL)
    return EventCounts(a, b, d, exchanges, fires, trips_of("ml"))


def live_tile_counts(graph: ChainGraph, plan: FusionPlan, geom: Optional[PlanGeometry] = None) -> dict:
    """Live regions of C and E in tiles (analyzer.py:118-151)."""
    geom = geom or plan_geometry(graph, plan)
    levels = geom.levels
    big = 10 ** 9

    def spans(dim: str, drivers) -> bool:
        depth = levels.get(dim)
        return depth is not None and any(levels.get(x, big) < depth for x in drivers)

    t = geom.trips
    if geom.completion_mode:
        c_live = {"m": t["m"] if spans("m", "l") else 1, "n": t["n"] if spans("n", "l") else 1}
        drivers = "n"
    else:
        c_live = {"m": 1, "n": 1}
        drivers = "nk"
    e_live = {"m": t["m"] if spans("m", drivers) else 1, "l": t["l"] if spans("l", drivers) else 1}
    return {"C": c_live, "E": e_live}


def place_tensor(footprint_bytes: int, levels, spill_floor: str, occupancy: dict, tensor_name: str = "?") -> dict:
    """Greedy fill of an ordered (name, capacity|None) sequence down to the floor (analyzer.py:159-185)."""
    out, left = {}, int(footprint_bytes)
    for name, cap in levels:
        if left <= 0:
            break
        room = left if cap is None else max(0, int(cap) - occupancy.get(name, 0))
        take = min(left, room)
        if take > 0:
            out[name] = take
            occupancy[name] = occupancy.get(name, 0) + take
            left -= take
        if name == spill_floor:
            break
    if left > 0:
        raise CapacityExceeded(tensor_name, spill_floor, left)
    return out


class ResourcePlacer:
    """Per-block capacities; smem allocations also debit the pooled dsm share
    (analyzer.py:188-253)."""

    def __init__(self, device: DeviceModel, geom: PlanGeometry):
        smem = int(device.smem.capacity_bytes)
        blocks = geom.num_clusters * geom.blocks
        l2 = int(device.l2.capacity_bytes) // blocks if device.l2 is not None and blocks > 0 else None
        self.capacity = {"reg": int(device.reg.capacity_bytes), "smem": smem, "dsm": smem, "l2": l2, "global": None}
        self.occupancy = dict.fromkeys(TIERS, 0)

    def levels_down_to(self, floor: str) -> list:
        out = []
        for name in TIERS:
            if name == "l2" and self.capacity["l2"] is None:
                continue
            out.append((name, self.capacity[name]))
            if name == floor:
                break
        return out

    def place(self, name: str, footprint: int, floor: str) -> dict:
        out, left = {}, int(footprint)
        for level, cap in self.levels_down_to(floor):
            if left <= 0:
                break
            room = left if cap is None else max(0, int(cap) - self.occupancy[level])
            take = min(left, room)
            if take > 0:
                out[level] = take
                self.occupancy[level] += take
                if level == "smem":
                    self.occupancy["dsm"] += take
                left -= take
            if level == floor:
                break
        if left > 0:
            raise CapacityExceeded(name, floor, left)
        return out

    def headroom(self) -> dict:
        return {t: (None if self.capacity[t] is None else max(0, self.capacity[t] - self.occupancy[t]))
                for t in TIERS}


def slot_tier_bytes(mapping: dict, region_tiles: int, tile_bytes: int) -> list:
    """Byte split of each region slot across the tiers it straddles (analyzer.py:256-277)."""
    spans, lo = [], 0
    for name in TIERS:
        if name in mapping:
            spans.append((lo, lo + mapping[name], name))
            lo += mapping[name]
    out = []
    for slot in range(region_tiles):
        s_lo, s_hi = slot * tile_bytes, (slot + 1) * tile_bytes
        split = {}
        for a, b, name in spans:
            n = min(s_hi, b) - max(s_lo, a)
            if n > 0:
                split[name] = split.get(name, 0) + n
        out.append(split)
    return out


def region_tier_totals(mapping: dict) -> dict:
    """Allocation level -> traffic tier; l2 residency is charged to global (analyzer.py:280-285)."""
    out = dict.fromkeys(TIERS, 0)
    for name, nbytes in mapping.items():
        out["global" if name == "l2" else name] += nbytes
    return out


def _input_load_totals(graph: ChainGraph, geom: PlanGeometry, ev: EventCounts) -> dict:
    """Global load bytes per input tensor (analyzer.py:293-315)."""
    elt = graph.dims.element_size
    blk = geom.block
    ntb = geom.num_clusters * geom.blocks
    out = {
        "A": ev.a_loads * blk["m"] * blk["k"] * elt * ntb,
        "D": ev.d_loads * geom.cluster.cls_shuffle * blk["n"] * blk["l"] * elt * ntb,
    }
    weights = ev.b_loads * blk["k"] * blk["n"] * elt * ntb
    if graph.kind == GATED_FFN:
        out["B0"] = out["B1"] = weights // 2
    else:
        out["B"] = weights
    return out


def _store_totals(graph: ChainGraph, geom: PlanGeometry, ev: EventCounts) -> tuple:
    """(plain store bytes, extra inter-cluster reduce bytes) of E (analyzer.py:318-328)."""
    blk = geom.block
    cl = geom.cluster
    total = geom.num_clusters * ev.stores * cl.cls_m * cl.cls_l * blk["m"] * blk["l"] * graph.dims.element_size
    base = total // (geom.grid["n"] * geom.grid["k"])
    return base, total - base


def dsm_traffic(graph: ChainGraph, plan: FusionPlan, acc_size: int = DEFAULT_ACC_SIZE,
                geom: Optional[PlanGeometry] = None, events: Optional[EventCounts] = None) -> dict:
    """Received fabric bytes per dsm_comm primitive (analyzer.py:331-354)."""
    geom = geom or plan_geometry(graph, plan)
    ev = events or _event_counts(geom, geom.levels)
    cl = geom.cluster
    blk = geom.block
    f_c = blk["m"] * blk["n"] * acc_size
    f_e = blk["m"] * blk["l"] * acc_size
    payload = 2 * f_c if plan.gated_lowering == LOWERING_DOUBLED_K and cl.cls_k > 1 else f_c
    n = geom.num_clusters
    return {
        "all_exchange": n * ev.exchanges * geom.blocks * (cl.cls_k - 1) * payload,
        "shuffle": n * ev.gemm1_fires * geom.blocks * (cl.cls_shuffle - 1) * f_c,
        "reduce_scatter": n * ev.stores * cl.cls_m * cl.cls_l * (cl.cls_reduce - 1) * f_e,
    }


def io_traffic(graph: ChainGraph, plan: FusionPlan, tensor_name: str, literal: bool = False) -> int:
    """Global bytes of one input/output tensor (analyzer.py:357-380)."""
    tensor = graph.tensor(tensor_name)
    if tensor.role == ROLE_INTERMEDIATE:
        raise WrongTensorClass(f"{tensor_name} is the intermediate; io_traffic covers inputs and outputs")
    geom = plan_geometry(graph, plan)
    if literal:
        blk = geom.block
        out = tile_footprint(tensor, blk, graph.dims.element_size)
        for d in DIMS:
            if tensor.indexed_by(d) and d in geom.levels:
                out *= -(-geom.eff[d] // blk[d])
        return out
    ev = _event_counts(geom, geom.levels)
    if tensor.role == ROLE_OUTPUT:
        return sum(_store_totals(graph, geom, ev))
    return _input_load_totals(graph, geom, ev)[tensor_name]


@dataclass
class AnalysisResult:
    volume: dict
    primitives: dict
    per_tensor: dict
    mapping: dict
    headroom: dict
    live_tiles: dict
    mode: str
    plan: FusionPlan

    def report_dict(self) -> dict:
        """analyzer.py:399-410."""
        return {
            "volume_bytes": {t: int(self.volume[t]) for t in TIERS},
            "primitives_bytes": {k: int(v) for k, v in sorted(self.primitives.items())},
            "per_tensor": {k: dict(v) for k, v in sorted(self.per_tensor.items())},
            "mapping": {t: dict(sorted(m.items())) for t, m in sorted(self.mapping.items())},
            "headroom_bytes": {k: (None if v is None else int(v)) for k, v in self.headroom.items()},
            "live_tiles": {t: dict(v) for t, v in sorted(self.live_tiles.items())},
            "mode": self.mode,
        }


def _volume_core(graph: ChainGraph, device: DeviceModel, plan: FusionPlan, acc_size: int,
                 geom: PlanGeometry, literal: bool = False):
    """The whole of Algorithm 1; returns (volume, prims, per_tensor, mapping, placer, live)."""
    ev = _event_counts(geom, geom.levels)
    blk = geom.block
    live = live_tile_counts(graph, plan, geom)
    f_c = blk["m"] * blk["n"] * acc_size
    f_e = blk["m"] * blk["l"] * acc_size

    placer = ResourcePlacer(device, geom)
    mapping = {
        "C": placer.place("C", live["C"]["m"] * live["C"]["n"] * f_c, graph.intermediate.spill_floor),
    }
    mapping["E"] = placer.place("E", live["E"]["m"] * live["E"]["l"] * f_e, graph.output.spill_floor)

    volume = dict.fromkeys(TIERS, 0)
    if literal:
        loads = {t.name: io_traffic(graph, plan, t.name, literal=True) for t in graph.inputs}
        base, extra = io_traffic(graph, plan, "E", literal=True), 0
    else:
        loads = _input_load_totals(graph, geom, ev)
        base, extra = _store_totals(graph, geom, ev)
    per_tensor = {}
    for name, nbytes in loads.items():
        per_tensor[name] = {"loads": nbytes}
        volume["global"] += nbytes
        volume["smem"] += nbytes
    per_tensor["E"] = {"stores": base + extra}
    volume["global"] += base + extra

    prims = dsm_traffic(graph, plan, acc_size, geom, ev)
    volume["dsm"] += sum(prims.values())
    prims["inter_cluster_reduce"] = extra

    scale = geom.num_clusters * geom.blocks
    t = geom.trips
    if geom.completion_mode:
        sweeps = (t["m"] // live["C"]["m"]) * (t["n"] // live["C"]["n"])
        touches = sweeps * (1 + t["l"])
        for tier, nbytes in region_tier_totals(mapping["C"]).items():
            volume[tier] += touches * nbytes * scale
    sweeps = (t["m"] // live["E"]["m"]) * (t["l"] // live["E"]["l"])
    touches = sweeps * (2 * (ev.gemm1_fires // (t["m"] * t["l"])) + 1)
    for tier, nbytes in region_tier_totals(mapping["E"]).items():
        volume[tier] += touches * nbytes * scale
    return volume, prims, per_tensor, mapping, placer, live


def analyze(graph: ChainGraph, device: DeviceModel, plan: FusionPlan,
            acc_size: int = DEFAULT_ACC_SIZE, literal: bool = False) -> AnalysisResult:
    """Algorithm 1 DataflowAnalyzer (analyzer.py:413-489)."""
    geom = plan_geometry(graph, plan)
    volume, prims, per_tensor, mapping, placer, live = _volume_core(graph, device, plan, acc_size, geom, literal)
    return AnalysisResult(volume, prims, per_tensor, mapping, placer.headroom(), live,
                          "completion" if geom.completion_mode else "increment", plan.with_mapping(mapping))


def placement_feasible(graph: ChainGraph, device: DeviceModel, plan: FusionPlan,
                       acc_size: int = DEFAULT_ACC_SIZE) -> bool:
    """Capacity rule (analyzer.py:492-509)."""
    try:
        geom = plan_geometry(graph, plan)
    except Exception:
        return False
    blk = geom.block
    live = live_tile_counts(graph, plan, geom)
    placer = ResourcePlacer(device, geom)
    try:
        placer.place("C", live["C"]["m"] * live["C"]["n"] * blk["m"] * blk["n"] * acc_size,
                     graph.intermediate.spill_floor)
        placer.place("E", live["E"]["m"] * live["E"]["l"] * blk["m"] * blk["l"] * acc_size,
                     graph.output.spill_floor)
    except CapacityExceeded:
        return False
    return True
