"""DOT views of a fused chain (the reference's tile graph,
tilegraph.py:24-113, drawn for the CLI's export-dot).

`export_tilegraph(graph, plan)` draws one cluster step of the *logical* plan:
the CTAs (im, in, ik) of the cluster with their GEMM0 partial tiles, the
dsm_comm primitives between them (all_exchange over the cls_k CTAs sharing a
C tile, the shuffle ring of cls_l/cls_k members, the reduce-scatter of the E
partials over the cls_reduce sets) and the input / output tiles, every edge
labelled with its bytes per step (inputs in element_size, exchanged
accumulators in acc_size, as the analyzer counts them, analyzer.py:331-354).

`export_launch_graph(graph, cfg)` draws what the sm_100a launch executes for
one ring: its members (CTAs or CTA pairs), the C chunk each publishes per
n-step and who consumes it (DSM push or L2 scratch), the E slice each
accumulates and the split-N reduction across rings.
"""

from __future__ import annotations

from .plan import LOWERING_SPATIAL_SPLIT, FusionPlan, plan_geometry
from .workload import DIMS, GATED_FFN, ChainGraph

DEFAULT_ACC_SIZE = 4


def _b(n: int) -> str:
    for unit, shift in (("MiB", 20), ("KiB", 10)):
        if n >= 1 << shift:
            return f"{n / (1 << shift):.1f}{unit}"
    return f"{n}B"


def _q(s: str) -> str:
    return '"' + s.replace('"', "'") + '"'


def export_tilegraph(graph: ChainGraph, plan: FusionPlan, acc_size: int = DEFAULT_ACC_SIZE) -> str:
    geo = plan_geometry(graph, plan)
    cl = geo.cluster
    tile = {d: geo.cover[d] // geo.split[d] for d in DIMS}  # one CTA's block
    elt = graph.dims.element_size
    gated = graph.kind == GATED_FFN
    spatial_split = gated and plan.gated_lowering == LOWERING_SPATIAL_SPLIT
    g1 = max(1, cl.cls_shuffle)
    c_acc = tile["m"] * tile["n"] * acc_size
    e_acc = tile["m"] * tile["l"] * acc_size
    out = [f"digraph {_q('cluster_step ' + plan.describe())} {{", "  rankdir=LR;",
           f"  label={_q(f'{graph.kind} {graph.dims.as_tuple()}  one cluster step: {cl.cls_m}x{cl.cls_n}x{cl.cls_k} CTAs')};",
           "  node [shape=box, fontsize=10];"]
    weights = ("B0", "B1") if gated else ("B",)
    tm, tn, tk, tl = tile["m"], tile["n"], tile["k"], tile["l"]
    out.append(f"  A [label={_q(f'A tile {tm}x{tk} ({_b(tm * tk * elt)})')}, shape=folder];")
    for w in weights:
        out.append(f"  {w} [label={_q(f'{w} tile {tk}x{tn} ({_b(tk * tn * elt)})')}, shape=folder];")
    out.append(f"  D [label={_q(f'D tile {tn}x{tl} ({_b(tn * tl * elt)})')}, shape=folder];")
    out.append(f"  E [label={_q(f'E store {tm}x{tl} ({_b(tm * tl * elt)})')}, shape=folder];")
    ctas = [(im, i_n, ik) for im in range(cl.cls_m) for i_n in range(cl.cls_n) for ik in range(cl.cls_k)]
    for im, i_n, ik in ctas:
        name = f"cta_{im}_{i_n}_{ik}"
        branch = ""
        if spatial_split:
            branch = " gate" if ik < cl.cls_k // 2 else " up"
        ir, il = i_n // g1, ik * g1 + i_n % g1
        out.append(f"  {name} [label={_q(f'CTA ({im},{i_n},{ik}){branch}\\nC partial {_b(c_acc)}  E[{il}] set {ir}')}];")
        out.append(f"  A -> {name} [label={_q(_b(tile['m'] * tile['k'] * elt))}];")
        w = ("B0" if ik < cl.cls_k // 2 else "B1") if spatial_split else weights[ik % len(weights)]
        out.append(f"  {w} -> {name} [label={_q(_b(tile['k'] * tile['n'] * elt))}];")
        out.append(f"  D -> {name} [label={_q(_b(tile['n'] * tile['l'] * elt))}, style=dotted];")
    # all_exchange over the cls_k CTAs sharing (im, in)
    for im in range(cl.cls_m):
        for i_n in range(cl.cls_n):
            for a in range(cl.cls_k):
                for b in range(cl.cls_k):
                    if a != b:
                        op = "Mul" if spatial_split else "Add"
                        out.append(f"  cta_{im}_{i_n}_{a} -> cta_{im}_{i_n}_{b} "
                                   f"[label={_q(f'all_exchange {op} {_b(c_acc)}')}, color=blue];")
    # shuffle ring among the g1 members of a reduce set
    if g1 > 1:
        for im in range(cl.cls_m):
            for ik in range(cl.cls_k):
                for ir in range(cl.cls_n // g1):
                    ring = [ir * g1 + j for j in range(g1)]
                    for j, i_n in enumerate(ring):
                        nxt = ring[(j + 1) % g1]
                        out.append(f"  cta_{im}_{i_n}_{ik} -> cta_{im}_{nxt}_{ik} "
                                   f"[label={_q(f'shuffle {_b(c_acc)}')}, color=darkgreen];")
    # reduce-scatter of the E partials over the cls_reduce sets, then the store
    for im, i_n, ik in ctas:
        out.append(f"  cta_{im}_{i_n}_{ik} -> E [label={_q(f'reduce_scatter {_b(e_acc // max(1, cl.cls_reduce))}')}, "
                   f"color=red];")
    out.append("}")
    return "\n".join(out) + "\n"


def export_launch_graph(graph: ChainGraph, cfg) -> str:
    """One ring of the physical sm_100a launch (ffKernelConfig from runtime.lower)."""
    G, S = int(cfg.ring), int(cfg.n_splits)
    pair = int(cfg.exchange) == 2
    transport = {0: "DSM push (cp.async.bulk.shared::cluster)", 1: "L2 scratch (TMA store / load)",
                 2: "L2 scratch, CTA pairs (cta_group::2)"}[int(cfg.exchange)]
    rows = 256 if pair else 128
    chunk = rows * int(cfg.nb) * graph.dims.element_size
    d = graph.dims
    out = [f"digraph {_q('launch ring')} {{", "  rankdir=LR;",
           f"  label={_q(f'{graph.kind} {d.as_tuple()}: {cfg.rings} rings x {G} members ({transport}), '
                         f'{S} N splits, {cfg.steps} n-steps / unit, {cfg.units} units')};",
           "  node [shape=box, fontsize=10];"]
    for p in range(G):
        who = "CTA pair" if pair else "CTA"
        out.append(f"  m{p} [label={_q(f'{who} {p}: E[:, {p * cfg.lb}:{(p + 1) * cfg.lb}] in TMEM\\n'
                                       f'GEMM0 chunk {rows}x{cfg.nb} per n-step')}];")
    for p in range(G):
        for h in range(1, G):
            out.append(f"  m{p} -> m{(p + h) % G} [label={_q(f'C chunk {_b(chunk)} (hop {h})')}, color=darkgreen];")
    if S > 1:
        out.append(f"  partials [label={_q(f'split-N reduce of {S} E partials (fp32)')}, shape=ellipse];")
        for p in range(G):
            out.append(f"  m{p} -> partials [color=red];")
        out.append(f"  partials -> E [label={_q('bf16 E rows')}];")
    else:
        for p in range(G):
            out.append(f"  m{p} -> E [label={_q('bf16 E slice')}];")
    out.append(f"  E [label={_q(f'E {d.m}x{d.l}')}, shape=folder];")
    out.append("}")
    return "\n".join(out) + "\n"
