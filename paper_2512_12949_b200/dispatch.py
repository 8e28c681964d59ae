"""Run-time M-bin dispatch (paper SIV-C3 / Alg. 2 line 10).

A serving layer sees the same FFN weights with a different token count M on
every call, and the fused chain's best physical launch (transport, ring,
N splits, chunk/slice widths) depends on M.  Offline, `build_table` profiles
the candidate launches of one chain family (kind, activation, n, k, l) at the
upper edge of each M bin on the device (ProfileBestFromList over the
runtime's lowerings and, when the plan cache has them, the reference search's
top plans); at run time `Dispatcher` maps M to its bin and launches the stored
configuration -- a table lookup, no search, no profiling.

    disp = Dispatcher.load("plans/dispatch/llama1b.json")      # or build_table(...)
    E = disp.run({"A": A, "B0": B0, "B1": B1, "D": D})          # any M up to the last bin

The stored fields (exchange, ring, n_splits, nb, lb) do not depend on M; the
derived fields (m tiles, units, rings) are recomputed for the actual M by the
launch (finish_config), so one entry serves the whole bin.
"""

from __future__ import annotations

import bisect
import json
import os
from dataclasses import dataclass, field
from typing import Optional

from . import _native as nat
from .workload import DimensionSpec, build_gated_ffn, build_standard_ffn

DEFAULT_BINS = (64, 128, 256, 512, 1024, 2048, 4096, 8192)
_FIELDS = ("ring", "n_splits", "nb", "lb", "exchange")


def family_graph(kind: str, activation: str, m: int, n: int, k: int, l: int):
    dims = DimensionSpec(m, n, k, l, 2)
    return build_gated_ffn(dims) if kind == "gated_ffn" else build_standard_ffn(dims, activation)


def config_from_dict(d: dict) -> nat.KernelConfig:
    cfg = nat.KernelConfig()
    for name in _FIELDS:
        setattr(cfg, name, int(d[name]))
    return cfg


@dataclass
class Dispatcher:
    """M-bin -> physical launch table for one chain family."""

    kind: str
    activation: str
    n: int
    k: int
    l: int
    bins: list
    configs: list  # one dict of _FIELDS (+ measured ms) per bin
    meta: dict = field(default_factory=dict)

    def bin_of(self, m: int) -> int:
        if m < 1:
            raise ValueError("M must be positive")
        i = bisect.bisect_left(self.bins, m)
        if i == len(self.bins):
            raise ValueError(f"M={m} exceeds the table's last bin {self.bins[-1]}; rebuild with larger bins")
        return i

    def config_for(self, m: int) -> nat.KernelConfig:
        return config_from_dict(self.configs[self.bin_of(m)])

    def graph_for(self, m: int):
        return family_graph(self.kind, self.activation, m, self.n, self.k, self.l)

    def run(self, tensors: dict, out=None, stream=None):
        """Fused chain for tensors of any M up to the last bin (runtime.launch)."""
        from . import runtime

        m = int(tensors["A"].shape[0])
        return runtime.launch(self.graph_for(m), self.config_for(m), tensors, out=out, stream=stream)

    def to_dict(self) -> dict:
        return {"family": {"kind": self.kind, "activation": self.activation, "n": self.n, "k": self.k,
                           "l": self.l}, "bins": list(self.bins), "configs": self.configs, "meta": self.meta}

    @classmethod
    def from_dict(cls, doc: dict) -> "Dispatcher":
        f = doc["family"]
        return cls(f["kind"], f["activation"], f["n"], f["k"], f["l"], list(doc["bins"]), list(doc["configs"]),
                   dict(doc.get("meta", {})))

    def save(self, path: str) -> None:
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "w") as fh:
            json.dump(self.to_dict(), fh, sort_keys=True, indent=1)

    @classmethod
    def load(cls, path: str) -> "Dispatcher":
        with open(path) as fh:
            return cls.from_dict(json.load(fh))


def candidate_configs(graph, plans=(), labelled: bool = False, deterministic: bool = False) -> list:
    """Distinct lowerings of the runtime's auto configuration under every
    transport, plus the given plans' lowerings (no GPU needed).  labelled: (cfg,
    [sources]) pairs, a source per plan / transport that lowers to the config.
    deterministic: only bit-reproducible launches (runtime.is_deterministic)."""
    from . import runtime

    seen, out = {}, []
    xs = ("pair", "l2", "dsm", "l2dsm")
    sources = [(None, -1, x) for x in xs] + [(p, j, x) for j, p in enumerate(plans) for x in xs]
    sources += [(cfg, -2, "l2dsm") for cfg in runtime.reproducible_configs(graph, 148)]
    for plan, j, x in sources:
        if j == -2:  # an explicit reproducible launch (runtime.reproducible_configs)
            cfg, plan = plan, None
        else:
            try:
                cfg = runtime.lower(graph, plan, 148, x)
            except nat.UnsupportedPlan:
                continue
        if deterministic and not runtime.is_deterministic(graph, cfg, 148):
            continue
        key = tuple(int(getattr(cfg, f)) for f in _FIELDS)
        label = (f"reproducible ring {cfg.ring} x {cfg.n_splits} splits nb {cfg.nb} lb {cfg.lb} [{x}]" if j == -2
                 else f"runtime-auto [{x}]" if plan is None else f"searched #{j} {plan.describe()} [{x}]")
        if key in seen:
            seen[key][1].append(label)
        else:
            seen[key] = (cfg, [label])
            out.append(seen[key])
    return out if labelled else [c for c, _ in out]


TIE = 1.01  # a bit-reproducible launch within 1 % of the fastest wins (run-to-run identical E for free)


def pick_reproducible(graph, timed):
    """timed: [(ms, cfg, ...)] sorted by ms.  The fastest entry, unless a bit-reproducible
    launch (runtime.is_deterministic) is within TIE of it: then that one."""
    from . import runtime

    for entry in timed:
        if entry[0] > timed[0][0] * TIE:
            break
        if runtime.is_deterministic(graph, entry[1], 148):
            return entry
    return timed[0]


def build_table(kind: str, activation: str, n: int, k: int, l: int, bins=DEFAULT_BINS, iters: int = 10,
                warmup: int = 3, seed: int = 0, plans_by_m: Optional[dict] = None,
                deterministic: bool = False) -> Dispatcher:
    """Profile every candidate launch at each bin's upper edge (L2 flushed
    between timed launches) and keep the fastest: ProfileBestFromList per bin.
    Candidates: the runtime's lowerings under every transport plus the lowerings of
    the reference search's top-K plans for that M (plans_by_m, default: the
    shipped plans/plan_bins.json -- the offline-search leg, PAPER.md SIV-C3).
    deterministic: bit-reproducible launches only (a reproducible-serving table:
    every bin's winner writes the same E bits on every run)."""
    import torch

    from . import plan_cache, runtime

    if plans_by_m is None:
        plans_by_m = plan_cache.plans_by_m(kind, activation, n, k, l, bins)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    gen = torch.Generator(device="cpu").manual_seed(seed)

    def u(*shape):
        return (torch.rand(*shape, generator=gen) * 2 - 1).to(torch.bfloat16).cuda()

    weights = {"D": u(n, l)}
    if kind == "gated_ffn":
        w = u(2, k, n)
        weights["B0"], weights["B1"] = w[0], w[1]
    else:
        weights["B"] = u(k, n)
    configs = []
    for m in bins:
        graph = family_graph(kind, activation, m, n, k, l)
        tensors = dict(weights, A=u(m, k))
        out = torch.empty((m, l), dtype=torch.bfloat16, device="cuda")
        timed = []
        plans = plans_by_m.get(m, ())
        for cfg, labels in candidate_configs(graph, plans, labelled=True, deterministic=deterministic):
            for _ in range(warmup):
                runtime.launch(graph, cfg, tensors, out=out)
            ts = []
            for _ in range(iters):
                flush.add_(1.0)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                runtime.launch(graph, cfg, tensors, out=out)
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b))
            timed.append((sorted(ts)[len(ts) // 2], cfg, labels))
        timed.sort(key=lambda x: x[0])
        ms, best, labels = pick_reproducible(graph, timed)
        entry = {f: int(getattr(best, f)) for f in _FIELDS}
        entry["ms"] = round(ms, 5)
        entry["candidates"] = len(timed)
        entry["searched_plans"] = len(plans)
        entry["won_by"] = labels
        entry["timed"] = [[round(t * 1e3, 2), " = ".join(lb)] for t, _, lb in timed]
        configs.append(entry)
    return Dispatcher(kind, activation, n, k, l, list(bins), configs,
                      {"device": torch.cuda.get_device_name(), "method": "median of %d cold-L2 launches" % iters,
                       "candidates": "runtime lowerings (pair / l2 / dsm) + lowerings of the reference search's "
                                     "top-K plans per M bin (plans/plan_bins.json)"
                                     + ("; bit-reproducible launches only" if deterministic else "")})


# BASELINE.json families shipped with the package (plans/dispatch/*.json)
FAMILIES = {
    "llama1b": ("gated_ffn", "silu", 8192, 2048, 2048),
    "gpt67b": ("standard_ffn", "relu", 16384, 4096, 4096),
    "gpt2s": ("standard_ffn", "gelu", 3072, 768, 768),
    "opt13b": ("standard_ffn", "relu", 8192, 2048, 2048),
}
TABLE_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "plans", "dispatch")


def shipped(name: str) -> Dispatcher:
    return Dispatcher.load(os.path.join(TABLE_DIR, f"{name}.json"))


if __name__ == "__main__":  # python -m paper_2512_12949_b200.dispatch  (on a GPU box)
    for name, fam in FAMILIES.items():
        table = build_table(*fam)
        table.save(os.path.join(TABLE_DIR, f"{name}.json"))
        print(name, [(b, c["exchange"], c["ring"], c["n_splits"], c["ms"]) for b, c in zip(table.bins, table.configs)])
