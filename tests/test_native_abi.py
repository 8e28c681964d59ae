"""The C-ABI library loads, exports exactly what include/*.h declares, its
struct layouts match the ctypes mirror, and the (host-only) lowering entry
points behave -- no GPU needed."""

import ctypes
import json
import os
import re
import subprocess

import pytest

from paper_2512_12949_b200 import _native as nat
from paper_2512_12949_b200 import runtime
from paper_2512_12949_b200 import workload as W
from paper_2512_12949_b200.errors import PlanError
from paper_2512_12949_b200.plan import make_plan, plan_from_dict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INC = os.path.join(ROOT, "include")


def declared_symbols():
    names = set()
    for fname in os.listdir(INC):
        text = open(os.path.join(INC, fname)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names |= set(re.findall(r"\b(ff_\w+)\s*\(", text))
    return names


@pytest.fixture(scope="module")
def lib():
    from paper_2512_12949_b200 import build

    build.build()
    return nat.load()


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", nat.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (ff_\w+)", out))
    declared = declared_symbols()
    assert declared, "no declarations parsed"
    assert declared <= exported, f"missing: {declared - exported}"
    assert set(nat.EXPORTS) <= exported


def test_struct_layouts_match_the_header(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include "ff_chain.h"\n'
                   'int main(void){printf("%zu %zu %zu %zu %zu\\n", sizeof(ffChainDesc), sizeof(ffPlanDesc),'
                   ' sizeof(ffKernelConfig), sizeof(ffTensors), sizeof(ffConvDesc));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", INC, str(src), "-o", str(exe)], check=True)
    sizes = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert sizes == [ctypes.sizeof(nat.ChainDesc), ctypes.sizeof(nat.PlanDesc), ctypes.sizeof(nat.KernelConfig),
                     ctypes.sizeof(nat.Tensors), ctypes.sizeof(nat.ConvDesc)]


def _check_cfg(graph, cfg):
    d = graph.dims
    width = 2 if cfg.exchange == nat.XCHG_L2_PAIR else 1
    assert d.l % (cfg.ring * cfg.lb) == 0
    if cfg.exchange == nat.XCHG_L2_PAIR:  # ceil(chunks / S) chunks per split, ragged last n-step
        assert d.n % cfg.nb == 0
        chunks = d.n // cfg.nb
        per = -(-chunks // cfg.n_splits)
        assert chunks - (cfg.n_splits - 1) * per >= 1
        assert cfg.steps == -(-per // cfg.ring)
    else:
        assert d.n % (cfg.n_splits * cfg.ring * cfg.nb) == 0
    assert cfg.m_tiles == -(-d.m // (128 * width))
    assert cfg.units == cfg.m_tiles * cfg.l_clusters * cfg.n_splits
    assert 1 <= cfg.rings <= cfg.units
    assert cfg.grid_ctas == cfg.rings * cfg.ring * width <= 148
    if cfg.exchange == nat.XCHG_DSM:
        assert cfg.ring <= 16


def test_lowering_of_reference_top_plans(lib):
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "search_results.json")))
    lowered = 0
    for name, case in gold.items():
        if not name.startswith("b200_"):
            continue
        g = case["graph"]
        dims = W.DimensionSpec(g["m"], g["n"], g["k"], g["l"], 2)
        graph = W.build_gated_ffn(dims) if g["kind"] == "gated_ffn" else W.build_standard_ffn(dims, "relu")
        for entry in case["result"]["top"][:3]:
            plan = plan_from_dict(entry["plan"])
            for exchange in ("dsm", "l2", "pair"):
                try:
                    cfg = runtime.lower(graph, plan, 148, exchange)
                except nat.UnsupportedPlan:
                    continue
                _check_cfg(graph, cfg)
                lowered += 1
    assert lowered >= 10


@pytest.mark.parametrize("dims,kind", [((512, 8192, 2048, 2048), "gated_ffn"), ((512, 16384, 4096, 4096), "standard_ffn"),
                                       ((512, 3072, 768, 768), "standard_ffn"), ((3136, 64, 576, 256), "standard_ffn"),
                                       ((4096, 8192, 2048, 2048), "standard_ffn"), ((200, 768, 256, 768), "standard_ffn"),
                                       ((512, 11008, 4096, 4096), "gated_ffn"), ((256, 8960, 1536, 1536), "standard_ffn")])
def test_auto_config_invariants(lib, dims, kind):
    d = W.DimensionSpec(*dims, 2)
    graph = W.build_gated_ffn(d) if kind == "gated_ffn" else W.build_standard_ffn(d, "relu")
    ok = 0
    for exchange in ("dsm", "l2", "pair"):
        try:
            cfg = runtime.lower(graph, None, 148, exchange)
        except nat.UnsupportedPlan:
            continue
        _check_cfg(graph, cfg)
        ok += 1
    assert ok >= 1


@pytest.mark.parametrize("dims,kind,expect", [
    ((512, 11008, 4096, 4096), "gated_ffn", (16, 2, 3)),      # LLaMA-7B: 86 chunks, 43 per split, last step 11 of 16
    ((256, 8960, 1536, 1536), "standard_ffn", (6, 4, 2)),     # 35 chunks: splits of 9, 9, 9, 8
    ((512, 16384, 4096, 4096), "standard_ffn", (16, 2, 2)),   # whole steps: unchanged
])
def test_pair_lowering_takes_ragged_rings(lib, dims, kind, expect):
    """The pair transport keeps the widest ring when N / nb is not a ring multiple
    (ceil(chunks / S) chunks per split, ragged last n-step) instead of falling back
    to l clusters that recompute GEMM0."""
    d = W.DimensionSpec(*dims, 2)
    graph = W.build_gated_ffn(d) if kind == "gated_ffn" else W.build_standard_ffn(d, "relu")
    cfg = runtime.lower(graph, None, 148, "pair")
    assert (cfg.ring, cfg.n_splits, cfg.steps) == expect and cfg.l_clusters == 1
    _check_cfg(graph, cfg)


def test_status_codes_map_to_reference_exceptions(lib):
    graph = W.build_standard_ffn(W.DimensionSpec(256, 1024, 256, 1024, 2), "relu")
    bad = make_plan("ml", "nk", (64, 256, 256, 256), (1, 4, 1, 4))  # l grid-spatial (Rule 4)
    with pytest.raises(PlanError):
        runtime.lower(graph, bad, 148, "dsm")
    gated_plan_on_standard = make_plan("n", "klm", (64, 256, 256, 256), (1, 4, 1, 4), "doubled_k")
    with pytest.raises(PlanError):
        runtime.lower(graph, gated_plan_on_standard, 148, "l2")
    odd = W.build_standard_ffn(W.DimensionSpec(256, 1000, 256, 1024, 2), "relu")  # n not a multiple of 64
    with pytest.raises(nat.UnsupportedPlan):
        runtime.lower(odd, None, 148, "l2")
    f32 = W.build_standard_ffn(W.DimensionSpec(256, 1024, 256, 1024, 4), "relu")
    with pytest.raises(nat.UnsupportedPlan):
        runtime.lower(f32, None, 148, "l2")


def test_workspace_sizes(lib):
    graph = W.build_standard_ffn(W.DimensionSpec(512, 16384, 4096, 4096, 2), "relu")
    for exchange in ("dsm", "l2", "pair"):
        cfg = runtime.lower(graph, None, 148, exchange)
        ch = runtime.chain_desc(graph)
        need = lib.ff_chain_workspace_bytes(ctypes.byref(ch), ctypes.byref(cfg))
        if cfg.n_splits > 1:
            assert need >= 512 * 4096 * 4
        if exchange != "dsm" and cfg.ring > 1:
            assert need >= 512 * 16384 * 2


def test_launch_argument_errors_without_touching_the_gpu(lib):
    """ff_chain_launch rejects bad arguments before any CUDA work (FF_ERR_ARG = 5)."""
    graph = W.build_standard_ffn(W.DimensionSpec(256, 1024, 256, 1024, 2), "relu")
    cfg = runtime.lower(graph, None, 148, "l2")
    ch = runtime.chain_desc(graph)
    need = lib.ff_chain_workspace_bytes(ctypes.byref(ch), ctypes.byref(cfg))
    assert need > 0
    null = nat.Tensors(None, None, None, None, None)
    assert lib.ff_chain_launch(ctypes.byref(ch), ctypes.byref(cfg), ctypes.byref(null), None, 0, None) == 5
    odd = nat.Tensors(0x1000 + 8, 0x2000, None, 0x3000, 0x4000)  # A not 16-byte aligned
    assert lib.ff_chain_launch(ctypes.byref(ch), ctypes.byref(cfg), ctypes.byref(odd), 0x100000, need, None) == 5
    ok = nat.Tensors(0x1000, 0x2000, None, 0x3000, 0x4000)
    assert lib.ff_chain_launch(ctypes.byref(ch), ctypes.byref(cfg), ctypes.byref(ok), 0x100000, need - 1, None) == 5
    assert b"workspace" in lib.ff_last_error()
    bad_dtype = runtime.chain_desc(graph)
    bad_dtype.dtype = 7
    assert lib.ff_chain_launch(ctypes.byref(bad_dtype), ctypes.byref(cfg), ctypes.byref(ok), 0x100000, need, None) == 5


def test_run_plan_rejects_plans_without_lowering(lib):
    """ff_chain_run_plan / ff_plan_workspace_bytes on a plan the lowering refuses: a
    status code and a message, workspace size 0, nothing launched (no GPU needed)."""
    graph = W.build_standard_ffn(W.DimensionSpec(256, 1024, 256, 1024), "relu")
    plan = make_plan("n", "klm", (64, 256, 512, 256), (1, 4, 1, 4), "doubled_k")  # gated lowering, standard chain
    ch, pd = runtime.chain_desc(graph), runtime.plan_desc(plan)
    assert lib.ff_plan_workspace_bytes(ctypes.byref(ch), ctypes.byref(pd)) == 0
    t = nat.Tensors(256, 256, None, 256, 256)
    rc = lib.ff_chain_run_plan(ctypes.byref(ch), ctypes.byref(pd), ctypes.byref(t), None, 0, None)
    assert rc == nat.FF_ERR_PLAN
    assert b"gated lowering" in lib.ff_last_error()
    with pytest.raises(PlanError):
        nat.check(rc)


def test_deterministic_predicate_and_selection(lib):
    """ff_config_deterministic: one N split, the DSM reduce-scatter and the pair kernel's region
    finish are bit-reproducible; 1-CTA rings that reduce-add their splits are not.  lower(...,
    deterministic=True) picks a reproducible launch or refuses (host logic, no GPU)."""
    gpt2s = W.build_standard_ffn(W.DimensionSpec(512, 3072, 768, 768, 2), "relu")
    llama = W.build_gated_ffn(W.DimensionSpec(512, 8192, 2048, 2048, 2))
    opt = W.build_standard_ffn(W.DimensionSpec(4096, 8192, 2048, 2048, 2), "relu")
    for g in (gpt2s, llama):
        l2 = runtime.lower(g, None, 148, "l2")
        assert l2.n_splits > 1 and not runtime.is_deterministic(g, l2)
        assert runtime.is_deterministic(g, runtime.lower(g, None, 148, "l2dsm"))
        assert runtime.is_deterministic(g, runtime.lower(g, None, 148, "pair"))
        with pytest.raises(nat.UnsupportedPlan):
            runtime.lower(g, None, 148, "l2", deterministic=True)
        det = runtime.lower(g, None, 148, "auto", deterministic=True)
        assert runtime.is_deterministic(g, det)
    one = runtime.lower(opt, None, 148, "l2")
    assert one.n_splits == 1 and runtime.is_deterministic(opt, one)
    # a multi-unit pair launch with N splits finishes by reduce-adds
    multi = runtime.lower(opt, None, 148, "pair")
    multi.n_splits = 2
    assert not runtime.is_deterministic(opt, multi)
    out = ctypes.c_int32(7)
    assert lib.ff_config_deterministic(ctypes.byref(runtime.chain_desc(opt)), None, 148, ctypes.byref(out)) == nat.FF_ERR_ARG


def test_config_finish_and_reproducible_configs(lib):
    """ff_config_finish completes an explicit launch like ff_chain_launch will; the explicit DSM
    reduce-scatter launches are all bit-reproducible and co-resident (host logic, no GPU)."""
    g = W.build_standard_ffn(W.DimensionSpec(512, 3072, 768, 768, 2), "gelu")
    cfg = runtime.explicit_config(g, 6, 4, 128, 128, "l2dsm")
    assert (cfg.m_tiles, cfg.l_clusters, cfg.steps, cfg.units, cfg.rings, cfg.grid_ctas) == (4, 1, 1, 16, 16, 96)
    with pytest.raises(nat.UnsupportedPlan):
        runtime.explicit_config(g, 6, 8, 128, 128, "l2dsm")  # 192 CTAs in clusters of 8: not co-resident
    with pytest.raises(nat.UnsupportedPlan):
        runtime.explicit_config(g, 5, 2, 128, 128, "l2")  # 5 x 128 columns do not tile l = 768
    rc = runtime.reproducible_configs(g)
    assert rc and all(runtime.is_deterministic(g, c) and c.grid_ctas <= 148 for c in rc)
    assert any((c.ring, c.n_splits, c.nb, c.lb) == (6, 4, 128, 128) for c in rc)
