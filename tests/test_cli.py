"""CLI front door (reference cli.py:110-296 subcommands and exit codes): the
planning commands on CPU, `simulate` / `run` on the GPU."""

import json

import pytest

from paper_2512_12949_b200 import cli


def _run(capsys, argv):
    rc = cli.main(argv)
    out = capsys.readouterr().out
    return rc, (json.loads(out) if out.strip() else None)


def test_list_presets_matches_the_reference_catalog(capsys):
    rc, doc = _run(capsys, ["list-presets"])
    assert rc == 0
    ids = [r["id"] for r in doc["presets"]]
    assert ids[:3] == ["G1", "G2", "G3"] and "S8" in ids and "C8" in ids and len(ids) == 26


def test_search_analyze_roundtrip_and_determinism(capsys, tmp_path):
    out = tmp_path / "top.json"
    argv = ["search", "--dims", "128,512,128,256", "--activation", "relu", "--device", "b200",
            "--no-simulator-refine", "--top-k", "3", "--out", str(out)]
    assert cli.main(argv) == 0
    first = out.read_text()
    assert cli.main(argv) == 0
    assert out.read_text() == first  # byte-identical JSON for identical invocations
    doc = json.loads(first)
    assert len(doc["top"]) == 3
    rc, rep = _run(capsys, ["analyze", "--dims", "128,512,128,256", "--activation", "relu", "--device", "b200",
                            "--plan", f"{out}#0"])
    assert rc == 0 and rep["report"]["volume_bytes"]["global"] > 0


def test_count_space_and_exit_codes(capsys):
    rc, doc = _run(capsys, ["count-space", "--preset", "G1", "--rules", "0,5"])
    assert rc == 0 and [s["stage"] for s in doc["stages"]] == ["initial", "rule5"]
    assert cli.main(["search", "--preset", "G1", "--dims", "1,2,3,4"]) == 2      # usage error
    assert cli.main(["search", "--preset", "NOPE"]) == 1                         # UnknownPreset
    capsys.readouterr()


@pytest.mark.gpu
def test_simulate_runs_the_fused_kernel_and_verifies(capsys, tmp_path):
    out = tmp_path / "top.json"
    assert cli.main(["search", "--dims", "256,1024,256,512", "--activation", "relu", "--device", "b200",
                     "--no-simulator-refine", "--top-k", "2", "--out", str(out)]) == 0
    rc, doc = _run(capsys, ["simulate", "--dims", "256,1024,256,512", "--activation", "relu", "--device", "b200",
                            "--plan", f"{out}#0", "--check-traffic", "--compare-baseline"])
    assert rc == 0, doc
    assert doc["verify"]["numerics_pass"] and doc["verify"]["parity_pass"]
    assert doc["verify"]["max_rel_error"] <= 1e-2
    rc, doc = _run(capsys, ["run", "--dims", "512,8192,2048,2048", "--gated", "--iters", "5"])
    assert rc == 0 and doc["tflops"] > 100 and doc["exchange"] in ("pair", "l2", "dsm")
    rc, doc = _run(capsys, ["run", "--dims", "512,3072,768,768", "--activation", "gelu", "--exchange", "l2dsm",
                            "--deterministic", "--iters", "5"])
    assert rc == 0 and doc["bit_reproducible"] and doc["exchange"] == "l2dsm"


def test_export_dot_plan_and_launch(capsys, tmp_path):
    out = tmp_path / "top.json"
    assert cli.main(["search", "--dims", "256,1024,256,512", "--activation", "relu", "--device", "b200",
                     "--no-simulator-refine", "--top-k", "1", "--out", str(out)]) == 0
    capsys.readouterr()
    assert cli.main(["export-dot", "--dims", "256,1024,256,512", "--activation", "relu", "--plan", f"{out}#0"]) == 0
    dot = capsys.readouterr().out
    assert dot.startswith("digraph") and dot.rstrip().endswith("}") and dot.count("{") == dot.count("}")
    assert "cta_0_0_0" in dot and "->" in dot
    assert cli.main(["export-dot", "--dims", "512,8192,2048,2048", "--gated", "--launch", "pair"]) == 0
    dot = capsys.readouterr().out
    assert "CTA pair 0" in dot and "split-N reduce" in dot
    assert cli.main(["export-dot", "--dims", "512,8192,2048,2048", "--gated"]) == 2  # needs --plan or --launch


def test_export_tilegraph_cluster_structure():
    from paper_2512_12949_b200 import tilegraph, workload as W
    from paper_2512_12949_b200.plan import make_plan

    g = W.build_gated_ffn(W.DimensionSpec(512, 8192, 2048, 2048))
    p = make_plan("n", "klm", (64, 1024, 2048, 512), (1, 8, 2, 4), "spatial_split")
    dot = tilegraph.export_tilegraph(g, p)
    assert dot.count("[label=\"CTA (") == 16                       # cls_m * cls_n * cls_k
    assert dot.count("all_exchange Mul") == 8 * 2                 # the two branch CTAs of each (im, in)
    assert dot.count("shuffle") == 2 * 8                          # cls_shuffle = 2: rings of 2 per (ik, set)
