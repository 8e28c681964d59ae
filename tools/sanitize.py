"""Small fused chains for compute-sanitizer (racecheck / synccheck / memcheck) on the
GPU box: every transport (DSM ring, L2 ring, CTA pair, weight-multicast quad),
standard and gated, single and split N, each checked against the CPU oracle.

    compute-sanitizer --tool racecheck python tools/sanitize.py > profiles/r02/sanitizer_racecheck.log
"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (checker only)
from paper_2512_12949_b200 import _native as nat, runtime  # noqa: E402
from paper_2512_12949_b200 import dispatch  # noqa: E402
from paper_2512_12949_b200 import workload as W  # noqa: E402

CASES = [  # (kind, m, n, k, l, explicit CTA-pair config or None = auto lowering per transport)
    ("standard_ffn", 256, 2048, 512, 512, None),
    ("gated_ffn", 256, 1024, 512, 512, None),
    ("standard_ffn", 512, 1024, 256, 512, None),
    # ragged pair ring whose last split has members without a chunk (E/C swap, empty drains)
    ("standard_ffn", 17, 3328, 512, 512, None),
    # whole n-steps (non-ragged pair kernels; quads with an even m-tile count), split-N
    # reduce-scatter tail and the C-scratch discard
    ("standard_ffn", 512, 2048, 512, 512, dict(ring=2, n_splits=4, nb=256, lb=256, exchange=2)),
    ("gated_ffn", 512, 2048, 512, 512, dict(ring=2, n_splits=8, nb=128, lb=256, exchange=2)),
    ("standard_ffn", 2048, 2048, 256, 512, dict(ring=2, n_splits=1, nb=256, lb=256, exchange=2)),
    # DSM reduce-scatter of the split-N partials (FF_XCHG_L2_DSMR): split clusters of 2 / 4 / 8
    ("standard_ffn", 256, 2048, 256, 512, dict(ring=2, n_splits=4, nb=128, lb=256, exchange=3)),
    ("gated_ffn", 256, 1024, 256, 512, dict(ring=2, n_splits=8, nb=64, lb=256, exchange=3)),
    ("standard_ffn", 200, 1024, 256, 256, dict(ring=1, n_splits=2, nb=128, lb=256, exchange=3)),
]


def main():
    lib = nat.load()
    bad = 0
    for kind, m, n, k, l, fixed in CASES:
        dims = W.DimensionSpec(m, n, k, l, 2)
        graph = W.build_gated_ffn(dims) if kind == "gated_ffn" else W.build_standard_ffn(dims, "relu")
        host = {a: oracle.round_bf16(v) for a, v in oracle.make_inputs(kind, m, n, k, l, seed=11).items()}
        dev = {a: torch.from_numpy(v).cuda().to(torch.bfloat16) for a, v in host.items()}
        ref = oracle.dense_chain(kind, graph.activation, host, bf16_intermediate=True)
        if fixed:
            runs = (("pair", 2), ("pair", 4)) if fixed["exchange"] == 2 else (("l2dsm", 0),)
        else:
            runs = (("dsm", 0), ("l2", 0), ("pair", 2), ("pair", 4))
        for exchange, variant in runs:
            lib.ff_set_variant(variant)
            try:
                cfg = dispatch.config_from_dict(fixed) if fixed else runtime.lower(graph, None, None, exchange)
                out = runtime.launch(graph, cfg, dev)
                torch.cuda.synchronize()
                err = oracle.max_relative_error(out.float().cpu().numpy(), ref)
            except Exception as exc:  # report and go on
                print(f"{kind} {(m, n, k, l)} [{exchange} v{variant}] ERROR {exc!r}", flush=True)
                bad += 1
                continue
            ok = np.isfinite(err) and err <= 1e-2
            bad += not ok
            print(f"{kind} {(m, n, k, l)} [{exchange} v{variant}] {cfg.as_dict()} max_rel_err={err:.2e} "
                  f"{'ok' if ok else 'FAIL'}", flush=True)
    lib.ff_set_variant(0)
    print("sanitize cases done, failures:", bad)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
