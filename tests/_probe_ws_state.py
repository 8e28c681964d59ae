# Diagnostics: zero-invariant workspace regions (split counters, fp32 E zone) after each launch.
import sys, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import test_gpu_chain as T
from paper_2512_12949_b200 import runtime, _native as nat
cases = T.CASES + T._random_cases(10, 2025)
for case in cases:
    for x in ("dsm", "l2", "pair"):
        g = T._graph(*case)
        try:
            cfg = runtime.lower(g, None, 148, x)
        except nat.UnsupportedPlan:
            continue
        host, dev = T._inputs(case[0], *case[2:], seed=3)
        out = runtime.launch(g, cfg, dev)
        torch.cuda.synchronize()
        import oracle
        err = oracle.max_relative_error(out.float().cpu().numpy(), oracle.dense_chain(case[0], case[1], host, True))
        ws = list(runtime._workspaces.values())[0]
        cnt = ws[(1 << 20):(1 << 20) + (256 << 10)].view(torch.int32)
        zone = ws[(1 << 20) + (256 << 10):(1 << 20) + (256 << 10) + (32 << 20)].view(torch.float32)
        nzc, nzz = int((cnt != 0).sum()), int((zone != 0).sum())
        flag = "  <-- DIRTY" if nzc or nzz else ""
        print(f"{case} {x} {cfg.as_dict()['ring']},{cfg.n_splits},{cfg.nb},{cfg.lb} err {err:.1e} counters {nzc} zone {nzz}{flag}", flush=True)
