import sys, torch, ctypes
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import test_gpu_chain as T
from paper_2512_12949_b200 import runtime, _native as nat
lib = nat.load()
for case, x, dbg in [(("gated_ffn", "silu", 128, 3328, 256, 1792), "pair", 0), (("gated_ffn", "silu", 128, 3328, 256, 1792), "pair", 64),
                     (("standard_ffn", "relu", 128, 3328, 256, 1792), "pair", 0), (("gated_ffn", "silu", 256, 3328, 256, 1792), "pair", 0),
                     (("gated_ffn", "silu", 128, 3328, 256, 512), "pair", 0), (("gated_ffn", "silu", 128, 1024, 256, 512), "pair", 0)]:
    runtime._workspaces.clear()
    lib.ff_set_debug_mode(dbg)
    g = T._graph(*case)
    cfg = runtime.lower(g, None, 148, x)
    host, dev = T._inputs(case[0], *case[2:], seed=3)
    out = runtime.launch(g, cfg, dev)
    torch.cuda.synchronize()
    ws = list(runtime._workspaces.values())[0]
    zone = ws[(1 << 20) + (256 << 10):(1 << 20) + (256 << 10) + (32 << 20)].view(torch.float32)
    cnt = ws[(1 << 20):(1 << 20) + (256 << 10)].view(torch.int32)
    print(case, x, dbg, cfg.as_dict(), "zone nonzero", int((zone != 0).sum()), "cnt", int((cnt != 0).sum()), flush=True)
lib.ff_set_debug_mode(0)
