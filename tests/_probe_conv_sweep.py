# Diagnostics: cold-L2 event time of conv-chain configs (ring, n_splits, nb, lb, exchange).
import sys, torch
sys.path.insert(0, '.')
from paper_2512_12949_b200 import runtime, workload as W, _native as nat
flush_buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device='cuda')
def run(cfg, shape, kc):
    ic, h, w, oc1, oc2, k1, k2 = shape
    g = torch.Generator(device="cpu").manual_seed(1)
    x = (torch.rand(1, h, w, ic, generator=g) * 2 - 1).to(torch.bfloat16).cuda()
    w1 = ((torch.rand(k1, k1, ic, oc1, generator=g) * 2 - 1) / (k1 * k1 * ic) ** 0.5).to(torch.bfloat16).cuda()
    w2s = (oc1, oc2) if k2 == 1 else (k2, k2, oc1, oc2)
    w2 = ((torch.rand(*w2s, generator=g) * 2 - 1) / (k2 * k2 * oc1) ** 0.5).to(torch.bfloat16).cuda()
    y = torch.empty(1, h, w, oc2, dtype=torch.bfloat16, device="cuda")
    f = lambda: runtime.launch_conv(cfg, kc, x, w1, w2, out=y)
    for _ in range(3): f()
    ts = []
    for _ in range(15):
        flush_buf.add_(1.0)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
    return sorted(ts)[7]
shape = (64, 56, 56, 64, 256, 3, 1)
cfg = W.ConvChainConfig(*shape)
for (ring, S, nb, lb, x) in [(1,1,64,256,1),(1,1,64,256,0),(2,1,64,128,1),(2,1,64,128,0),(4,1,64,64,0),(4,1,64,64,1),(1,1,64,128,1),(1,1,64,64,1)]:
    kc = nat.KernelConfig(); kc.ring, kc.n_splits, kc.nb, kc.lb, kc.exchange = ring, S, nb, lb, x
    try:
        print(f"C5 ring {ring} S {S} nb {nb} lb {lb} x{x}: {run(cfg, shape, kc):.1f} us", flush=True)
    except Exception as e:
        print(f"C5 ring {ring} S {S} nb {nb} lb {lb} x{x}: {repr(e)[:80]}", flush=True)
