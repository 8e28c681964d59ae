"""Per-CTA phase timeline of a fused-chain launch (diagnostics, GPU box only).

    python tools/timeline.py [gpt67b|llama|opt|gpt2s|conv_c5|conv_1x1_3x3 ...] [x0|x1] [warm] [rings] [variant=0x..] [cfg=r,S,nb,lb,x,..]

Every CTA stamps %globaltimer at fixed points (slots 16..31 of the profile
buffer, ff_set_profile_buffer); this prints min / mean / max per stamp relative
to the first CTA's entry, for the median of 5 launches on a cold L2 (flushed
before each launch, as bench.py does).  x0 / x1 select the 1-CTA DSM / L2
kernels (default: the CTA-pair kernel)."""

import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_12949_b200 import _native as nat  # noqa: E402

ST = 32
NAMES = {0: 'entry', 1: 'setup', 2: 'cfull0', 3: 'drained0', 4: 'stored0', 5: 'cfull1', 6: 'E_summed',
         7: 'drained1', 8: 'E_staged', 9: 'E_slabs_out', 10: 'E_finished', 11: 'E_flags_in', 12: 'E_loaded',
         13: 'E_sum0', 14: 'E_start', 15: 'exit'}
COUNTERS = ['prod_total', 'prod_w_empty', 'prod_w_flag', 'mma_total', 'mma_w_full_g0', 'mma_w_full_hop',
            'mma_w_cempty', 'mma_w_own', 'mma_w_eempty', 'epi_total', 'epi_w_cfull', 'epi_w_ofree', 'epi_drainC',
            'epi_store', 'epi_E']
SHAPES = {"llama": (512, 8192, 2048, 2048, 2, True), "gpt67b": (512, 16384, 4096, 4096, 1, False),
          "opt": (4096, 8192, 2048, 2048, 1, False), "gpt2s": (512, 3072, 768, 768, 3, False),
          "opt32k": (32768, 8192, 2048, 2048, 1, False),
          # phase probes: GEMM0-dominated (one ring member, L = 256) and hop-dominated (K = 128)
          "g0only": (32768, 8192, 4096, 256, 1, False), "hopsonly": (32768, 8192, 128, 2048, 1, False)}


def setup(m, n, k, l, act, gated, xchg, lib):
    a = (torch.rand(m, k, device='cuda') * 2 - 1).bfloat16()
    if gated:
        b01 = (torch.rand(2, k, n, device='cuda') * 2 - 1).bfloat16()
        b, b1 = b01[0], b01[1]
    else:
        b = (torch.rand(k, n, device='cuda') * 2 - 1).bfloat16()
        b1 = b
    d = (torch.rand(n, l, device='cuda') * 2 - 1).bfloat16()
    e = torch.zeros(m, l, device='cuda', dtype=torch.bfloat16)
    ch = nat.ChainDesc(1 if gated else 0, 2 if gated else act, m, n, k, l, 2, 0)
    kc = nat.KernelConfig()
    nat.check(lib.ff_auto_config_ex(ctypes.byref(ch), 148, xchg, ctypes.byref(kc)))
    ws = torch.zeros(lib.ff_chain_workspace_bytes(ctypes.byref(ch), ctypes.byref(kc)) or 256, device='cuda',
                     dtype=torch.uint8)
    t = nat.Tensors(a.data_ptr(), b.data_ptr(), b1.data_ptr(), d.data_ptr(), e.data_ptr())
    return (a, b, b1, d, e, ws), ch, kc, t


CONVS = {"conv_c5": (64, 56, 56, 64, 256, 3, 1), "conv_1x1_3x3": (256, 56, 56, 64, 64, 1, 3)}


def setup_conv(shape, xchg, lib):
    """A conv chain (bench.py's CONV_WORKLOADS shapes) launched through ff_conv_chain_launch."""
    from paper_2512_12949_b200 import runtime, workload as W
    ic, h, w, oc1, oc2, k1, k2 = shape
    cfg = W.ConvChainConfig(*shape) if k2 == 1 else W.ConvBlockConfig(*shape)
    x = (torch.rand(1, h, w, ic, device='cuda') * 2 - 1).bfloat16()
    w1 = ((torch.rand(k1, k1, ic, oc1, device='cuda') * 2 - 1) / (k1 * k1 * ic) ** 0.5).bfloat16()
    w2 = ((torch.rand(*((oc1, oc2) if k2 == 1 else (k2, k2, oc1, oc2)), device='cuda') * 2 - 1) /
          (k2 * k2 * oc1) ** 0.5).bfloat16()
    y = torch.empty(1, h, w, oc2, dtype=torch.bfloat16, device='cuda')
    kc = runtime.lower_conv(cfg, 1, "dsm" if xchg == 0 else "l2")
    cd = runtime.conv_desc(cfg, 1)
    ws = torch.zeros(lib.ff_conv_chain_workspace_bytes(ctypes.byref(cd), ctypes.byref(kc)) or 256,
                     device='cuda', dtype=torch.uint8)
    t = nat.Tensors(x.data_ptr(), w1.data_ptr(), None, w2.data_ptr(), y.data_ptr())
    return (x, w1, w2, y, ws), cd, kc, t


def main(argv):
    lib = nat.load()
    flush_buf = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device='cuda')
    sink = torch.empty((), dtype=torch.float32, device='cuda')
    sel = [a for a in argv if a in SHAPES or a in CONVS] or ["gpt67b", "llama"]
    variant = next((int(a.split("=")[1], 0) for a in argv if a.startswith("variant=")), 0)
    lib.ff_set_variant(variant)
    xchg = 0 if 'x0' in argv else (1 if 'x1' in argv else (3 if 'x3' in argv else 2))
    for name in sel:
        conv = name in CONVS
        keep, ch, kc, t = setup_conv(CONVS[name], xchg, lib) if conv else setup(*SHAPES[name], xchg, lib)
        ws = keep[-1]
        cfg = next((a.split("=")[1] for a in argv if a.startswith("cfg=")), None)
        if cfg:  # an explicit launch (all eleven ffKernelConfig fields, e.g. bench.py's "launch")
            for (fname, _), val in zip(nat.KernelConfig._fields_, cfg.split(",")):
                setattr(kc, fname, int(val))
            ws = torch.zeros(lib.ff_chain_workspace_bytes(ctypes.byref(ch), ctypes.byref(kc)) or 256, device='cuda',
                             dtype=torch.uint8)
            keep = keep + (ws,)

        def f():
            if conv:
                return nat.check(lib.ff_conv_chain_launch(ctypes.byref(ch), ctypes.byref(kc), ctypes.byref(t),
                                                          ws.data_ptr(), ws.numel(), None))
            nat.check(lib.ff_chain_launch(ctypes.byref(ch), ctypes.byref(kc), ctypes.byref(t), ws.data_ptr(),
                                          ws.numel(), None))
        extra = 64  # CTAs past kc.grid_ctas (GEMM0 helper pairs) stamp rows of their own
        buf = torch.zeros((kc.grid_ctas + extra) * ST + 64, dtype=torch.int64, device='cuda')
        for _ in range(3):
            f()
        runs = []
        for _ in range(5):
            if 'rflush' in argv:  # read-only flush: leaves clean lines (no dirty evictions afterwards)
                torch.sum(flush_buf, dim=0, out=sink)
            elif 'warm' not in argv:
                flush_buf.add_(1.0)
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            buf.zero_()
            lib.ff_set_profile_buffer(ctypes.c_void_p(buf.data_ptr()))
            ea.record()
            f()
            eb.record()
            lib.ff_set_profile_buffer(None)
            torch.cuda.synchronize()
            w = buf[:kc.grid_ctas * ST].view(kc.grid_ctas, ST).double()
            wx = buf[kc.grid_ctas * ST:(kc.grid_ctas + extra) * ST].view(extra, ST).double()
            runs.append((ea.elapsed_time(eb) * 1e3, w[:, 16:].clone(), w[:, :16].clone(), wx[:, 16:].clone()))
        runs.sort(key=lambda r: r[0])
        us, v, cnt, vx = runs[2]
        t_zero = v[v[:, 0] > 0][:, 0].min()
        vx = vx[vx[:, 0] > 0]
        if vx.numel():  # helper pairs: entry, setup, then one stamp per published chunk
            relx = (vx - t_zero) / 1e3
            relx[vx == 0] = float('nan')
            print(f"   helper CTAs {vx.shape[0]}: chunk publish times (mean over helper CTAs, us):",
                  " ".join(f"{relx[:, i][~torch.isnan(relx[:, i])].mean().item():6.1f}"
                           for i in range(2, 14) if (~torch.isnan(relx[:, i])).any()))
        valid = v[:, 0] > 0
        v = v[valid]
        rel = (v - v[:, 0].min()) / 1e3
        rel[v == 0] = float('nan')
        print(f"== {name} variant {variant:#x} {kc.as_dict()}: events {us:.1f} us, active CTAs {int(valid.sum())}")
        for i in range(16):
            col = rel[:, i]
            col = col[~torch.isnan(col)]
            if col.numel():
                print(f"   {NAMES[i]:11s} min {col.min().item():7.1f} mean {col.mean().item():7.1f} "
                      f"max {col.max().item():7.1f} us")
        if 'res' in argv:  # globaltimer resolution: distinct raw values of the entry and exit stamps
            for i in (0, 10, 15):
                raw = v[:, i][v[:, i] > 0].long()
                u = torch.unique(raw)
                d = (u[1:] - u[:-1]) if u.numel() > 1 else u
                print(f"   stamp {NAMES[i]}: {u.numel()} distinct of {raw.numel()}, min step {int(d.min())} ns, "
                      f"values mod 1000: {sorted(set((raw % 1000).tolist()))[:8]}")
        if 'counters' in argv:  # per-role wait counters (clock64 cycles, FF_TIMED): mean / max over CTAs
            live = cnt[valid]
            for i, nm in enumerate(COUNTERS):
                col = live[:, i]
                col = col[col > 0]
                if col.numel():
                    print(f"   {nm:15s} mean {col.mean().item() / 1e3:9.1f} max {col.max().item() / 1e3:9.1f} kcyc")
        if 'members' in argv:  # last-MMA time (E_start) per ring member pair, to see systematic skew
            g2 = kc.ring * 2
            es = rel[:, 14]
            for r in range(kc.rings):
                vals = [es[r * g2 + 2 * p_: r * g2 + 2 * p_ + 2].mean().item() for p_ in range(kc.ring)]
                print(f"   ring {r} E_start per member: " + " ".join(f"{x:5.1f}" for x in vals))
        if 'rings' in argv:
            g2 = kc.ring * 2
            for r in range(kc.rings):
                blk = rel[r * g2:(r + 1) * g2]
                cols = {k: blk[:, i] for i, k in ((2, 'cfull0'), (5, 'cfull1'), (14, 'E_start'), (15, 'exit'))}
                print("   ring %d: " % r + " ".join(
                    f"{k} {c[~torch.isnan(c)].mean().item():6.1f}/{c[~torch.isnan(c)].max().item():6.1f}"
                    for k, c in cols.items()))


if __name__ == "__main__":
    main(sys.argv[1:])
    nat.load().ff_set_variant(0)
