# Diagnostics: per-CTA globaltimer timeline of the pair kernel on a COLD L2
# (flush before each launch, as in bench.py); median launch of 5.
import sys, ctypes, torch
sys.path.insert(0, '.')
ARGV = list(sys.argv)
sys.argv = sys.argv[:1] + ['x']
exec(open('tests/_probe_kernel.py').read().split("for pack in")[0])
ST = 32
flush_buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device='cuda')
NAMES = {0:'entry',1:'setup',2:'cfull0',3:'drained0',4:'stored0',5:'cfull1',6:'E_summed',7:'drained1',8:'E_staged',
         9:'E_slabs_out',10:'E_finished',11:'E_flags_in',12:'E_loaded',13:'E_sum0',14:'E_start',15:'exit'}
SHAPES = {"llama": (512,8192,2048,2048,2,True), "gpt67b": (512,16384,4096,4096,1,False),
          "opt": (4096,8192,2048,2048,1,False), "gpt2s": (512,3072,768,768,3,False)}
mode = int(ARGV[1]) if len(ARGV) > 1 and ARGV[1].isdigit() else 0
sel = [a for a in ARGV[1:] if a in SHAPES] or ["gpt67b", "llama"]
for name in sel:
    lib.ff_set_debug_mode(mode)
    XCHG = 0 if 'x0' in ARGV else (1 if 'x1' in ARGV else 2)
    A,B,B1,D,E,ch,kc,ws,t = setup(*SHAPES[name],None,XCHG)
    f=lambda: nat.check(lib.ff_chain_launch(ctypes.byref(ch),ctypes.byref(kc),ctypes.byref(t),ws.data_ptr(),ws.numel(),None))
    buf = torch.zeros(kc.grid_ctas*ST + 64, dtype=torch.int64, device='cuda')
    for _ in range(3): f()
    runs = []
    for it in range(5):
        if 'warm' not in ARGV: flush_buf.add_(1.0)
        ea = torch.cuda.Event(enable_timing=True); eb = torch.cuda.Event(enable_timing=True)
        buf.zero_()
        lib.ff_set_profile_buffer(ctypes.c_void_p(buf.data_ptr())); ea.record(); f(); eb.record(); lib.ff_set_profile_buffer(None)
        torch.cuda.synchronize()
        v = buf[:kc.grid_ctas*ST].view(kc.grid_ctas, ST)[:, 16:].double()
        runs.append((ea.elapsed_time(eb)*1e3, v.clone()))
    runs.sort(key=lambda r: r[0])
    ms, v = runs[2]
    valid = v[:, 0] > 0
    v = v[valid]
    t0 = v[:, 0].min()
    rel = (v - t0) / 1e3
    rel[v == 0] = float('nan')
    print(f"== {name} {kc.as_dict()} dbg {mode}: events {ms:.1f} us, active CTAs {int(valid.sum())}")
    for i in range(16):
        col = rel[:, i]; col = col[~torch.isnan(col)]
        if col.numel() == 0: continue
        print(f"   {NAMES[i]:11s} min {col.min().item():7.1f} mean {col.mean().item():7.1f} max {col.max().item():7.1f} us")
    if 'rings' in ARGV:
        G2 = kc.ring * 2  # CTAs per ring (pairs)
        for r in range(kc.rings):
            blk = rel[r * G2:(r + 1) * G2]
            cols = {k: blk[:, i] for i, k in ((2, 'cfull0'), (5, 'cfull1'), (14, 'E_start'), (15, 'exit'))}
            print("   ring %d: " % r + " ".join(f"{k} {c[~torch.isnan(c)].mean().item():6.1f}/{c[~torch.isnan(c)].max().item():6.1f}" for k, c in cols.items()))
lib.ff_set_debug_mode(0)
# helper segment completion stamps (slots 18.. of the helper CTAs)
if 'helpers' in ARGV:
    for name in sel:
        A,B,B1,D,E,ch,kc,ws,t = setup(*SHAPES[name],None,2)
        if kc.helpers == 0: continue
        f=lambda: nat.check(lib.ff_chain_launch(ctypes.byref(ch),ctypes.byref(kc),ctypes.byref(t),ws.data_ptr(),ws.numel(),None))
        buf = torch.zeros(kc.grid_ctas*ST + 64, dtype=torch.int64, device='cuda')
        for _ in range(3): f()
        if 'warm' not in ARGV: flush_buf.add_(1.0)
        buf.zero_()
        lib.ff_set_profile_buffer(ctypes.c_void_p(buf.data_ptr())); f(); lib.ff_set_profile_buffer(None)
        torch.cuda.synchronize()
        v = buf[:kc.grid_ctas*ST].view(kc.grid_ctas, ST)[:, 16:].double()
        t0 = v[:kc.grid_ctas - 2*kc.helpers, 0].min()
        for hcta in range(kc.grid_ctas - 2*kc.helpers, kc.grid_ctas, 2):
            row = v[hcta]
            segs = [f"{(a - t0).item()/1e3:6.1f}/{(b - t0).item()/1e3:6.1f}" for a, b in zip(row[2:8], row[8:14]) if a > 0]
            print(f"   helper cta {hcta}: entry {(row[0]-t0).item()/1e3:5.1f} segs mma-done/drained {' '.join(segs)}")
            cnt = buf[:kc.grid_ctas*ST].view(kc.grid_ctas, ST)[hcta, :16].double() / 1.965e3
            print(f"      prod total {cnt[0]:.1f} w_empty {cnt[1]:.1f} w_flag {cnt[2]:.1f} | mma total {cnt[3]:.1f} w_full {cnt[4]:.1f} w_buf {cnt[8]:.1f} us")
