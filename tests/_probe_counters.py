# Diagnostics: per-role wait-cycle counters of the pair kernel's members (cold L2, one launch).
import sys, ctypes, torch
sys.path.insert(0, '.')
ARGV = list(sys.argv)
sys.argv = sys.argv[:1] + ['x']
exec(open('tests/_probe_kernel.py').read().split("for pack in")[0])
ST = 32
flush_buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device='cuda')
names = ["prod_total","prod_w_empty","prod_w_flag","mma_total","mma_w_full_g0","mma_w_full_hop","mma_w_cempty","mma_w_ownfull","mma_w_eempty",
         "epi_total","epi_w_cfull","epi_w_ownfree","epi_drainC","epi_store","epi_E"]
SHAPES = {"llama": (512,8192,2048,2048,2,True), "gpt67b": (512,16384,4096,4096,1,False)}
for name in [a for a in ARGV[1:] if a in SHAPES] or list(SHAPES):
    A,B,B1,D,E,ch,kc,ws,t = setup(*SHAPES[name],None,2)
    f=lambda: nat.check(lib.ff_chain_launch(ctypes.byref(ch),ctypes.byref(kc),ctypes.byref(t),ws.data_ptr(),ws.numel(),None))
    buf = torch.zeros(kc.grid_ctas*ST + 64, dtype=torch.int64, device='cuda')
    for _ in range(3): f()
    flush_buf.add_(1.0); torch.cuda.synchronize()
    lib.ff_set_profile_buffer(ctypes.c_void_p(buf.data_ptr())); f(); lib.ff_set_profile_buffer(None)
    torch.cuda.synchronize()
    v = buf[:kc.grid_ctas*ST].view(kc.grid_ctas, ST)[:, :16].double() / 1.965e3
    lead = v[0::2]
    print(f"== {name} {kc.as_dict()}")
    for i, nm in enumerate(names):
        col = (lead if nm.startswith("mma") else v)[:, i]
        print(f"   {nm:16s} mean {col.mean().item():8.1f}us  max {col.max().item():8.1f}us")
