"""Compare a tail-split launch with the no-tail-split variant row block by row block (diagnostics)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2512_12949_b200 import _native as nat
    from paper_2512_12949_b200 import runtime
    from paper_2512_12949_b200 import workload as W

    m = int(sys.argv[1]) * 256 if len(sys.argv) > 1 else 11 * 256
    n, k, l = 8192, 512, 2048
    g = W.build_standard_ffn(W.DimensionSpec(m, n, k, l), "relu")
    torch.manual_seed(0)
    dev = {"A": (torch.rand(m, k, device="cuda") * 2 - 1).bfloat16(),
           "B": ((torch.rand(k, n, device="cuda") * 2 - 1) / 8).bfloat16(),
           "D": ((torch.rand(n, l, device="cuda") * 2 - 1) / 16).bfloat16()}
    lib = nat.load()
    runtime._workspace(1 << 30, torch.device("cuda", 0), torch.cuda.current_stream())
    outs = {}
    for v in (0x800, 0x0):
        lib.ff_set_variant(v)
        cfg = runtime.lower(g, None, 148, "pair")
        outs[v] = runtime.launch(g, cfg, dev).float().clone()
        torch.cuda.synchronize()
        print(hex(v), cfg.as_dict())
    lib.ff_set_variant(0)
    cref = torch.relu(dev["A"].float() @ dev["B"].float())
    ref = (cref.bfloat16().float() @ dev["D"].float())
    # the intermediate as the tail-split launch materialises it (c_debug dump): which columns are wrong
    cdbg = torch.zeros((m, n), dtype=torch.bfloat16, device="cuda")
    cfg = runtime.lower(g, None, 148, "pair")
    runtime.launch(g, cfg, dev, c_debug=cdbg)
    torch.cuda.synchronize()
    cerr = (cdbg.float() - cref).abs()
    print("C max err", cerr.max().item(), "C ref max", cref.abs().max().item())
    for mt in range(m // 256):
        blk = cerr[mt * 256:(mt + 1) * 256]
        bad = [c for c in range(0, n, 256) if blk[:, c:c + 256].max().item() > 0.05 * cref.abs().max().item()]
        if bad:
            print(f"   C m tile {mt}: wrong 256-col chunks {[c // 256 for c in bad]}")
    if os.environ.get("FF_CHAIN_LIB", "").endswith("libff_ab_tail3.so"):
        # FF_AB_TAIL=3 build: tail E rows hold only the own split's partial -- compare per split
        St = 4
        o = outs[0x0]
        for mt in range(9, m // 256):
            for half in range(2):
                r0 = mt * 256 + half * 128
                R = 128 // St
                for sp in range(St):
                    rows = slice(r0 + sp * R, r0 + (sp + 1) * R)
                    cols = slice(sp * (n // St), (sp + 1) * (n // St))
                    part = cref[rows, cols].bfloat16().float() @ dev["D"].float()[cols]
                    e = (o[rows] - part).abs().max().item()
                    print(f"   tail m tile {mt} half {half} split {sp}: |E_rows - partial_sp| max {e:.3f} "
                          f"(partial max {part.abs().max().item():.2f})")
    for v, o in outs.items():
        err = (o - ref).abs()
        print(hex(v), "max err", err.max().item(), "ref max", ref.abs().max().item())
        for mt in range(m // 256):
            for half in range(2):
                r0 = mt * 256 + half * 128
                blk = err[r0:r0 + 128]
                cols = [blk[:, c:c + 256].max().item() for c in range(0, l, 256)]
                if max(cols) > 1e-2 * ref.abs().max().item():
                    print(f"   m tile {mt} half {half}: col-slice max err " + " ".join(f"{x:.2f}" for x in cols))


if __name__ == "__main__":
    main()
