import torch, sys
torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = True
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for (m, n, k) in [(32768, 8192, 4096), (32768, 256, 8192), (32768, 2048, 8192), (32768, 8192, 128)]:
    a = torch.randn(m, k, device="cuda").bfloat16(); b = torch.randn(k, n, device="cuda").bfloat16()
    for _ in range(3): c = a @ b
    ts = []
    for _ in range(10):
        flush.add_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[5]
    print(f"cublas {m}x{n}x{k}: {ms*1e3:.1f} us {2*m*n*k/ms/1e9:.0f} TF/s", flush=True)
