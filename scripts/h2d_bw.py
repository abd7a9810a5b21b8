import torch, time
n = 8000
h = torch.empty((n, n), dtype=torch.float64, pin_memory=True).fill_(1.0)
d = torch.empty((n, n), dtype=torch.float64, device="cuda")
for rows in (1024, 8000):
    for _ in range(3):
        torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); d[:rows].copy_(h[:rows], non_blocking=True); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    print(rows, "rows", f"{ms:.3f} ms", f"{rows * n * 8 / ms / 1e6:.1f} GB/s")
