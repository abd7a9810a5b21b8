"""Measure FP64 GEMM throughput (cuBLAS DGEMM via torch) -- the FP64 roofline denominator."""
import json, torch
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3): c = a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
x = torch.empty(2**30 // 8, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
for _ in range(3): y.copy_(x)
torch.cuda.synchronize(); bc = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); y.copy_(x); e1.record(); torch.cuda.synchronize(); bc = min(bc, e0.elapsed_time(e1))
print(json.dumps({"dgemm_tflops": 2 * n**3 / (best * 1e-3) / 1e12, "dgemm_ms": best, "n": n,
                  "copy_f64_gbs": 2 * 2**30 / (bc * 1e-3) / 1e9,
                  "l2_bytes": torch.cuda.get_device_properties(0).L2_cache_size,
                  "sms": torch.cuda.get_device_properties(0).multi_processor_count}))
