"""Measure FP64 (DGEMM via cuBLAS) and HBM copy on the GPU box; complements tools/fp64_peak."""
import json, torch
torch.cuda.init()
res = {}
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
    for _ in range(3): a @ b
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); a @ b; e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
    res[f"dgemm_{n}_tflops"] = 2 * n**3 / best / 1e9
x = torch.empty(2**30, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
best = 1e9
for _ in range(6):
    e0.record(); y.copy_(x); e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
res["copy_gbs"] = 2 * x.numel() * 8 / best / 1e6
print(json.dumps(res))
