"""cuBLAS DGEMM reference peak (torch.matmul float64) on the box; one JSON line per shape."""
import json
import torch

dev = torch.device("cuda:0")
for n in (2048, 4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(5):
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(json.dumps({"what": "cublas_dgemm", "n": n, "ms": best, "tflops": 2 * n**3 / best / 1e9}))
x = torch.empty(2**30 // 8, dtype=torch.float64, device=dev)
y = torch.empty_like(x)
for _ in range(3):
    y.copy_(x)
torch.cuda.synchronize()
best = 1e30
for _ in range(10):
    e0.record(); y.copy_(x); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(json.dumps({"what": "copy", "gbs": 2 * 2**30 / best / 1e6}))
