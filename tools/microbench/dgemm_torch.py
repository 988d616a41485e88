"""cuBLAS DGEMM (torch.matmul fp64) and HBM copy reference numbers on this B200."""
import json, torch
torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda:0")
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(2):
        c = a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(json.dumps({"test": "cublas_dgemm", "n": n, "ms": best, "tflops": 2 * n**3 / best / 1e9}))
x = torch.empty(2**30 // 8 * 8, dtype=torch.float64, device=dev)  # 8 GiB
y = torch.empty_like(x)
y.copy_(x); torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); y.copy_(x); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(json.dumps({"test": "hbm_copy_fp64", "bytes": 2 * x.numel() * 8, "ms": best, "gbs": 2 * x.numel() * 8 / best / 1e6}))
