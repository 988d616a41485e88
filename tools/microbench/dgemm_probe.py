"""One cuBLAS DGEMM (torch.matmul fp64, 8192^3) inside a profiler range, for ncu --profile-from-start off."""
import torch
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()
torch.cuda.profiler.start()
c = a @ b
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
