"""One cuBLAS DGEMM (torch.matmul fp64, 8192^3) for ncu comparison with gemm_f64_kernel."""
import torch
a = torch.randn(8192, 8192, device='cuda', dtype=torch.float64)
b = torch.randn(8192, 512, device='cuda', dtype=torch.float64)
c = torch.randn(8192, 8192, device='cuda', dtype=torch.float64)
for _ in range(2):
    c.addmm_(b, b.T, alpha=-1.0)
torch.cuda.synchronize()
print("ok")
