"""LU panel building block sf_lu_panel at cfg2-like sizes, for ncu kernel durations."""
import sys, torch
sys.path.insert(0, '.')
import paper_1812_02056_b200 as sf
info = torch.zeros(1, dtype=torch.int64, device='cuda')
for m, w in ((4096, 32), (4096, 64), (2048, 64)):
    n = m
    A = torch.rand(n, n, device='cuda', dtype=torch.float64) * 2 - 1
    A += torch.eye(n, device='cuda', dtype=torch.float64) * n
    for _ in range(2):
        assert sf.lib().sf_lu_panel(m, w, n - w, 0, A.data_ptr(), n, 0, 1e-300, info.data_ptr(), None) == 0
torch.cuda.synchronize()
