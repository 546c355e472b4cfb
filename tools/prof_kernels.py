"""Representative single launches for ncu --set full (one flush SYRK at m ~ n/2, one panel)."""
import sys
import torch
sys.path.insert(0, '.')
import paper_1812_02056_b200 as sf
m, k = (int(sys.argv[1]) if len(sys.argv) > 1 else 8192), 512
R = torch.randn(k, m, device='cuda', dtype=torch.float64)   # column-major m x k
C = torch.randn(m, m, device='cuda', dtype=torch.float64)
for _ in range(2):
    assert sf.lib().sf_syrk_sub(m, k, 0, R.data_ptr(), m, C.data_ptr(), m, None) == 0
P = torch.randn(64, 8192, device='cuda', dtype=torch.float64)  # m=8192 x w=64 column-major
P[:, :64] = torch.eye(64, device='cuda', dtype=torch.float64) * 100
P.T[:64, :64] += torch.eye(64, device='cuda', dtype=torch.float64) * 100
info = torch.zeros(1, dtype=torch.int64, device='cuda')
for _ in range(2):
    assert sf.lib().sf_chol_panel(8192, 64, 0, P.data_ptr(), 8192, 0, info.data_ptr(), None) == 0
torch.cuda.synchronize()
print("ok")
