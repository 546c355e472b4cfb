"""One leaf-sized panel (w = 32) per m, for ncu kernel durations."""
import sys, torch
sys.path.insert(0, '.')
import paper_1812_02056_b200 as sf
info = torch.zeros(1, dtype=torch.int64, device='cuda')
for m in (2000, 16384, 65536):
    w = 32
    P = torch.randn(w, m, device='cuda', dtype=torch.float64) * 0.01
    P.T[:w, :w] += torch.eye(w, device='cuda', dtype=torch.float64) * 4
    assert sf.lib().sf_chol_panel(m, w, 0, P.data_ptr(), m, 0, info.data_ptr(), None) == 0
torch.cuda.synchronize()
