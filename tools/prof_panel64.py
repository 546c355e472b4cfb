"""One fp64 Cholesky panel (m x w) through sf_chol_panel, for the ncu launch list."""
import sys, torch
sys.path.insert(0, '.')
import paper_1812_02056_b200 as sf
m, w = int(sys.argv[1]), int(sys.argv[2])
info = torch.zeros(1, dtype=torch.int64, device='cuda')
P = torch.randn(w, m, device='cuda', dtype=torch.float64) * 0.01
P.T[:w, :w] += torch.eye(w, device='cuda', dtype=torch.float64) * 4
P0 = P.clone()
for _ in range(3):
    P.copy_(P0)
    assert sf.lib().sf_chol_panel(m, w, 0, P.data_ptr(), m, 0, info.data_ptr(), None) == 0
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
assert sf.lib().sf_chol_panel(m, w, 0, P.data_ptr(), m, 0, info.data_ptr(), None) == 0
e1.record(); torch.cuda.synchronize()
print(f"panel f64 m={m} w={w}: {e0.elapsed_time(e1)*1e3:.1f} us")
