"""Time single Cholesky leaves (w = 32) and a w = 512 panel at several m (fp64)."""
import sys, torch
sys.path.insert(0, '.')
import paper_1812_02056_b200 as sf
info = torch.zeros(1, dtype=torch.int64, device='cuda')
for m, w in [(2000, 32), (16384, 32), (65536, 32), (2000, 200), (16384, 512), (65536, 512)]:
    P = torch.randn(w, m, device='cuda', dtype=torch.float64) * 0.01
    P.T[:w, :w] += torch.eye(w, device='cuda', dtype=torch.float64) * 4
    P0 = P.clone()
    ts = []
    for it in range(6):
        P.copy_(P0)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        assert sf.lib().sf_chol_panel(m, w, 0, P.data_ptr(), m, 0, info.data_ptr(), None) == 0
        e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"chol panel m={m} w={w}: {sorted(ts[1:])[2]:.1f} us (incl. init/finish_info)")
