"""Time the Cholesky panel building block alone (m x w, in place) and capture the leaf for ncu."""
import sys, torch
sys.path.insert(0, '.')
import paper_1812_02056_b200 as sf
info = torch.zeros(1, dtype=torch.int64, device='cuda')
for m, w in [(16384, 32), (16384, 64), (16384, 512), (8192, 512)]:
    P = torch.randn(w, m, device='cuda', dtype=torch.float64) * 0.01   # column-major m x w
    P.T[:w, :w] += torch.eye(w, device='cuda', dtype=torch.float64) * 4
    P0 = P.clone()
    def run():
        P.copy_(P0)
        assert sf.lib().sf_chol_panel(m, w, 0, P.data_ptr(), m, 0, info.data_ptr(), None) == 0
    run(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    c0 = torch.cuda.Event(enable_timing=True); c1 = torch.cuda.Event(enable_timing=True)
    c0.record(); [P.copy_(P0) for _ in range(10)]; c1.record()
    e0.record(); [run() for _ in range(10)]; e1.record(); torch.cuda.synchronize()
    print(f"chol panel m={m} w={w}: {(e0.elapsed_time(e1) - c0.elapsed_time(c1)) / 10 * 1e3:.1f} us  info={int(info.item())}")
