"""SYRK flush rate vs K (is the 15% DMMA idle in the main loop or in the per-tile prologue/epilogue?)."""
import sys, torch
sys.path.insert(0, '.')
import paper_1812_02056_b200 as sf
m = 16384
C = torch.randn(m, m, device='cuda', dtype=torch.float64)
for k in (128, 256, 512, 1024, 2048, 4096):
    R = torch.randn(k, m, device='cuda', dtype=torch.float64)
    for _ in range(2): sf.lib().sf_syrk_sub(m, k, 0, R.data_ptr(), m, C.data_ptr(), m, None)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): sf.lib().sf_syrk_sub(m, k, 0, R.data_ptr(), m, C.data_ptr(), m, None)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    tf = k * m * (m + 1) / ms / 1e9
    print(f"syrk m={m} k={k}: {ms:.3f} ms {tf:.2f} TF/s ({tf / 37.037 * 100:.1f}% of DMMA peak)")
