"""DMMA flush variants (SF_DMMA / SF_DMMA_BULK / SF_DMMA_SHORTK env): SYRK rate vs K and m."""
import os, sys, torch
sys.path.insert(0, '.')
import paper_1812_02056_b200 as sf
PEAK = 37.037
def run(m, k, reps=5):
    C = torch.randn(m, m, device='cuda', dtype=torch.float64)
    R = torch.randn(k, m, device='cuda', dtype=torch.float64)
    for _ in range(2): sf.lib().sf_syrk_sub(m, k, 0, R.data_ptr(), m, C.data_ptr(), m, None)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): sf.lib().sf_syrk_sub(m, k, 0, R.data_ptr(), m, C.data_ptr(), m, None)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    tf = k * m * (m + 1) / ms / 1e9
    return ms, tf
tag = " ".join(f"{k}={os.environ[k]}" for k in ("SF_DMMA", "SF_DMMA_BULK", "SF_DMMA_SHORTK") if k in os.environ)
for m, k in [(16384, 64), (16384, 128), (16384, 256), (16384, 512), (16384, 1024), (16384, 4096), (32768, 512)]:
    ms, tf = run(m, k)
    print(f"[{tag}] syrk m={m} k={k}: {ms:.3f} ms {tf:.2f} TF/s ({tf / PEAK * 100:.1f}%)", flush=True)
