"""Representative fp32 launches for ncu: one fp32 Cholesky panel (m x 512) and/or one 3xTF32
SYRK flush (m x m, k = 512) through the C ABI building blocks.
    python tools/prof_f32.py panel|syrk [m]"""
import sys
import torch
sys.path.insert(0, '.')
import paper_1812_02056_b200 as sf
what = sys.argv[1]
m = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
k = 512
if what == "syrk":
    R = torch.randn(k, m, device='cuda', dtype=torch.float32)
    C = torch.randn(m, m, device='cuda', dtype=torch.float32)
    for _ in range(2):
        assert sf.lib().sf_syrk_sub(m, k, sf.SF_F32, R.data_ptr(), m, C.data_ptr(), m, None) == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        assert sf.lib().sf_syrk_sub(m, k, sf.SF_F32, R.data_ptr(), m, C.data_ptr(), m, None) == 0
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 3
    fl = 3.0 * k * m * (m + 1)
    print(f"syrk f32 m={m} k={k}: {t:.3f} ms (incl. split)  {fl / t / 1e9:.1f} TF/s tensor  {fl / 3 / t / 1e9:.1f} useful")
else:
    P = torch.randn(k, m, device='cuda', dtype=torch.float32)
    P.T[:k, :k] += torch.eye(k, device='cuda') * 1000
    info = torch.zeros(1, dtype=torch.int64, device='cuda')
    Q = P.clone()
    for _ in range(2):
        Q.copy_(P)
        assert sf.lib().sf_chol_panel(m, k, sf.SF_F32, Q.data_ptr(), m, 0, info.data_ptr(), None) == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    Q.copy_(P)
    assert sf.lib().sf_chol_panel(m, k, sf.SF_F32, Q.data_ptr(), m, 0, info.data_ptr(), None) == 0
    e1.record(); torch.cuda.synchronize()
    print(f"panel f32 m={m} w={k}: {e0.elapsed_time(e1):.3f} ms, info={int(info.item())}")
