"""One short-K flush (LU-style C -= A B, K = 64 and 128) at m = 4032, for ncu."""
import sys, torch
sys.path.insert(0, '.')
import paper_1812_02056_b200 as sf
m = 4032
for k in (64, 128):
    A = torch.randn(k, m, device='cuda', dtype=torch.float64)   # column-major m x k
    B = torch.randn(m, k, device='cuda', dtype=torch.float64)   # column-major k x m
    C = torch.randn(m, m, device='cuda', dtype=torch.float64)
    for _ in range(2):
        assert sf.lib().sf_gemm_sub(m, m, k, 0, A.data_ptr(), m, 0, B.data_ptr(), k, 0, C.data_ptr(), m, None) == 0
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        sf.lib().sf_gemm_sub(m, m, k, 0, A.data_ptr(), m, 0, B.data_ptr(), k, 0, C.data_ptr(), m, None)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"gemm_sub m={m} k={k}: {ms*1e3:.1f} us  {2*m*m*k/ms/1e9:.2f} TF/s")
