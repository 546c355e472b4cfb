"""DMMA GEMM rate by operand layout (M-major 'nt' as in the flushes vs K-major 'tn'), next to
cuBLAS DGEMM (torch.addmm) on the same shapes and layouts: what the instruction set allows."""
import sys, torch
sys.path.insert(0, '.')
import paper_1812_02056_b200 as sf
PEAK = 37.037
def timeit(f, reps=5):
    for _ in range(2): f()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
L = sf.lib()
for m, k in [(8192, 512), (16384, 512), (16384, 4096), (16384, 128), (16384, 64)]:
    Ct = torch.randn(m, m, device='cuda', dtype=torch.float64)
    At = torch.randn(k, m, device='cuda', dtype=torch.float64)   # A[i + k*lda]: M-major
    Bt = torch.randn(k, m, device='cuda', dtype=torch.float64)
    Ak = torch.randn(m, k, device='cuda', dtype=torch.float64)   # A[k + i*lda]: K-major
    Bk = torch.randn(m, k, device='cuda', dtype=torch.float64)
    fl = 2.0 * m * m * k
    rows = []
    rows.append(("sf nt (M-major A, N-major B)", timeit(lambda: L.sf_gemm_sub(m, m, k, 0, At.data_ptr(), m, 0, Bt.data_ptr(), m, 1, Ct.data_ptr(), m, None))))
    rows.append(("sf tn (K-major both)", timeit(lambda: L.sf_gemm_sub(m, m, k, 0, Ak.data_ptr(), k, 1, Bk.data_ptr(), k, 0, Ct.data_ptr(), m, None))))
    rows.append(("sf nn (M-major A, K-major B)", timeit(lambda: L.sf_gemm_sub(m, m, k, 0, At.data_ptr(), m, 0, Bk.data_ptr(), k, 0, Ct.data_ptr(), m, None))))
    rows.append(("cublas nt", timeit(lambda: Ct.addmm_(Bt.T, At, alpha=-1.0))))
    rows.append(("cublas tn", timeit(lambda: Ct.addmm_(Bk, Ak.T, alpha=-1.0))))
    rows.append(("cublas nn", timeit(lambda: Ct.addmm_(Bk, At, alpha=-1.0))))
    for name, ms in rows:
        tf = fl / ms / 1e9
        print(f"m={m} k={k} {name}: {ms:.3f} ms {tf:.2f} TF/s ({tf / PEAK * 100:.1f}%)", flush=True)
