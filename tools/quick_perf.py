"""Quick device-time probe of the three factorizations (development aid, not the bench)."""
import sys, time, json
import torch
sys.path.insert(0, '.')
import paper_1812_02056_b200 as sf
import synth

def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts)

out = {}
info = torch.zeros(1, dtype=torch.int64, device='cuda')
for (n, s) in [(16384, 512), (16384, 256), (16384, 64), (16384, 1024), (16384, 168)]:
    A = synth.gen_torch('spd_scaled', n, 0)
    L = torch.zeros_like(A)
    ms = timeit(lambda: sf.chol_colmajor(n, s, A, n, L, n, info))
    out[f'chol_{n}_{s}'] = {'ms': ms, 'gflops': n**3/3/ms/1e6}
    print(f'chol n={n} s={s}: {ms:.2f} ms  {n**3/3/ms/1e6:.0f} GFLOP/s', flush=True)
    del A, L
n, s = 4096, 64
A = synth.gen_torch('diag_dominant', n, 0); LU = torch.empty_like(A)
ms = timeit(lambda: sf.lu_colmajor(n, s, A, n, LU, n, info))
print(f'lu n={n} s={s}: {ms:.2f} ms {2*n**3/3/ms/1e6:.0f} GFLOP/s', flush=True)
n, s = 8192, 128
A = synth.gen_torch('gaussian', n, 0); Q = torch.empty_like(A); R = torch.empty_like(A)
ms = timeit(lambda: sf.qr_colmajor(n, s, A, n, Q, n, R, n, info))
print(f'qr n={n} s={s}: {ms:.2f} ms {4*n**3/3/ms/1e6:.0f} GFLOP/s classical', flush=True)
# raw SYRK kernel rate
m, k = 16384, 512
Rm = torch.randn(k, m, device='cuda', dtype=torch.float64)  # column-major m x k buffer: rows contiguous
C = torch.randn(m, m, device='cuda', dtype=torch.float64)
ms = timeit(lambda: sf.lib().sf_syrk_sub(m, k, 0, Rm.data_ptr(), m, C.data_ptr(), m, None))
print(f'syrk m={m} k={k}: {ms:.2f} ms {k*m*(m+1)/ms/1e9:.2f} TFLOP/s', flush=True)
Bm = torch.randn(m, k, device='cuda', dtype=torch.float64)
ms = timeit(lambda: sf.lib().sf_gemm_sub(m, m, k, 0, Rm.data_ptr(), m, 0, Bm.data_ptr(), k, 0, C.data_ptr(), m, None))
print(f'gemm NN m={m} k={k}: {ms:.2f} ms {2*k*m*m/ms/1e9:.2f} TFLOP/s', flush=True)
