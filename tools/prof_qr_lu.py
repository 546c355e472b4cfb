"""Representative launches: one MGS panel (n=8192, w=128) and one LU factorization (cfg2)."""
import sys, time
import torch
sys.path.insert(0, '.')
import paper_1812_02056_b200 as sf
import synth
n, w = 8192, 128
V = torch.randn(w, n, device='cuda', dtype=torch.float64)   # column-major n x w
info = torch.zeros(1, dtype=torch.int64, device='cuda')
for _ in range(2):
    V.normal_()
    assert sf.lib().sf_qr_panel(n, w, 0, V.data_ptr(), n, 0, 1e-30, info.data_ptr(), None) == 0
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    assert sf.lib().sf_qr_panel(n, w, 0, V.data_ptr(), n, 0, 1e-30, info.data_ptr(), None) == 0
torch.cuda.synchronize()
print(f"mgs panel n={n} w={w}: {(time.perf_counter()-t0)/5*1e3:.3f} ms (incl. host sync)")
m = 4096
A = synth.gen_torch('diag_dominant', m, 0).mT.contiguous(); LU = torch.empty_like(A)
sf.lu_colmajor(m, 64, A, m, LU, m, info)
torch.cuda.synchronize()
print("ok")
