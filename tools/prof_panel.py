"""Standalone panel timings (CUDA events, warm): sf_lu_panel / sf_chol_panel at given sizes.
    python tools/prof_panel.py lu 4096 64        # m, w  (LU: ncr = m - w U columns)
    python tools/prof_panel.py chol 65536 512"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_02056_b200 as sf  # noqa: E402

kind, m, w = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
g = torch.Generator(device="cuda"); g.manual_seed(0)
if kind == "lu":
    P = 2 * torch.rand(m, m, generator=g, device="cuda", dtype=torch.float64) - 1   # column-major m x m
    P.view(-1)[:: m + 1] += m
    call = lambda B: sf.lib().sf_lu_panel(m, w, m - w, 0, B.data_ptr(), m, 0, 1e-300, info.data_ptr(), None)
else:
    R = torch.randn(w, m, generator=g, device="cuda", dtype=torch.float64)
    P = R.clone() / m
    P.view(-1)[:: m + 1] += 1.0       # column j of the buffer: rows 0..m-1 of panel column j
    call = lambda B: sf.lib().sf_chol_panel(m, w, 0, B.data_ptr(), m, 0, info.data_ptr(), None)
info = torch.zeros(1, dtype=torch.int64, device="cuda")
B = P.clone()
for _ in range(3):
    B.copy_(P); assert call(B) == 0
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    B.copy_(P)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); call(B); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1000)
ts.sort()
print(f"{kind} panel m={m} w={w}: median {ts[len(ts) // 2]:.1f} us, min {ts[0]:.1f} us (info {int(info.item())})")
