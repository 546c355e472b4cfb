"""Graph-replayed time of small factorizations (lookahead on/off A/B via SF_LOOKAHEAD)."""
import os, sys, torch
sys.path.insert(0, '.')
import paper_1812_02056_b200 as sf, synth
info = torch.zeros(1, dtype=torch.int64, device='cuda')
def t(fn):
    for _ in range(3): fn()
    torch.cuda.synchronize(); ts = []
    for _ in range(9):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[4]
la = os.environ.get("SF_LOOKAHEAD", "1")
for n, s in [(256, 16), (512, 32), (1024, 64), (2000, 200)]:
    A = torch.from_numpy(synth.gen_numpy("spd_shift", n, 0)).cuda(); L = torch.empty_like(A)
    print(f"LA={la} chol n={n} s={s}: {t(lambda: sf.chol_colmajor(n, s, A, n, L, n, info))*1e3:.1f} us")
for n, s in [(1024, 64), (4096, 64)]:
    B = torch.from_numpy(synth.gen_numpy("diag_dominant", n, 0)).cuda().mT.contiguous(); O = torch.empty_like(B)
    print(f"LA={la} lu n={n} s={s}: {t(lambda: sf.lu_colmajor(n, s, B, n, O, n, info))*1e3:.1f} us")
