mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "qr or QR or graph or lookahead or dist" > gpurun_out/qrw_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/qrw_pytest.log
python - <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_1812_02056_b200 as sf, synth
info = torch.zeros(1, dtype=torch.int64, device='cuda')
for n, s in [(2000, 100), (4000, 200), (8192, 128), (8192, 256), (4000, 400)]:
    A = torch.from_numpy(synth.gen_numpy("paper_spd", n, 0)).cuda().mT.contiguous()
    Q = torch.empty_like(A); R = torch.empty_like(A)
    for _ in range(2): sf.qr_colmajor(n, s, A, n, Q, n, R, n, info)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); sf.qr_colmajor(n, s, A, n, Q, n, R, n, info); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"qr n={n} s={s}: {sorted(ts)[2]:.2f} ms info={int(info.item())}")
PY
