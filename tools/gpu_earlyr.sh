mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "qr or QR or graph or concurrent or solve" 2>&1 | tail -1
export SF_BENCH_ALLOW_SHORT=1
for v in 1 0 1 0; do
  SF_QR_EARLY_R=$v timeout 300 python bench.py --workload qr_f64_n8192_s128 --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('EARLY=$v cfg4', round(d['ms_per_step'],2), 'ms', round(d['value']), 'upd', round(r['achieved'],2), 'R', round(r['qr_r_ms_per_step'],2), 'panel', round(r['panel_ms_per_step'],2))"
done
python - <<'PY'
import sys, torch, os
sys.path.insert(0, '.')
import paper_1812_02056_b200 as sf, synth
info = torch.zeros(1, dtype=torch.int64, device='cuda')
for n, s in [(8192, 128), (4000, 200), (2000, 100)]:
    A = torch.from_numpy(synth.gen_numpy("gaussian", n, 0)).cuda().mT.contiguous()
    Q = torch.empty_like(A); R = torch.empty_like(A)
    for _ in range(3): sf.qr_colmajor(n, s, A, n, Q, n, R, n, info)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); sf.qr_colmajor(n, s, A, n, Q, n, R, n, info); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"graph qr n={n} s={s}: {sorted(ts)[2]:.2f} ms EARLY={os.environ.get('SF_QR_EARLY_R','1')}")
PY
