mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for v in 1 0; do echo "SHORTK8=$v"; SF_GEMM_SHORTK8=$v python tools/prof_shortk.py; done
export SF_BENCH_ALLOW_SHORT=1
for w in lu_f64_n4096_s64 qr_f64_n8192_s128 chol_f64_n16384_s512; do
for v in 1 0 1 0; do
  SF_GEMM_SHORTK8=$v timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('SHORTK8=$v $w', round(d['ms_per_step'],2), 'ms', 'upd', round(r['achieved'],2), 'panel', round(r['panel_ms_per_step'],2))"
done
done
