mkdir -p gpurun_out
SF_LEAF_ROT=1 timeout 900 python -m pytest tests -m gpu -x -q -k "chol and not dist" > gpurun_out/rot_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/rot_pytest.log
export SF_BENCH_ALLOW_SHORT=1
for v in 1 0 1 0; do
  SF_LEAF_ROT=$v timeout 300 python bench.py --workload chol_f64_n16384_s512 --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ROT=$v cfg3', round(d['ms_per_step'],2), 'ms', round(d['value']), round(d['roofline']['frac'],4), round(d['roofline'].get('panel_ms_per_step'),2))"
done
for v in 1 0; do
  SF_LEAF_ROT=$v timeout 300 python bench.py --workload chol_f32_n16384_s512 --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ROT=$v cfg3 f32', round(d['ms_per_step'],2), 'ms', round(d['roofline'].get('panel_ms_per_step'),2))"
done
