mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_strassen_gpu.py -x -q > gpurun_out/strassen_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/strassen_pytest.log
export SF_BENCH_ALLOW_SHORT=1
for w in lu_f64_n4096_s64 qr_f64_n8192_s128 chol_f64_n16384_s512; do
  for st in 0 2048; do
    timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu --no-e2e --strassen $st 2>gpurun_out/strassen_$w.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w strassen=$st', round(d['ms_per_step'],3), 'ms', round(d['value']), 'upd', round(d['roofline']['achieved'],2))"
  done
done
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --strassen 8192 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5 strassen=8192', round(d['ms_per_step'],1), 'ms', round(d['value']), 'upd', round(d['roofline']['achieved'],2))"
