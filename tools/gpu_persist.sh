mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "syrk or cfg3 or cfg5 or cfg4 or lu_cfg2 or graph or planted" > gpurun_out/persist_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/persist_pytest.log
for v in 1 0; do echo "PERSIST=$v"; SF_GEMM_PERSIST=$v python tools/prof_syrk_k.py; SF_GEMM_PERSIST=$v python tools/prof_shortk.py; done
export SF_BENCH_ALLOW_SHORT=1
for v in 1 0; do
  SF_GEMM_PERSIST=$v timeout 300 python bench.py --workload chol_f64_n16384_s512 --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PERSIST=$v cfg3', round(d['ms_per_step'],2), 'ms', round(d['value']), round(d['roofline']['frac'],4))"
done
for v in 1 0; do
  SF_GEMM_PERSIST=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PERSIST=$v cfg5', round(d['ms_per_step'],2), 'ms', round(d['value']), round(d['roofline']['frac'],4), d['clocks'])"
done
