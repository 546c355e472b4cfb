mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "qr or QR or smoke or graph" > gpurun_out/qr_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/qr_pytest.log
timeout 120 python tools/prof_qr_lu.py 2>&1 | tail -3
export SF_BENCH_ALLOW_SHORT=1
timeout 300 python bench.py --workload qr_f64_n8192_s128 --steps 3 --warmup 3 --no-cpu 2>/dev/null | cut -c1-330
timeout 300 python bench.py --workload qr_f64_n8192_s128 --steps 3 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['roofline'])"
