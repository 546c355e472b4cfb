mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "lu or LU or solve or graph or lookahead" > gpurun_out/lu_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/lu_pytest.log
python tools/prof_luleaf.py && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:lu_leaf --csv python tools/prof_luleaf.py 2>/dev/null | grep -o '"gpu__time_duration.sum","ns","[0-9,.]*"' | head -12
export SF_BENCH_ALLOW_SHORT=1
timeout 300 python bench.py --workload lu_f64_n4096_s64 --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2', round(d['ms_per_step'],3), 'ms', round(d['value']), d['roofline'].get('panel_ms_per_step'))"
