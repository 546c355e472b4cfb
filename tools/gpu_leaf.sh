# Leaf variants: parity tests (Cholesky) + leaf/panel timings + cfg3 bench, old vs right-looking leaf
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "chol or graph or host or variable or dist" > gpurun_out/leaf_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/leaf_pytest.log
echo "== rl leaf"; timeout 120 python tools/prof_leaf.py
echo "== warp leaf"; SF_LEAF_RL=0 timeout 120 python tools/prof_leaf.py
export SF_BENCH_ALLOW_SHORT=1
for v in 1 0; do
  SF_LEAF_RL=$v timeout 300 python bench.py --workload chol_f64_n16384_s512 --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('RL=$v cfg3', round(d['ms_per_step'],2), 'ms', round(d['value']), d['roofline']['frac'], d['roofline'].get('panel_ms_per_step'))"
done
SF_LEAF_RL=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('RL=1 cfg5', round(d['ms_per_step'],2), 'ms', round(d['value']), d['roofline']['frac'], d['roofline'].get('panel_ms_per_step'))"
