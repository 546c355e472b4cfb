mkdir -p gpurun_out
for v in 1 0; do SF_LU_LEAF_ROT=$v timeout 900 python -m pytest tests -m gpu -x -q -k "lu or LU or solve" 2>&1 | tail -1; done
for v in 1 0; do echo "ROT=$v"; SF_LU_LEAF_ROT=$v ncu --metrics gpu__time_duration.sum --clock-control none -k regex:lu_leaf --csv python tools/prof_luleaf.py 2>/dev/null | grep -o '"gpu__time_duration.sum","ns","[0-9,.]*"' | head -4; done
export SF_BENCH_ALLOW_SHORT=1
for v in 1 0 1 0; do
  SF_LU_LEAF_ROT=$v timeout 300 python bench.py --workload lu_f64_n4096_s64 --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ROT=$v cfg2', round(d['ms_per_step'],3), 'ms', round(d['roofline'].get('panel_ms_per_step'),2))"
done
