export SF_BENCH_ALLOW_SHORT=1
for k in 128 256 128 256; do
  for s in 256 512; do
    SF_GEMM_SHORTK8_MAXK=$k timeout 300 python bench.py --workload chol_f64_n16384_s512 --s $s --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('MAXK=$k s=$s cfg3', round(d['ms_per_step'],2), 'ms upd', round(r['achieved'],2), 'panel', round(r['panel_ms_per_step'],2))"
  done
done
