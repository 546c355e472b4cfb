#!/bin/bash
# one-launch 64-wide panels (panel64.cu): parity + cfg2/cfg1/cfg3 timings
mkdir -p gpurun_out
O=gpurun_out/exp_p64.log
: > $O
timeout 1200 python -m pytest -x -q tests/test_parity_gpu.py -k "lu_ or graph or lookahead or variable or host or qr_rank" >> $O 2>&1
SF_CHOL_P64_MAXM=100000 timeout 900 python -m pytest -x -q tests/test_parity_gpu.py -k "chol_small or chol_cfg1 or planted or not_pd or variable" >> $O 2>&1
SF_CHOL_P64_MAXM=100000 timeout 900 python -m pytest -x -q tests/test_fp32_gpu.py -k "chol" >> $O 2>&1
timeout 900 python -m pytest -x -q tests/test_fp32_gpu.py tests/test_dist_gpu.py -k "lu" >> $O 2>&1
export SF_BENCH_ALLOW_SHORT=1
for v in "SF_LU_P64=0" "SF_LU_P64=1"; do
  echo "== $v" >> $O
  env $v timeout 300 python bench.py --workload lu_f64_n4096_s64 --steps 20 --warmup 5 --no-e2e --no-cpu | cut -c1-200 >> $O 2>&1
  env $v timeout 300 python bench.py --workload lu_f32_n4096_s64 --steps 20 --warmup 5 --no-e2e --no-cpu 2>/dev/null | cut -c1-200 >> $O 2>&1
done
for v in "SF_CHOL_P64_MAXM=0" "SF_CHOL_P64_MAXM=100000"; do
  echo "== $v" >> $O
  env $v timeout 300 python bench.py --workload chol_f64_n256_s16 --steps 50 --warmup 5 --no-e2e --no-cpu | cut -c1-200 >> $O 2>&1
  env $v timeout 300 python bench.py --workload chol_f64_n16384_s512 --steps 5 --warmup 3 --no-e2e --no-cpu | cut -c1-200 >> $O 2>&1
  env $v timeout 300 python bench.py --workload chol_f64_n16384_s512 --s 64 --steps 5 --warmup 3 --no-e2e --no-cpu | cut -c1-200 >> $O 2>&1
  env $v timeout 300 python bench.py --workload chol_f32_n16384_s512 --steps 5 --warmup 3 --no-e2e --no-cpu | cut -c1-200 >> $O 2>&1
done
for v in "SF_MGS_COOP=0" "SF_MGS_COOP=1"; do
  echo "== $v" >> $O
  env $v timeout 300 python bench.py --workload qr_f64_n8192_s128 --steps 5 --warmup 3 --no-e2e --no-cpu | cut -c1-200 >> $O 2>&1
done
grep -v "^$" $O | tail -40
