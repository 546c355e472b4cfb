#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/exp_tf32.log
: > $O
timeout 1200 python -m pytest -x -q tests/test_fp32_gpu.py >> $O 2>&1
timeout 900 python -m pytest -x -q tests/test_dist_gpu.py -k "fp32" >> $O 2>&1
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py -k "chol32 or graph or host_lower" >> $O 2>&1
for v in "SF_TF32_PERSIST=0" "SF_TF32_TPC=0" "SF_TF32_TPC=2" "SF_TF32_TPC=4" "SF_TF32_TPC=8"; do
  echo "== $v" >> $O
  env $v python tools/prof_f32.py syrk 32768 >> $O 2>&1
  env $v python tools/prof_f32.py syrk 16384 >> $O 2>&1
done
export SF_BENCH_ALLOW_SHORT=1
for v in "SF_TF32_PERSIST=0" "SF_TF32_TPC=0" "SF_TF32_TPC=4" "SF_TF32_TPC=8"; do
  echo "== bench $v" >> $O
  env $v python bench.py --workload chol_f32_n65536_s512 --steps 2 --warmup 3 --no-e2e --no-cpu | cut -c1-330 >> $O 2>&1
  env $v python bench.py --workload chol_f32_n16384_s512 --steps 5 --warmup 3 --no-e2e --no-cpu | cut -c1-330 >> $O 2>&1
done
cat $O | grep -v "^$"
