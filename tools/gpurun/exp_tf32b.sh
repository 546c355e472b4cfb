#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/exp_tf32b.log
: > $O
timeout 1200 python -m pytest -x -q tests/test_fp32_gpu.py >> $O 2>&1
timeout 900 python -m pytest -x -q tests/test_dist_gpu.py -k "fp32" >> $O 2>&1
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py -k "chol32 or graph or host_lower or qr_rank or qr_mgs or qr_cfg4 or qr_small or qr_wide" >> $O 2>&1
export SF_BENCH_ALLOW_SHORT=1
for v in "SF_TF32_PERSIST_MIN=0" "SF_TF32_RESERVE=16" "SF_TF32_RESERVE=32" "SF_TF32_PERSIST_MIN=300" "SF_TF32_PERSIST_MIN=1000"; do
  echo "== bench $v" >> $O
  env $v python bench.py --workload chol_f32_n65536_s512 --steps 2 --warmup 3 --no-e2e --no-cpu | cut -c1-150 >> $O 2>&1
  env $v python bench.py --workload chol_f32_n16384_s512 --steps 5 --warmup 3 --no-e2e --no-cpu | cut -c1-150 >> $O 2>&1
done
echo "== qr" >> $O
python bench.py --workload qr_f64_n8192_s128 --steps 5 --warmup 3 --no-e2e --no-cpu | cut -c1-150 >> $O 2>&1
python tools/trace.py qr 8192 128 --steps-shown 1 2>&1 | grep -v "^\s*[0-9]" | grep -v Warn | grep -v _warn >> $O
cat $O | grep -v "^$"
