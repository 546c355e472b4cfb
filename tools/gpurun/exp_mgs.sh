#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/exp_mgs.log
: > $O
timeout 1500 python -m pytest -x -q tests/test_parity_gpu.py -k "qr" >> $O 2>&1
timeout 900 python -m pytest -x -q tests/test_dist_gpu.py tests/test_fp32_gpu.py tests/test_solve_gpu.py -k "qr" >> $O 2>&1
export SF_BENCH_ALLOW_SHORT=1
for v in "SF_MGS_NR=64" "SF_MGS_NR=32"; do
  echo "== $v" >> $O
  env $v python bench.py --workload qr_f64_n8192_s128 --steps 5 --warmup 3 --no-e2e --no-cpu | cut -c1-150 >> $O 2>&1
  env $v python bench.py --workload qr_f32_n8192_s128 --steps 5 --warmup 3 --no-e2e --no-cpu | cut -c1-150 >> $O 2>&1
  env $v python tools/trace.py qr 8192 128 --steps-shown 1 2>&1 | grep -v "^\s*[0-9]" | grep -v Warn | grep -v _warn >> $O
done
cat $O | grep -v "^$"
