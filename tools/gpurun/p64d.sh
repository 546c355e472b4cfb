#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/p64d.log
: > $O
./calib/p64_probe | tail -2 >> $O 2>&1
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py -k "lu_ or graph or variable" >> $O 2>&1
SF_CHOL_P64_MAXM=100000 timeout 900 python -m pytest -x -q tests/test_parity_gpu.py -k "chol_small or chol_cfg1 or planted or not_pd" >> $O 2>&1
SF_CHOL_P64_MAXM=100000 timeout 900 python -m pytest -x -q tests/test_fp32_gpu.py -k "chol" >> $O 2>&1
timeout 900 python -m pytest -x -q tests/test_fp32_gpu.py tests/test_dist_gpu.py -k "lu" >> $O 2>&1
export SF_BENCH_ALLOW_SHORT=1
python bench.py --workload lu_f64_n4096_s64 --steps 20 --warmup 5 --no-e2e --no-cpu | cut -c1-220 >> $O 2>&1
python bench.py --workload lu_f32_n4096_s64 --steps 20 --warmup 5 --no-e2e --no-cpu | cut -c1-220 >> $O 2>&1
for v in 0 100000; do
  echo "== SF_CHOL_P64_MAXM=$v" >> $O
  SF_CHOL_P64_MAXM=$v python bench.py --workload chol_f64_n256_s16 --steps 50 --warmup 5 --no-e2e --no-cpu | cut -c1-220 >> $O 2>&1
  SF_CHOL_P64_MAXM=$v python bench.py --workload chol_f64_n16384_s512 --s 64 --steps 5 --warmup 3 --no-e2e --no-cpu | cut -c1-220 >> $O 2>&1
  SF_CHOL_P64_MAXM=$v python bench.py --workload chol_f64_n16384_s512 --steps 5 --warmup 3 --no-e2e --no-cpu | cut -c1-220 >> $O 2>&1
  SF_CHOL_P64_MAXM=$v python bench.py --workload chol_f32_n16384_s512 --steps 5 --warmup 3 --no-e2e --no-cpu | cut -c1-220 >> $O 2>&1
  SF_CHOL_P64_MAXM=$v python tools/prof_panel.py chol 65536 512 >> $O 2>&1
done
cat $O
