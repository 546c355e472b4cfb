#!/bin/bash
# DMMA flush variant sweep: SF_DMMA selects the tile variant.
mkdir -p gpurun_out
O=gpurun_out/exp_dmma2.log
: > $O
for v in "SF_DMMA=0" "SF_DMMA=4" "SF_DMMA=3" "SF_DMMA=2" "SF_DMMA=5" "SF_DMMA=6" "SF_DMMA=3 SF_DMMA_SHORTK=3" "SF_DMMA=3 SF_DMMA_SHORTK=5" "SF_DMMA=3 SF_DMMA_SHORTK=6"; do
  env $v timeout 300 python tools/exp_dmma.py >> $O 2>&1
done
for v in "SF_DMMA=3 SF_DMMA_SHORTK=3" "SF_DMMA=5 SF_DMMA_SHORTK=5"; do
  env $v timeout 900 python -m pytest -x -q tests/test_parity_gpu.py -k "chol_small_grid or lu_small_grid or qr_small_grid or planted or syrk or cfg1 or cfg2 or graph" >> $O 2>&1
done
for v in "SF_DMMA=3 SF_DMMA_SHORTK=3" "SF_DMMA=5 SF_DMMA_SHORTK=5"; do
  echo "== bench $v" >> $O
  env $v SF_BENCH_ALLOW_SHORT=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu >> $O 2>&1
  env $v SF_BENCH_ALLOW_SHORT=1 timeout 600 python bench.py --workload lu_f64_n4096_s64 --steps 10 --warmup 3 --no-e2e --no-cpu >> $O 2>&1
  env $v SF_BENCH_ALLOW_SHORT=1 timeout 600 python bench.py --workload qr_f64_n8192_s128 --steps 5 --warmup 3 --no-e2e --no-cpu >> $O 2>&1
  env $v SF_BENCH_ALLOW_SHORT=1 timeout 600 python bench.py --workload chol_f64_n16384_s512 --steps 5 --warmup 3 --no-e2e --no-cpu >> $O 2>&1
done
cat $O | grep -v "^$" | cut -c1-300
